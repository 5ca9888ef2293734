# ncu --set full of the cfg4 search_kernel launches (warm-up wave, rank cascade, sweep)
set -x
python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_plain.json 2> gpurun_out/ncu_plain.err && \
/usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:search_kernel -c 3 \
    -o gpurun_out/r2_sweep python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_run.log 2>&1
echo "ncu rc=$?"
tail -3 gpurun_out/ncu_run.log
