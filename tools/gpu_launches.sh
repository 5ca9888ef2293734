# ncu launch list (per-kernel device time, cold-cache serialised) of one default bench step
set -x
python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ll_plain.json 2>&1 && \
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ll_ncu.log 2>&1
echo "rc=$?"
