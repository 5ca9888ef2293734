# full GPU test suite + default bench
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/r2_gputest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r2_gputest.log
grep -a "criterion" gpurun_out/r2_gputest.log | head -12
python bench.py --steps 5 --warmup 3 > gpurun_out/r2_bench_cfg4.json 2> gpurun_out/r2_bench_cfg4.err; echo "bench rc=$?"
cut -c1-400 gpurun_out/r2_bench_cfg4.json
