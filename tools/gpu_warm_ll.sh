# prep-kernel parity, phase timings of the current build vs a saved one, and
# ncu launch lists (per-kernel device time) of cfg4 plans for two builds (warm-start A/B)
set -x
python -m pytest tests/test_gpu_prep.py -q -p no:cacheprovider -x > gpurun_out/prep_tests.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/prep_tests.log
python tools/plan_timing.py paper_2010_05371_b200/libeapdtw_b200.so bisect_libs/lib_fix2.so 2>&1 | tail -2
export REPS=2
for f in lib_fd1975a lib_fix2; do
  /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/warm_$f.csv \
    python tools/plan_timing.py bisect_libs/$f.so > gpurun_out/warm_$f.log 2>&1
  echo "rc=$?"
done
