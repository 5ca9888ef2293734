# ncu launch lists (per-kernel device time) of a cfg4 plan for two library builds (warm-start A/B)
set -x
for f in lib_fd1975a lib_fix2; do
  /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/warm_$f.csv \
    REPS=2 python tools/plan_timing.py bisect_libs/$f.so > gpurun_out/warm_$f.log 2>&1
  echo "rc=$?"
done
