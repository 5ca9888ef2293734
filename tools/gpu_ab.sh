# A/B of two library builds: cfg4 and cfg3 phase timings, alternating
for c in cfg4 cfg3; do
  for f in bisect_libs/lib_head.so bisect_libs/lib_f2.so bisect_libs/lib_head.so bisect_libs/lib_f2.so; do CFG=$c python tools/plan_timing.py $f 2>&1 | tail -1; done
done
