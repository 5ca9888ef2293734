for f in bisect_libs/lib_lanes32.so bisect_libs/lib_lanes16.so bisect_libs/lib_lanes8.so; do
  python tools/plan_timing.py $f 2>&1 | tail -1
  OPTS=prep_overlap=0 python tools/plan_timing.py $f 2>&1 | tail -1
done
