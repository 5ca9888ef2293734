set -x
for f in bisect_libs/lib_fd1975a.so bisect_libs/lib_fix.so bisect_libs/lib_fix2.so bisect_libs/lib_9a2fe7a.so bisect_libs/lib_fix2.so; do
  python tools/plan_timing.py $f 2>&1 | tail -1
done
