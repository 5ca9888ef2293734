set -x
for rep in 1 2; do for f in lib_g8 lib_g16 lib_g4; do python tools/plan_timing.py bisect_libs/$f.so 2>&1 | tail -1; done; done
