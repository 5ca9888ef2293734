# stats-chain variants (lanes_tile_depth) and warm-start probe options: cfg4 phase timings
set -x
for f in bisect_libs/lib_chain_*.so; do python tools/plan_timing.py $f 2>&1 | tail -1; done
OPTS=probe_warm=0 python tools/plan_timing.py bisect_libs/lib_chain_32_64_3.so 2>&1 | tail -1
OPTS=probe_strips=0 python tools/plan_timing.py bisect_libs/lib_chain_32_64_3.so 2>&1 | tail -1
