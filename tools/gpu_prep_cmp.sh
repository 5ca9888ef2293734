# phase timings of chain-kernel variants at cfg2/3/4 (+ prep parity of each)
set -x
for f in bisect_libs/lib_tile64.so bisect_libs/lib_tile128.so; do
  cp $f paper_2010_05371_b200/libeapdtw_b200.so
  python -m pytest tests/test_gpu_prep.py -q -p no:cacheprovider -x -k stats 2>&1 | tail -1
  for c in cfg2 cfg3 cfg4; do CFG=$c python tools/plan_timing.py $f 2>&1 | tail -1; done
done
