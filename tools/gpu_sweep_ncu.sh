# ncu --set full of the cfg4 sweep launch (3rd search_kernel launch of a plan) + plain timing first
set -x
REPS=2 python tools/plan_timing.py paper_2010_05371_b200/libeapdtw_b200.so 2>&1 | tail -1
REPS=2 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:search_kernel --launch-skip 2 -c 1 \
  -o gpurun_out/sweep_full --force-overwrite python tools/plan_timing.py paper_2010_05371_b200/libeapdtw_b200.so > gpurun_out/sweep_ncu.log 2>&1; echo "ncu rc=$?"
