# warm-start option A/B at cfg4 (phase timings)
for o in "" probe_warm=0 warm_f32=0 probe_warm=0,warm_f32=0 probe_warm=0,rank_ub=0 rank_k=8192 rank_k=32768; do
  OPTS=$o python tools/plan_timing.py paper_2010_05371_b200/libeapdtw_b200.so 2>&1 | tail -1
done
