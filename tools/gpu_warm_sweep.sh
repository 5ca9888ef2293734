# warm-start knobs at cfg4 with the round-2 engine
set -x
L=paper_2010_05371_b200/libeapdtw_b200.so
for o in "" "rank_k=8192" "rank_k=4096" "rank_k=32768" "rank_stride=32" "rank_stride=8" "rank_ub_k=32" "rank_ub_k=8" "rank_ub_w=2" "rank_ub_w=8" "probe_warm=1" "warm_f32=0" "rank_k=8192,rank_stride=32"; do
  OPTS=$o python tools/plan_timing.py $L 2>&1 | tail -1
done
OPTS="" python tools/plan_timing.py $L 2>&1 | tail -1
