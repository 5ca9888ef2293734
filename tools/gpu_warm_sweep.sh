# warm-start knobs at cfg3 / cfg2 with the round-2 engine (speculative statistics on)
set -x
L=paper_2010_05371_b200/libeapdtw_b200.so
for c in cfg3 cfg2; do
for o in "" "rank_k=8192" "rank_k=4096" "rank_k=2048" "rank_k=1024" "rank_stride=32" "rank_stride=64" "rank_k=4096,rank_stride=32" "rank_k=2048,rank_stride=64" "probe=512" "probe=512,rank_k=4096" "rank_stride=0" "probe_warm=1" ""; do
  CFG=$c OPTS=$o python tools/plan_timing.py $L 2>&1 | tail -1
done
done
