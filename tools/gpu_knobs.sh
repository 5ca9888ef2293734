# option sweeps on the round-2 engine
set -x
L=paper_2010_05371_b200/libeapdtw_b200.so
for o in "" "screen_rows=0" "screen_rows=4" "screen_rows=8" "cb_strip=2" "probe=4096" ""; do
  OPTS=$o python tools/plan_timing.py $L 2>&1 | tail -1
done
for o in "" "nn1_splits=6" "nn1_splits=8" "nn1_splits=12" "nn1_splits=16" "nn1_splits=24" "probe_strips=0" "probe_strips=2" "nn1_warm=0" ""; do
  a=""; for kv in $(echo $o | tr ',' ' '); do a="$a --opt $kv"; done
  python bench.py --config cfg5 --steps 3 --warmup 2 --no-cpu-baseline $a > gpurun_out/k.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/k.json'));print('cfg5 [$o]', round(d['ms_per_step'],2))"
done
for o in "" "screen_rows=0" "screen_rows=4" "screen_rows=8" "probe_strips=2" "probe_strips=0"; do
  a=""; for kv in $(echo $o | tr ',' ' '); do a="$a --opt $kv"; done
  python bench.py --config cfg3-nolb --steps 3 --warmup 2 --no-cpu-baseline $a > gpurun_out/k.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/k.json'));print('cfg3-nolb [$o]', round(d['ms_per_step'],2))"
done
