#!/bin/bash
# cfg4 total/phase times for warm-start knob settings (one box, back to back)
for r in "16:16384" "32:16384" "16:8192" "32:8192" "8:16384" "16:32768"; do
  EAPDTW_RANK=$r python bench.py --no-cpu-baseline --steps 5 --warmup 3 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$r', round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['phase_ms'].items()}, d['result'])"
done
