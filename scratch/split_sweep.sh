#!/bin/bash
# cfg4 e2e (host-pointer, streamed) vs part-1 share in eighths
for r in 1 2; do for sp in 2 3 4; do
  EAPDTW_STREAM_SPLIT=$sp python bench.py --no-cpu-baseline 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('split $sp', round(d['ms_per_step'],2), '%.4g' % d['e2e']['value'], round(1e8/d['e2e']['value']*1e3,2), 'ms')"
done; done
