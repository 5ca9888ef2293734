#!/bin/bash
# cfg5 device time vs database splits per query (blocks = 1000 x splits)
for sp in ${SPLITS:-2 3 4 6 8}; do
  EAPDTW_NN1_SPLITS=$sp python bench.py --config cfg5 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('splits $sp', round(d['ms_per_step'],2), d['cells_per_step'])"
done
