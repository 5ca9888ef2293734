#!/bin/bash
# A/B: the in-tree .so (base) vs scratch/variants/$1.so on the given configs
V=$1; shift
L=paper_2010_05371_b200/libeapdtw_b200.so
cp $L /tmp/base.so
ms() { python bench.py --config $1 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],2), d.get('result', ''))"; }
for v in base $V base $V; do
  if [ $v = base ]; then cp /tmp/base.so $L; else cp scratch/variants/$v.so $L; fi
  line="$v"
  for c in "$@"; do line="$line | $c $(ms $c)"; done
  echo "$line"
done
cp /tmp/base.so $L
