#!/bin/bash
# A/B of the FP32 engine's step-block size in the search: base (4) vs s8 (8)
L=paper_2010_05371_b200/libeapdtw_b200.so
cp $L /tmp/base.so
ms() { python bench.py --config $1 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],2), d.get('result', ''))"; }
for v in base s8 base s8; do
  if [ $v = base ]; then cp /tmp/base.so $L; else cp scratch/variants/$v.so $L; fi
  echo "$v cfg4 $(ms cfg4)  cfg3-nolb $(ms cfg3-nolb) cfg3 $(ms cfg3)"
done
cp /tmp/base.so $L
echo "base cfg5 $(ms cfg5)"
