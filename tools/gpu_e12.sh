# A/B: per-step band test dropped in the FP32 screen; LB producers by SM
set -x
for rep in 1 2; do
for f in bisect_libs/lib_head.so bisect_libs/lib_noband.so; do
  for o in "" "producer_sms=3" "producer_sms=4" "producer_sms=2"; do
    OPTS=$o python tools/plan_timing.py $f 2>&1 | tail -1
  done
done
done
for c in cfg3 cfg2; do for f in bisect_libs/lib_head.so bisect_libs/lib_noband.so; do CFG=$c python tools/plan_timing.py $f 2>&1 | tail -1; done; done
cp bisect_libs/lib_noband.so paper_2010_05371_b200/libeapdtw_b200.so
python -m pytest tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider -x 2>&1 | tail -3
for c in cfg3-nolb cfg5; do python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/e12_$c.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/e12_$c.json'));print('noband $c', d['ms_per_step'])"; done
