# A/B: the dropped probe's frontier minimum in the continuing pass's bound
set -x
for rep in 1 2; do
  OPTS="" python tools/plan_timing.py bisect_libs/lib_ec.so 2>&1 | tail -1
  for o in "probe_excess=0" "probe_excess=1"; do
    OPTS=$o python tools/plan_timing.py bisect_libs/lib_px2.so 2>&1 | tail -1
  done
done
for c in cfg3 cfg2; do for o in "probe_excess=0" "probe_excess=1"; do CFG=$c OPTS=$o python tools/plan_timing.py bisect_libs/lib_px2.so 2>&1 | tail -1; done; done
python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/px_cfg4.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/px_cfg4.json'));print('cfg4', d['ms_per_step'], d['sweep_counters'], d['result'])"
python bench.py --config cfg3-nolb --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/px_cfg3n.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/px_cfg3n.json'));print('cfg3-nolb', d['ms_per_step'], d['result'])"
python -m pytest tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider -x 2>&1 | tail -3
