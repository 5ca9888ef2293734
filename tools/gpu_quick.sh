# quick GPU check: probe tests + benches for probe_strips 0/1
set -x
python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "probe or baseline_configs" > gpurun_out/quick_tests.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/quick_tests.log
for c in cfg4 cfg3-nolb cfg3; do for k in 1 0; do
  python bench.py --config $c --steps 5 --warmup 2 --no-cpu-baseline --opt probe_strips=$k > gpurun_out/q.json 2> gpurun_out/q_err.txt; echo "bench $c k=$k rc=$?"
  python -c "import json;d=json.load(open('gpurun_out/q.json'));print('$c k=$k', d['ms_per_step'], d['phase_ms'], d['sweep_counters'])"
done; done
for k in 1 0; do
  python bench.py --config cfg5 --steps 3 --warmup 1 --opt probe_strips=$k > gpurun_out/q.json 2>> gpurun_out/q_err.txt; echo "bench cfg5 k=$k rc=$?"
  python -c "import json;d=json.load(open('gpurun_out/q.json'));print('cfg5 k=$k', d['ms_per_step'], d['cells_per_step'])"
done
