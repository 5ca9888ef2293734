set -x
python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "probe or baseline_configs or nn1" > gpurun_out/quick_tests.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/quick_tests.log
for c in cfg4 cfg3-nolb cfg3 cfg2; do
  python bench.py --config $c --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/q.json 2> gpurun_out/q_err.txt; echo "bench $c rc=$?"
  python -c "import json;d=json.load(open('gpurun_out/q.json'));print('$c', d['ms_per_step'], d['phase_ms'], d['result'])"
done
python bench.py --config cfg5 --steps 3 --warmup 1 > gpurun_out/q.json 2>> gpurun_out/q_err.txt; echo "bench cfg5 rc=$?"
python -c "import json;d=json.load(open('gpurun_out/q.json'));print('cfg5', d['ms_per_step'], d['cells_per_step'])"
