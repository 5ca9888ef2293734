# full GPU suite + default bench line
set -x
python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/gpu_tests.log
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/bench_cfg4.json'));print(d['ms_per_step'], d.get('phase_ms'), d['e2e'])"
