# speculative statistics: parity, then A/B at cfg2/3/4
set -x
python -m pytest tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider -x -k "speculative" 2>&1 | tail -15
python -m pytest tests -q -m gpu -p no:cacheprovider -x 2>&1 | tail -4
for c in cfg2 cfg3 cfg4; do
  python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/spec_${c}.json 2> gpurun_out/spec_${c}.err; echo "rc=$?"
  python -c "import json;d=json.load(open('gpurun_out/spec_${c}.json'));print('$c', round(d['ms_per_step'],3), d['phase_ms'], d['speculative_stats'], d['prep_kernels'])"
done
