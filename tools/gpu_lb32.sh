# A/B: LB_Keogh terms in FP32
set -x
for rep in 1 2 3; do for f in lib_l64 lib_l32; do python tools/plan_timing.py bisect_libs/$f.so 2>&1 | tail -1; done; done
for c in cfg3 cfg2; do for f in lib_l64 lib_l32; do CFG=$c python tools/plan_timing.py bisect_libs/$f.so 2>&1 | tail -1; done; done
cp bisect_libs/lib_l32.so paper_2010_05371_b200/libeapdtw_b200.so
python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/k.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/k.json'));print('cfg4 l32', d['ms_per_step'], d['sweep_counters'], d['result'])"
python -m pytest tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider -x 2>&1 | tail -3
