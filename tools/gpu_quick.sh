set -x
for o in "probe_warm=1" "probe_warm=0"; do
  python bench.py --steps 5 --warmup 2 --no-cpu-baseline --opt $o > gpurun_out/q.json 2> gpurun_out/q_err.txt; echo "bench cfg4 $o rc=$?"
  python -c "import json;d=json.load(open('gpurun_out/q.json'));print('cfg4 $o', d['ms_per_step'], d['phase_ms'])"
done
cd paper_2010_05371_b200 && /usr/local/cuda/bin/nvcc -O3 -lineinfo -std=c++17 -fmad=false -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC,-ffp-contract=off -DEAPDTW_SEARCH_STEP_BLOCK=16 -DEAPDTW_NN1_STEP_BLOCK=16 -shared -o libeapdtw_b200.so csrc/kernels.cu csrc/capi.cu csrc/trace.cu csrc/bounds.cu && cd ..
for c in cfg4 cfg3-nolb; do
  python bench.py --config $c --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/q.json 2> gpurun_out/q_err.txt; echo "bench BLK16 $c rc=$?"
  python -c "import json;d=json.load(open('gpurun_out/q.json'));print('BLK16 $c', d['ms_per_step'], d['phase_ms'])"
done
python bench.py --config cfg5 --steps 3 --warmup 1 > gpurun_out/q.json 2>> gpurun_out/q_err.txt; echo "bench BLK16 cfg5 rc=$?"
python -c "import json;d=json.load(open('gpurun_out/q.json'));print('BLK16 cfg5', d['ms_per_step'])"
