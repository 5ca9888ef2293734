# phase-clock build of the library (warp-cycles per phase of the sweep, strips per DTW task), cfg4
set -x
cd paper_2010_05371_b200 && /usr/local/cuda/bin/nvcc -O3 -lineinfo -std=c++17 -fmad=false -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC,-ffp-contract=off -DEAPDTW_PHASE_CLOCKS -shared -o libeapdtw_b200.so csrc/kernels.cu csrc/capi.cu csrc/trace.cu csrc/bounds.cu && cd ..
for k in 1 0; do
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --opt probe_strips=$k > gpurun_out/ph.json 2> gpurun_out/ph_k$k.err; echo "rc=$?"
  grep -a "phase warp\|lane eff\|strips/DTW" gpurun_out/ph_k$k.err | tail -9
done
