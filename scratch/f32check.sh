set -x
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_gpu.log
for f in 1 0; do
  EAPDTW_F32=$f timeout 300 python bench.py --no-cpu-baseline > gpurun_out/b_cfg4_f$f.json 2> gpurun_out/b_cfg4_f$f.err; echo rc=$?
  EAPDTW_F32=$f timeout 300 python bench.py --config cfg3-nolb --no-cpu-baseline > gpurun_out/b_nolb_f$f.json 2> gpurun_out/b_nolb_f$f.err; echo rc=$?
done
