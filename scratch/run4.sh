timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/b_cfg4.json 2> gpurun_out/b_cfg4.err; echo rc=$?
