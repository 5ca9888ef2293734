# full GPU test suite + default bench
set -x
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2_gputest.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/r2_gputest.log
python -m pytest tests/test_acceptance_gpu.py -m gpu -q -s -p no:cacheprovider 2>&1 | grep -a "criterion"
