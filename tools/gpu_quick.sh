set -x
python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "long_series" > gpurun_out/quick_tests.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/quick_tests.log
