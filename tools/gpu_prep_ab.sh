# prep parity + cfg4 phase timings of the current build + ncu full captures of the prep kernels
set -x
python -m pytest tests/test_gpu_prep.py -q -p no:cacheprovider -x > gpurun_out/prep_tests.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/prep_tests.log
python tools/plan_timing.py paper_2010_05371_b200/libeapdtw_b200.so 2>&1 | tail -1
python tools/prep_profile.py > gpurun_out/prep_plain.log 2>&1; echo "plain rc=$?"
/usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:"stats_chain" -c 1 \
  -o gpurun_out/prep_full --force-overwrite python tools/prep_profile.py > gpurun_out/prep_ncu.log 2>&1; echo "ncu rc=$?"
