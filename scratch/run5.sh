timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
bash scratch/abvar.sh "lbf64 lbf32" "cfg4 cfg3 cfg2" 3 2
cp scratch/variants/lbf32.so paper_2010_05371_b200/libeapdtw_b200.so
bash scratch/ab_env.sh "ovl0=EAPDTW_OVERLAP_PREP=0 ovl1=EAPDTW_OVERLAP_PREP=1" "cfg4" 3 2
