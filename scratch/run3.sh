set -x
timeout 300 python bench.py --config cfg5 > gpurun_out/b_cfg5_f1.json 2> gpurun_out/b_cfg5_f1.err; echo rc=$?
EAPDTW_F32=0 timeout 300 python bench.py --config cfg5 > gpurun_out/b_cfg5_f0.json 2> gpurun_out/b_cfg5_f0.err; echo rc=$?
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/b_cfg4.json 2> gpurun_out/b_cfg4.err; echo rc=$?
bash scratch/ab_env.sh "c64=EAPDTW_COARSE_STRIDE=64 c0=EAPDTW_COARSE_STRIDE=0 c128=EAPDTW_COARSE_STRIDE=128 c256=EAPDTW_COARSE_STRIDE=256 p256=EAPDTW_PROBE=256 c512_64=EAPDTW_COARSE_STRIDE=512:64" "cfg4" 3 1
