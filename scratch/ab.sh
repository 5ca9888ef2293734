for c in cfg3 cfg3-nolb cfg4; do
  timeout 200 python bench.py --config $c --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/seed0_$c.json 2> gpurun_out/seed0_$c.err
done
EAPDTW_SEED_UB=4.632683082896913 timeout 200 python bench.py --config cfg3 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/seed1_cfg3.json 2>&1
EAPDTW_SEED_UB=4.632683082896913 timeout 200 python bench.py --config cfg3-nolb --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/seed1_cfg3-nolb.json 2>&1
EAPDTW_SEED_UB=3.748871965313156 timeout 200 python bench.py --config cfg4 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/seed1_cfg4.json 2>&1
