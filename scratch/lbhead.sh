for h in 64 128 256 512 100000; do for c in cfg3 cfg4; do
  EAPDTW_LB_HEAD=$h timeout 200 python bench.py --config $c --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/lbh_${h}_$c.json 2> gpurun_out/lbh_${h}_$c.err
done; done
