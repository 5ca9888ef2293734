for c in cfg2 cfg3 cfg3-nolb cfg4; do
  timeout 200 python bench.py --config $c --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/co_$c.json 2> gpurun_out/co_$c.err
done
