cp scratch/variants/clk.so paper_2010_05371_b200/libeapdtw_b200.so
for c in cfg4 cfg3-nolb cfg5; do timeout 300 python bench.py --config $c --no-cpu-baseline --steps 1 --warmup 1 > gpurun_out/clk_$c.json 2> gpurun_out/clk_$c.err; done
cp scratch/variants/blk.so paper_2010_05371_b200/libeapdtw_b200.so
