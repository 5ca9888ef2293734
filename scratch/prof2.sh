set -x
cp scratch/variants/clk.so paper_2010_05371_b200/libeapdtw_b200.so
timeout 300 python bench.py --no-cpu-baseline --steps 2 --warmup 1 > gpurun_out/clk_cfg4.json 2> gpurun_out/clk_cfg4.err; echo rc=$?
timeout 300 python bench.py --config cfg3-nolb --no-cpu-baseline --steps 2 --warmup 1 > gpurun_out/clk_nolb.json 2> gpurun_out/clk_nolb.err; echo rc=$?
cp scratch/variants/base.so paper_2010_05371_b200/libeapdtw_b200.so
timeout 600 ncu --set full --clock-control none --import-source on -k regex:search_kernel -s 2 -c 1 -o gpurun_out/prof_cfg4_f32 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_f.log 2>&1; echo ncu_f=$?
