# copy one tools/gpu_r2_final.sh run from gpurun_out/ into profiles/ and regenerate the summaries
set -e
for c in cfg4 cfg1 cfg2 cfg3 cfg3-nolb cfg5 grid ref; do cp gpurun_out/r2_bench_$c.json profiles/r2_bench_$c.json; done
cp gpurun_out/r2_launches_cfg4.csv profiles/r2_cfg4_launches.csv
cp gpurun_out/r2_launches_cfg3.csv profiles/r2_cfg3_launches.csv
cp gpurun_out/r2_shard_emul.txt profiles/r2_shard_emul.txt
python profiles/summarize.py launches profiles/r2_cfg4_launches.csv profiles/r2_cfg4_launches.md > /dev/null
python profiles/summarize.py launches profiles/r2_cfg3_launches.csv profiles/r2_cfg3_launches.md > /dev/null
python profiles/summarize.py report gpurun_out/r2_sweep_full.ncu-rep profiles/r2_cfg4_search_kernel_ncu.txt cfg4 | tail -1
python profiles/summarize.py report gpurun_out/r2_nn1.ncu-rep profiles/r2_cfg5_nn1_kernel_ncu.txt cfg5 | tail -1
ncu -i gpurun_out/r2_sweep_full.ncu-rep --page source --csv --print-source sass > gpurun_out/r2_sweep_src.csv 2>/dev/null
rm -rf /tmp/cub && mkdir /tmp/cub
(cd /tmp/cub && cuobjdump -xelf kernels.sm_100a.cubin $OLDPWD/paper_2010_05371_b200/libeapdtw_b200.so > /dev/null && nvdisasm -g -c kernels.sm_100a.cubin > lines.txt 2>/dev/null)
python tools/ncu_regions.py gpurun_out/r2_sweep_src.csv /tmp/cub/lines.txt "search_kernelILi0ELb0ELb0" 100000 > /tmp/regions.txt 2>&1
python tools/bench_table.py
