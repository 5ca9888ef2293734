for r in 1 2; do for v in base nn3; do cp scratch/variants/$v.so paper_2010_05371_b200/libeapdtw_b200.so; timeout 300 python bench.py --config cfg5 --steps 2 --warmup 1 > gpurun_out/nn_${v}_$r.json 2>/dev/null; done; done
cp scratch/variants/base.so paper_2010_05371_b200/libeapdtw_b200.so
