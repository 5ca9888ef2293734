for v in $1; do cp scratch/variants/$v.so paper_2010_05371_b200/libeapdtw_b200.so; timeout 120 python scratch/stats_time.py $v >> gpurun_out/stats_var.txt 2>&1; done
