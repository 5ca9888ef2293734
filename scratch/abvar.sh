# usage: bash scratch/abvar.sh "v1 v2 ..." "cfgA cfgB" steps rounds
for r in $(seq 1 $4); do for v in $1; do cp scratch/variants/$v.so paper_2010_05371_b200/libeapdtw_b200.so
  for c in $2; do timeout 300 python bench.py --config $c --steps $3 --warmup 2 --no-cpu-baseline > gpurun_out/ab_${v}_${c}_$r.json 2> gpurun_out/ab_${v}_${c}_$r.err; done; done; done
