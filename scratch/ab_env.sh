# usage: bash scratch/ab_env.sh "NAME=ENVSTR ..." "cfgs" steps rounds   (ENVSTR: comma-separated K=V)
for r in $(seq 1 $4); do for spec in $1; do name=${spec%%=*}; envs=${spec#*=}
  for c in $2; do env $(echo $envs | tr ',' ' ') timeout 300 python bench.py --config $c --steps $3 --warmup 2 --no-cpu-baseline > gpurun_out/ab_${name}_${c}_$r.json 2> gpurun_out/ab_${name}_${c}_$r.err; done; done; done
