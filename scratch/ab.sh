for cfg in "0 16" "1 16" "3 16" "5 16"; do
  set -- $cfg
  for c in cfg3 cfg3-nolb cfg4; do
    export EAPDTW_AD_K=$1
    export EAPDTW_SCREEN_ROWS=$2
    timeout 200 python bench.py --config $c --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ab_${1}_${2}_$c.json 2> gpurun_out/ab_${1}_${2}_$c.err
    echo "K=$1 R=$2 $c rc=$?"
  done
done
