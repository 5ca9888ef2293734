# ncu launch lists of cfg4 plans for stats-chain variants
export REPS=2
for f in lib_chain_32_64_3 lib_chain_16_128_3; do
  /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/chain_$f.csv \
    python tools/plan_timing.py bisect_libs/$f.so > gpurun_out/chain_$f.log 2>&1
  echo "rc=$?"
done
