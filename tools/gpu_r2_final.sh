# round-2 final evidence: GPU tests, every bench line, launch lists, ncu --set full captures, shard emulation
set -x
python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/r2_gputest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2_gputest.log
python bench.py --steps 10 --warmup 3 > gpurun_out/r2_bench_cfg4.json 2> gpurun_out/r2_bench_cfg4.err; echo "bench rc=$?"
for c in cfg1 cfg2 cfg3 cfg3-nolb cfg5 grid; do
  python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/r2_bench_$c.json 2> gpurun_out/r2_bench_$c.err; echo "bench $c rc=$?"
done
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2_bench_ref.json 2> gpurun_out/r2_bench_ref.err; echo "ref rc=$?"
python tools/shard_emul.py 1 2 4 8 > gpurun_out/r2_shard_emul.txt 2>&1; echo "shard rc=$?"
for c in cfg4 cfg3; do
python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ll_plain_$c.json 2>&1 && \
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_$c.csv \
    python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ll_ncu_$c.log 2>&1
echo "ll $c rc=$?"
done
python tools/prep_profile.py > gpurun_out/prep_plain.log 2>&1 && \
/usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:'stats_|envelope' -c 6 \
   -o gpurun_out/r2_prep --force-overwrite python tools/prep_profile.py > gpurun_out/prep_ncu.log 2>&1; echo "prep ncu rc=$?"
/usr/local/cuda/bin/ncu --set full --clock-control none -k regex:'fast_stats|stats_verify' -c 2 \
   -o gpurun_out/r2_spec --force-overwrite python bench.py --config cfg3 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/spec_ncu.log 2>&1; echo "spec ncu rc=$?"
REPS=2 python tools/plan_timing.py paper_2010_05371_b200/libeapdtw_b200.so 2>&1 | tail -1
REPS=2 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:search_kernel --launch-skip 2 -c 1 \
  -o gpurun_out/r2_sweep_full --force-overwrite python tools/plan_timing.py paper_2010_05371_b200/libeapdtw_b200.so > gpurun_out/sweep_ncu.log 2>&1; echo "ncu rc=$?"
python bench.py --config cfg5 --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1 && \
/usr/local/cuda/bin/ncu --set full --clock-control none -k regex:nn1_kernel -c 1 \
  -o gpurun_out/r2_nn1 --force-overwrite python bench.py --config cfg5 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/nn1_ncu.log 2>&1; echo "nn1 ncu rc=$?"
ls -la gpurun_out | head -60
