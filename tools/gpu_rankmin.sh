# rank_min rule: tests + bench lines of the small configs
set -x
python -m pytest tests -q -m gpu -p no:cacheprovider -x 2>&1 | tail -3
for c in cfg2 cfg3 cfg3-nolb grid cfg4; do
  python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/r2_bench_$c.json 2> gpurun_out/r2_bench_$c.err; echo "bench $c rc=$?"
  python -c "import json;d=json.load(open('gpurun_out/r2_bench_$c.json'));print('$c', round(d['ms_per_step'],3), '%.3e'%d['value'], 'e2e %.3e'%d['e2e']['value'], d.get('phase_ms'))"
done
python tools/shard_emul.py 1 2 4 8 > gpurun_out/r2_shard_emul.txt 2>&1; grep "N=" gpurun_out/r2_shard_emul.txt
for c in cfg3; do
python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ll_plain_$c.json 2>&1 && \
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_$c.csv \
    python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ll_ncu_$c.log 2>&1
echo "ll $c rc=$?"
done
