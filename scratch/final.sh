set -x
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench_rc=$?
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref_rc=$?
for c in cfg1 cfg5 cfg2 cfg3 cfg3-nolb; do timeout 600 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo $c rc=$?; done
for c in cfg1 cfg5; do timeout 600 python bench.py --config $c --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref_$c.json 2> gpurun_out/bench_ref_$c.err; echo ref $c rc=$?; done
python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/plain_l.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg4.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_l.log 2>&1; echo ncu_l=$?
ncu --set full --clock-control none --import-source on -k regex:search_kernel -s 2 -c 1 -o gpurun_out/prof_cfg4_final python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_f.log 2>&1; echo ncu_f=$?
