# streamed host-pointer search: part 1's share (eighths) vs e2e at cfg4
set -x
for k in 3 2 1 4 3 2; do
  python bench.py --steps 3 --warmup 2 --no-cpu-baseline --opt stream_split=$k > gpurun_out/sp.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/sp.json'));print('stream_split=$k e2e %.4g subseq/s = %.2f ms; device %.2f ms' % (d['e2e']['value'], 99998977/d['e2e']['value']*1e3, d['ms_per_step']))"
done
