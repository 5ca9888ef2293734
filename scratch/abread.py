import glob, json, re, collections, sys
res = collections.defaultdict(list)
for f in sorted(glob.glob('/root/repo/gpurun_out/ab_*.json')):
    m = re.match(r'.*/ab_(.+)_(cfg[^_]+)_(\d+)\.json', f)
    try:
        d = json.load(open(f))
    except Exception:
        continue
    res[(m.group(2), m.group(1))].append(d['phase_ms']['sweep'])
for k in sorted(res):
    v = res[k]
    print(k, 'sweep ms', ' '.join(f'{x:.2f}' for x in v), 'min', f'{min(v):.2f}')
