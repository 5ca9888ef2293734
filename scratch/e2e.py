"""e2e timing of the public host-pointer search at cfg4 (pinned host reference)."""
import os, sys, time, statistics
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2010_05371_b200 as g
n, m = 100_000_000, 1024
ref = g.random_walk_normal(n, 20261019); q = g.random_walk_normal(m, 20261020)
pinned = torch.from_numpy(ref).pin_memory()
cfg = g.SearchConfig(window_ratio=205 / 1024)
ctx = g.Context(0)
ts = []
for it in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    r = g.similarity_search(pinned.numpy(), q, cfg, ctx=ctx)
    torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
print(os.environ.get('EAPDTW_STREAM_SPLIT'), os.environ.get('EAPDTW_STREAMED'), 'e2e ms', [round(t*1e3, 1) for t in ts[1:]], r.best.location, r.best.distance_sq)
