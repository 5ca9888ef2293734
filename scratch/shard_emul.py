"""Per-shard time of cfg4 at N GPUs, emulated on one GPU: a search over the
first 1e8/N candidates of the cfg4 reference (device-resident), phases from
the plan's CUDA events.  No threshold exchange (a lower bound on the benefit
the other shards' thresholds would give)."""
import os, sys, statistics
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2010_05371_b200 as g
from paper_2010_05371_b200.sharded import GpuShard
N = int(sys.argv[1]) if len(sys.argv) > 1 else 8
n, m = 100_000_000, 1024
ref = g.random_walk_normal(n, 20261019); q = g.random_walk_normal(m, 20261020)
ncand = (n - m + 1) // N
npts = ncand + m - 1
cfg = g.SearchConfig(window_ratio=205 / 1024)
ctx = g.Context(0)
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
dref = torch.from_numpy(ref[:npts]).cuda()
key = torch.full((1,), 0, dtype=torch.int64, device="cuda")
sh = GpuShard(dref.data_ptr(), npts, q, cfg, 0, key, ctx=ctx)
tot = []
for it in range(4):
    sh.reset(); sh.prepare(); sh.run(0, sh.candidates); r = sh.result()
    t = sh.plan.timings()
    tot.append(sum(t.values()))
print(N, os.environ.get('EAPDTW_PROBE'), os.environ.get('EAPDTW_RANK'), 'total ms', [round(x, 2) for x in tot[1:]], {k: round(v, 2) for k, v in t.items()}, r.best.location)
