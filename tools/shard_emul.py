"""One shard's search of cfg4 sharded N ways, timed on one GPU (no threshold
exchange: the shard converges on its own): the per-shard fixed costs that
bound the scaling of DESIGN.md section 7.
    python tools/shard_emul.py [N ...]"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2010_05371_b200 as g  # noqa: E402

n, m, ratio = 100_000_000, 1024, 205 / 1024
ref = g.random_walk_normal(n, 20261019)
q = g.random_walk_normal(m, 20261020)
ctx = g.Context(0)
stream = torch.cuda.current_stream()
ctx.set_stream(stream.cuda_stream)
cfg = g.SearchConfig(query_length=m, window_ratio=ratio)
for kv in filter(None, os.environ.get("OPTS", "").split(",")):  # engine options, e.g. OPTS=rank_stride=0
    k, v = kv.split("=")
    ctx.set_option(k, int(v))
for N in [int(a) for a in sys.argv[1:]] or [1, 2, 4, 8]:
    seg = -(-(n - m + 1) // 100_000)
    ncand = min(n - m + 1, -(-seg // N) * 100_000)
    npts = ncand + m - 1
    dref = torch.from_numpy(ref[:npts]).cuda()
    for spec in ([0, 1] if ncand <= 40_000_000 and "SPEC_AB" in os.environ else [-1]):
        ctx.set_option("spec_stats", spec)
        plan = g.SearchPlan(dref.data_ptr(), npts, q, cfg, ctx=ctx)
        ms, ph = [], []
        for it in range(6):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            plan.reset()
            plan.prepare()
            plan.run(0, ncand)
            res = plan.result()
            e1.record(stream)
            torch.cuda.synchronize()
            if it > 0:
                ms.append(e0.elapsed_time(e1))
                ph.append(plan.timings())
        med = {k: round(statistics.median(p[k] for p in ph), 2) for k in ph[0]}
        print(f"N={N} shard of {ncand} candidates, spec_stats={spec}: {statistics.median(ms):.2f} ms "
              f"{med} best={res.best.location} (ideal 1/N of N=1)", flush=True)
        plan.close()
    del dref
