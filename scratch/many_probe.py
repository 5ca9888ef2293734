"""search_many throughput: 16 queries (m=512, w=51) on the 1e7 cfg3 reference."""
import time
import torch
import paper_2010_05371_b200 as g

ref = g.random_walk_normal(10_000_000, 20261019)
qs = [g.random_walk_normal(512, 7000 + k) for k in range(16)]
cfg = g.SearchConfig(window_ratio=0.1)
dref = g.DeviceSeries(ref)
for conc in (1, 2, 4, 8):
    g.search_many(dref, qs, cfg, concurrency=conc)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        res = g.search_many(dref, qs, cfg, concurrency=conc)
        ts.append((time.perf_counter() - t0) * 1e3)
    print("concurrency", conc, "ms per 16 queries", [round(t, 1) for t in ts],
          "first", res[0].best.location, res[0].best.distance_sq)
