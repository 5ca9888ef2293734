"""Grid timing: resident vs host reference, stats cache on/off."""
import os
import time
import numpy as np
import torch
import paper_2010_05371_b200 as g

ref = g.random_walk(1_000_000, 42)
q = g.random_walk(1024, 43)
L, R = (128, 256, 512, 1024), (0.1, 0.2, 0.3, 0.4, 0.5)
ctx = g.Context(0)
pinned = torch.from_numpy(ref).pin_memory().numpy()


def wall(f, n=3):
    f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return min(ts) * 1e3


dref = g.DeviceSeries(ref, ctx=ctx)
res = None


def grid(r):
    global res
    res = [x for *_, x in g.search_grid(r, q, L, R, ctx=ctx)]


print("resident grid ms", wall(lambda: grid(dref)))
print("per-search ms", [round(x.report.elapsed_seconds * 1e3, 2) for x in res])
print("host grid ms", wall(lambda: grid(pinned)))
print("upload+free ms", wall(lambda: g.DeviceSeries(pinned, ctx=ctx).close()))
t0 = time.perf_counter()
for _ in range(20):
    g.similarity_search_dev(dref.device_ptr, len(dref), q[:256], g.SearchConfig(window_ratio=0.1), ctx=ctx)
torch.cuda.synchronize()
print("uncached dev search len256 r0.1 ms", (time.perf_counter() - t0) / 20 * 1e3)
t0 = time.perf_counter()
for _ in range(20):
    dref.search(q[:256], g.SearchConfig(window_ratio=0.1))
print("cached series search len256 r0.1 ms", (time.perf_counter() - t0) / 20 * 1e3)
