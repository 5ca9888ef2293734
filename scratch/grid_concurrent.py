"""Grid with one context (stream) per query length, searches concurrent."""
import threading
import time
import torch
import paper_2010_05371_b200 as g

ref = g.random_walk(1_000_000, 42)
q = g.random_walk(1024, 43)
L, R = (128, 256, 512, 1024), (0.1, 0.2, 0.3, 0.4, 0.5)

ctx0 = g.Context(0)
d0 = g.DeviceSeries(ref, ctx=ctx0)


def serial():
    return [r for *_, r in g.search_grid(d0, q, L, R, ctx=ctx0)]


ctxs = [g.Context(0) for _ in L]
ds = [g.DeviceSeries(ref, ctx=c) for c in ctxs]
out = {}


def worker(k):
    out[k] = [r for *_, r in g.search_grid(ds[k], q, (L[k],), R, ctx=ctxs[k])]


def concurrent():
    th = [threading.Thread(target=worker, args=(k,)) for k in range(len(L))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    return [r for k in range(len(L)) for r in out[k]]


ctxr = [g.Context(0) for _ in R]
dr = [g.DeviceSeries(ref, ctx=c) for c in ctxr]
outr = {}


def worker_r(k):
    outr[k] = [r for *_, r in g.search_grid(dr[k], q, L, (R[k],), ctx=ctxr[k])]


def concurrent_ratio():
    th = [threading.Thread(target=worker_r, args=(k,)) for k in range(len(R))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    # back to the grid's (length, ratio) order
    return [outr[ki][li] for li in range(len(L)) for ki in range(len(R))]


for name, f in (("serial", serial), ("concurrent", concurrent), ("ratio-major", concurrent_ratio)):
    f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        res = f()
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    print(name, "ms", [round(t, 1) for t in ts], [(r.best.location, r.best.distance_sq) for r in res][:3])
a = serial()
b = concurrent_ratio()
print("same results", all((x.best.location, x.best.distance_sq) == (y.best.location, y.best.distance_sq) for x, y in zip(a, b)))
