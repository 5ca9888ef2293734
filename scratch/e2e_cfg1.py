"""Where the cfg1 end-to-end step goes: pinned H2D vs the pairwise call."""
import time
import numpy as np
import torch
import paper_2010_05371_b200 as g

npairs, L, w = 1024, 256, 25
a = np.stack([g.znormalize(g.random_walk_normal(L, 1000 + p)) for p in range(npairs)])
b = np.stack([g.znormalize(g.random_walk_normal(L, 500000 + p)) for p in range(npairs)])
ap = torch.from_numpy(a).pin_memory()
bp = torch.from_numpy(b).pin_memory()
ctx = g.Context(0)
d = torch.empty_like(ap, device="cuda")


def t(f, n=20):
    f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3


print("torch H2D 2MB pinned ms", t(lambda: d.copy_(ap, non_blocking=True)))
print("pairwise pageable ms", t(lambda: g.pairwise(a, b, g.Band.cells(w), None, ctx=ctx)))
an, bn = ap.numpy(), bp.numpy()
print("pairwise pinned ms", t(lambda: g.pairwise(an, bn, g.Band.cells(w), None, ctx=ctx)))
ex, _ = g.pairwise(an, bn, g.Band.cells(w), None, ctx=ctx)
ub = ex * 1.05
print("pairwise pinned ub ms", t(lambda: g.pairwise(an, bn, g.Band.cells(w), ub, ctx=ctx)))
print("pairwise pinned noprune ms", t(lambda: g.pairwise(an, bn, g.Band.cells(w), None, prune=False, ctx=ctx)))
