"""Engine microbenchmark: pairwise DTW, warp per pair, all engines."""
import os, sys, time, json
sys.path.insert(0, '/root/repo')
import numpy as np
import torch
import paper_2010_05371_b200 as g
from paper_2010_05371_b200 import _capi
import ctypes as C

def run(L, w, npairs, ubmul, reps=3):
    rng = np.random.default_rng(1)
    a = np.stack([g.znormalize(np.cumsum(rng.standard_normal(L))) for _ in range(npairs)])
    b = np.stack([g.znormalize(np.cumsum(rng.standard_normal(L))) for _ in range(npairs)])
    ctx = g.Context(0)
    da = torch.from_numpy(a).cuda(); db = torch.from_numpy(b).cuda()
    out = torch.empty(npairs, dtype=torch.float64, device='cuda')
    os.environ['EAPDTW_AD_K'] = '0'
    exact, _ = g.pairwise(a, b, g.Band(w), None, prune=False, ctx=ctx)
    ub = torch.from_numpy(exact * ubmul).cuda()
    res = {}
    for K in ('0', '1', '3', '5'):
        os.environ['EAPDTW_AD_K'] = K
        cells = C.c_uint64(0)
        best = 1e9
        for r in range(reps):
            torch.cuda.synchronize(); t = time.perf_counter()
            _capi.check(_capi.lib.eapdtw_pairwise_dev(ctx.handle, C.c_void_p(da.data_ptr()), C.c_void_p(db.data_ptr()), npairs, L, w, C.c_void_p(ub.data_ptr()), 1, C.c_void_p(out.data_ptr()), C.byref(cells)))
            torch.cuda.synchronize(); best = min(best, time.perf_counter() - t)
        o = out.cpu().numpy()
        ok = np.array_equal(o, np.where(exact <= exact * ubmul, exact, np.inf))
        res[K] = (best * 1e3, cells.value / best / 1e9, ok)
    return res

for (L, w, n, m) in [(512, 512, 8192, 1.0), (1024, 205, 8192, 1.0), (1024, 60, 8192, 1.0), (512, 51, 16384, 1.0), (1024, 205, 8192, 0.6)]:
    r = run(L, w, n, m)
    print(f"L={L} w={w} n={n} ubmul={m}: " + "  ".join(f"K{k}: {v[0]:.2f}ms {v[1]:.0f}GCUPS ok={v[2]}" for k, v in r.items()), flush=True)
