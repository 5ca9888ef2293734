"""Per-DTW cell counts: reference EAPrunedDTW vs the GPU engines, on cfg4
candidates that survive LB_Keogh EQ+EC at the converged threshold."""
import os, sys, time
sys.path.insert(0, '/root/repo')
import numpy as np
from scipy.ndimage import maximum_filter1d, minimum_filter1d
import paper_2010_05371_b200 as g
import oracle

SEED_REF, SEED_QUERY = 20261019, 20261020
n, m, w = 100_000_000, 1024, 205
ref = g.random_walk_normal(n, SEED_REF)
q = g.random_walk_normal(m, SEED_QUERY)
cfg = g.SearchConfig(window_ratio=205 / 1024) if hasattr(g, 'SearchConfig') else None
res = g.similarity_search(ref, q, g.SearchConfig(window_ratio=205 / 1024, query_length=m))
ub = res.best.distance_sq if hasattr(res.best, "distance_sq") else res.best.distance
print('final', res, flush=True)
qn = g.znormalize(q)
rng = np.random.default_rng(1)
pos = np.sort(rng.choice(n - m + 1, 400_000, replace=False))
U = maximum_filter1d(qn, 2 * w + 1, mode='nearest')
L = minimum_filter1d(qn, 2 * w + 1, mode='nearest')
surv = []
for s in range(0, len(pos), 20000):
    P = pos[s:s + 20000]
    X = ref[P[:, None] + np.arange(m)[None, :]]
    mu = X.mean(1, keepdims=True); sd = X.std(1, keepdims=True)
    Z = (X - mu) / sd
    eq = (np.where(Z > U, Z - U, np.where(Z < L, L - Z, 0.0)) ** 2).sum(1)
    Zu = maximum_filter1d(Z, 2 * w + 1, axis=1, mode='nearest')
    Zl = minimum_filter1d(Z, 2 * w + 1, axis=1, mode='nearest')
    ec = (np.where(qn > Zu, qn - Zu, np.where(qn < Zl, Zl - qn, 0.0)) ** 2).sum(1)
    keep = (eq <= ub) & (ec <= ub)
    surv.append(Z[keep])
Z = np.concatenate(surv)
print('survivors', len(Z), 'of', len(pos), flush=True)
o = oracle.Oracle()
oc = []
for z in Z:
    v, c = o.dtw(2, z, qn, w, ub)
    oc.append(c)
oc = np.array(oc)
print('oracle EAPrunedDTW cells/DTW mean %.0f median %.0f p90 %.0f' % (oc.mean(), np.median(oc), np.percentile(oc, 90)))
Q = np.broadcast_to(qn, Z.shape).copy()
ubs = np.full(len(Z), ub)
for k in ['0', '1', '3', '5']:
    os.environ['EAPDTW_AD_K'] = k
    out, cells = g.pairwise(Z, Q, g.Band.cells(w), ubs)
    print('gpu ad_k', k, 'cells/DTW %.0f' % (cells / len(Z)), 'ratio %.2f' % (cells / oc.sum()))
# cells the full band would hold for the first R rows
print('band cells per row ~', 2 * w + 1)
