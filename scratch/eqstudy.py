import sys, numpy as np
sys.path.insert(0, '/root/repo')
import paper_2010_05371_b200 as g
from scipy.ndimage import maximum_filter1d, minimum_filter1d
n, m, w = 20_000_000, 1024, 205
ref = g.random_walk_normal(n, 20261019)
q = g.random_walk_normal(m, 20261020)
qn = g.znormalize(q)
ub = 3.748871965313156
U = maximum_filter1d(qn, 2*w+1, mode='nearest'); L = minimum_filter1d(qn, 2*w+1, mode='nearest')
order = np.lexsort((np.arange(m), -np.abs(qn)))
rng = np.random.default_rng(0)
pos = rng.choice(n-m+1, 60000, replace=False)
X = ref[pos[:, None] + np.arange(m)]
Z = (X - X.mean(1, keepdims=True)) / X.std(1, keepdims=True)
kim = (qn[0]-Z[:,0])**2 + (qn[-1]-Z[:,-1])**2
Z = Z[kim <= ub]
print('after kim', len(Z), 'of', len(pos))
T = np.where(Z > U, Z-U, np.where(Z < L, L-Z, 0.0))**2
C = np.cumsum(T[:, order], axis=1)
cross = np.where(C[:, -1] > ub, np.argmax(C > ub, axis=1), m)
print('EQ survive frac', np.mean(cross == m))
pr = cross[cross < m]
print('pruned: crossing position quantiles', np.percentile(pr, [10, 25, 50, 75, 90, 99]))
print('mean positions per candidate (exact per-lane)', np.mean(np.minimum(cross + 1, m)))
# warp of 32 in arrival order: max over lanes, rounded up to 8
cw = np.minimum(cross + 1, m)
nw = len(cw) // 32
wm = np.ceil(cw[:nw*32].reshape(nw, 32).max(1) / 8) * 8
print('warp-lockstep positions per candidate', wm.mean())
for head in [64, 128, 256, 512]:
    h1 = np.minimum(cw, head)
    w1 = np.ceil(h1[:nw*32].reshape(nw, 32).max(1) / 8) * 8
    rest = cw[cw > head] - head
    nr = len(rest) // 32
    w2 = np.ceil(rest[:nr*32].reshape(nr, 32).max(1) / 8) * 8 if nr else np.zeros(1)
    tot = w1.sum() + w2.sum() * (len(rest) / max(1, nr * 32))
    print('head', head, 'lockstep positions per candidate', tot / (nw))
