import numpy as np, sys
sys.path.insert(0, '/root/repo')
import paper_2010_05371_b200 as g
r = g.random_walk(4000, 11); q = g.random_walk(64, 12)
for lb in (True, False):
    res = g.similarity_search(r, q, g.SearchConfig(window_ratio=0.1, use_lower_bounds=lb))
    print('rw lb', lb, res.best, res.report)
rng = np.random.default_rng(1)
ref = (rng.integers(0, 13, 2000) - 6).astype(float); qq = (rng.integers(0, 13, 48) - 6).astype(float)
ref[700:748] = qq
for lb in (True, False):
    res = g.similarity_search(ref, qq, g.SearchConfig(window_ratio=0.1, use_lower_bounds=lb))
    print('int lb', lb, res.best, res.report)
ref2 = ref.copy(); ref2[700:748] = qq + 0.5 * rng.standard_normal(48)
res = g.similarity_search(ref2, qq, g.SearchConfig(window_ratio=0.1))
print('int-noisy', res.best, res.report)
