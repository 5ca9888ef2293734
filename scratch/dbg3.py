import numpy as np, sys
sys.path.insert(0, '/root/repo')
import paper_2010_05371_b200 as g
rng = np.random.default_rng(1)
for (n, m, kind) in [(4000, 48, 'rw'), (4000, 40, 'rw'), (2000, 64, 'rw'), (4000, 64, 'int'), (2000, 48, 'int'), (4000, 63, 'rw'), (4000, 65, 'rw'), (4000, 50, 'rw')]:
    if kind == 'rw':
        r = g.random_walk(n, 11); q = g.random_walk(m, 12)
    else:
        r = (rng.integers(0, 13, n) - 6).astype(float); q = (rng.integers(0, 13, m) - 6).astype(float)
    res = g.similarity_search(r, q, g.SearchConfig(window_ratio=0.1))
    rep = res.report
    print(n, m, kind, 'kim', rep.pruned_kim, 'eq', rep.pruned_keogh_eq, 'ec', rep.pruned_keogh_ec, 'calls', rep.dtw_calls, 'tot', rep.candidates_total)
