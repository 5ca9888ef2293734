import sys, os, numpy as np
sys.path.insert(0, '/root/repo')
import paper_2010_05371_b200 as g
import oracle
UNB = oracle.UNBOUNDED
rng = np.random.default_rng(77)
L = 128
db = np.cumsum(rng.standard_normal((3000, L)), axis=1)
db[::3] *= 40.0
qs = np.cumsum(rng.standard_normal((5, L)), axis=1)
qs[1] *= 40.0
for band in [int(x) if x != 'u' else UNB for x in sys.argv[1:]]:
    try:
        arg, dist, _ = g.nn1(qs, db, g.Band(band))
        print('ok', band, arg, dist, flush=True)
    except Exception as e:
        print('FAIL', band, e, flush=True)
        break
