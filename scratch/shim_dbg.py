import numpy as np, sys
sys.path.insert(0, '/root/repo')
import paper_2010_05371_b200 as g
x = 12345
def lcg():
    global x
    x = (x * 6364136223846793005 + 1442695040888963407) % (1 << 64)
    return float((x >> 33) % 13) - 6.0
ref = np.array([lcg() for _ in range(2000)]); q = np.array([lcg() for _ in range(48)])
ref[700:748] = q
for it in range(5):
    r = g.similarity_search(ref, q, g.SearchConfig(window_ratio=0.1))
    rep = r.report
    print(r.best, rep.candidates_total, rep.pruned_kim + rep.pruned_keogh_eq + rep.pruned_keogh_ec + rep.dtw_calls, rep)
