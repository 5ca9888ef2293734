"""Drive the preparation kernels alone at cfg4 size (n = 1e8, m = 1024,
r = 205) through the public API, for ncu captures of stats_chain_kernel /
stats_convert_kernel / envelope_gw_kernel."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2010_05371_b200 as g  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
ref = g.random_walk_normal(n, 20261019)
mean, sd = g.sliding_stats(ref, 1024)
up, lo = g.sliding_envelope(ref, 205)
print("ok", float(mean[12345]), float(sd[12345]), float(up[777]), float(lo[777]))
