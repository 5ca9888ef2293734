"""Time the stats phase only (plan.prepare with a 1-candidate probe, no coarse pass)."""
import os, sys
os.environ["EAPDTW_PROBE"] = "1"
os.environ["EAPDTW_COARSE_STRIDE"] = "0"
sys.path.insert(0, "/root/repo")
import torch
import paper_2010_05371_b200 as g
n, m = 100_000_000, 1024
ref = torch.from_numpy(g.random_walk_normal(n, 20261019)).cuda()
q = g.random_walk_normal(m, 20261020)
cfg = g.SearchConfig(window_ratio=205 / 1024, query_length=m)
for it in range(3):
    plan = g.SearchPlan(ref.data_ptr(), n, q, cfg)
    plan.prepare()
    plan.run(0, 1)
    torch.cuda.synchronize()
    print(sys.argv[1] if len(sys.argv) > 1 else "", "timings", plan.timings())
    plan.close()
