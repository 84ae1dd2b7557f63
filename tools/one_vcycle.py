"""Set up config 3 (level --level), then run one eager (non-graph) V-cycle after a separator torch op,
so an ncu launch list can be cut at the separator.  Prints the V-cycle wall time."""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2506_04157_b200 as hhg
from bench import build_case
ap = argparse.ArgumentParser(); ap.add_argument("--level", type=int, default=5); ap.add_argument("--cycles", type=int, default=1)
a = ap.parse_args()
M, etas, v0, rhs, n_dof = build_case(a.level, 0)
mg = hhg.MG(M, 1, a.level, etas, v0, use_graph=False)
x = M.zeros(a.level, hhg.HHG_P2VEC)
mg.vcycle(rhs, x)
torch.cuda.synchronize()
sep = torch.ones(7, device="cuda").mul_(3.0)   # separator kernel in the launch list
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(a.cycles):
    mg.vcycle(rhs, x)
torch.cuda.synchronize()
print("vcycle ms", 1e3 * (time.perf_counter() - t0) / a.cycles, "x norm", float(x.norm()))
