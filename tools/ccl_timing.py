"""Per-phase timing of the shared-memory cluster coarse PCG (HHG_CCL_TIMING=1): config-3 hierarchy at --level,
--cycles graph-launched V-cycles, then the accumulated globaltimer ns per phase (CTA 0) on stderr."""
import argparse, os, sys
os.environ["HHG_CCL_TIMING"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2506_04157_b200 as hhg
from bench import build_case
ap = argparse.ArgumentParser(); ap.add_argument("--level", type=int, default=5); ap.add_argument("--cycles", type=int, default=4)
a = ap.parse_args()
M, etas, v0, rhs, n_dof = build_case(a.level, 0)
mg = hhg.MG(M, 1, a.level, etas, v0)
x = M.zeros(a.level, hhg.HHG_P2VEC)
for _ in range(a.cycles):
    mg.vcycle(rhs, x)
torch.cuda.synchronize()
print("coarse iterations per solve", mg.coarse_iterations(), "solves", a.cycles)
