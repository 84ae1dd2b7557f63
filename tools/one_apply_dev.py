"""One warm-up + one profiled epsilon_apply at --level with device-generated inputs (eta in [1, 1e6],
uniform u; for ncu captures at L6/L7 where the host-side workload recipe is too large)."""
import argparse, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2506_04157_b200 as hhg
from workload import icoshell

ap = argparse.ArgumentParser()
ap.add_argument("--level", type=int, default=6)
a = ap.parse_args()
L = a.level
M = hhg.Mesh.from_macro(icoshell(3, 2), L)
M.blend_map(hhg.HHG_BLEND_SHELL)
M.set_bc(hhg.HHG_BND_OUTER, hhg.HHG_BC_DIRICHLET0)
M.set_bc(hhg.HHG_BND_INNER, hhg.HHG_BC_FREESLIP)
g = torch.Generator(device="cuda").manual_seed(L)
e = torch.rand(M.vec_len(L, hhg.HHG_P1), dtype=torch.float64, device="cuda", generator=g)
M.interface_sum(L, hhg.HHG_P1, e)
eta = torch.exp(math.log(1e6) * e / 6.0)
u = torch.rand(M.vec_len(L, hhg.HHG_P2VEC), dtype=torch.float64, device="cuda", generator=g)
M.interface_sum(L, hhg.HHG_P2VEC, u)
u = M.apply_bc(L, u)
for _ in range(2):
    y = hhg.epsilon_apply(M, L, eta, u)
torch.cuda.synchronize()
print("ok", float(y.norm()))
