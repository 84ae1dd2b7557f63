"""Temperature operator (eq:WeakTemp) on one GPU: time of one L apply at --level and of the
FGMRES + CG(P) solve for a seeded velocity, Dirichlet data and rhs; one JSON line."""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2506_04157_b200 as hhg
from tests.harness import BC_SHELL, lib_mesh
from workload import icoshell, uniform_vec, uniform_from_keys, GAMMA_TALA
ap = argparse.ArgumentParser()
ap.add_argument("--level", type=int, default=4)
ap.add_argument("--tau", type=float, default=1e-3)
a = ap.parse_args()
L = a.level
PRM = dict(s=1.5, tau=a.tau, kappa=1.0, beta=0.5, gamma=GAMMA_TALA)
M = lib_mesh(icoshell(3, 2), L, True, BC_SHELL)
keys = M.canonical_keys(L, hhg.HHG_P2)
u = M.from_canonical(L, hhg.HHG_P2VEC, 100.0 * uniform_vec(keys, 2))
T = M.from_canonical(L, hhg.HHG_P2, uniform_from_keys(keys, 9, 0))
b = M.from_canonical(L, hhg.HHG_P2, uniform_from_keys(keys, 4, 0))
y = hhg.hhg_temp_apply(M, L, PRM, u, T)
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
torch.cuda.synchronize(); e0.record()
for _ in range(10):
    hhg.hhg_temp_apply(M, L, PRM, u, T, y)
e1.record(); torch.cuda.synchronize()
apply_ms = e0.elapsed_time(e1) / 10
uo = M.from_canonical(L, hhg.HHG_P2VEC, 100.0 * uniform_vec(keys, 5))
Th = hhg.hhg_mmoc(M, L, T, u, uo, a.tau)
torch.cuda.synchronize(); e0.record()
hhg.hhg_mmoc(M, L, T, u, uo, a.tau, Th)
e1.record(); torch.cuda.synchronize()
mmoc_ms = e0.elapsed_time(e1)
S = hhg.TempSolver(M, L, PRM, restart=50)
torch.cuda.synchronize(); e0.record()
T, it, rel = S.solve(u, b, T, tol=1e-10, max_iters=100, tol_cg=1e-12)
e1.record(); torch.cuda.synchronize()
print(json.dumps({"what": "temperature", "level": L, "p2_nodes": M.canonical_len(L, hhg.HHG_P2), "micro_tets": 240 * 8 ** L,
                  "apply_ms": apply_ms, "mmoc_ms": mmoc_ms, "solve_ms": e0.elapsed_time(e1), "fgmres_iters": it, "rel_res": rel, "prm": PRM,
                  "u": "100 x seeded uniform P2 velocity"}))
