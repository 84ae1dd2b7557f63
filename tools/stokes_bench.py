"""Config-4-style preconditioned Stokes solve on ONE GPU (the paper's config 4 is L6 on 8 GPUs):
blended shell(3,2) at --level, contrast 1e6 x 30 viscosity, TALA compressibility, buoyancy rhs from
the workload temperature, FGMRES + symmetric Uzawa with the V-cycle BFBT (or mass) Schur
approximation, Table-1 parameters (sigma 1, omega 0.3, tol_A 1e-2, tol_V 1e-1, tol_mass 1e-10,
V(3,3)/V(1,1) hierarchies with Chebyshev degree 2/1) and BASELINE's relative reduction 1e-8.
Prints one JSON line (time, iterations, residual)."""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2506_04157_b200 as hhg
from bench import build_case, GAMMA
from workload import temperature
ap = argparse.ArgumentParser()
ap.add_argument("--level", type=int, default=4)
ap.add_argument("--schur", default="vbfbt", choices=["vbfbt", "mass", "wbfbt"])
ap.add_argument("--omega", type=float, default=0.3, help="Uzawa pressure scaling (Table 1: 0.3; P:685: 0.0125 for w-BFBT)")
ap.add_argument("--a-l", type=float, default=1.0)
ap.add_argument("--a-r", type=float, default=1.0)
ap.add_argument("--uzawa", default="symmetric", choices=["symmetric", "inexact", "adjoint"])
ap.add_argument("--tol-A", type=float, default=1e-2)
ap.add_argument("--tol", type=float, default=1e-8)
ap.add_argument("--max-iters", type=int, default=60)
ap.add_argument("--restart", type=int, default=30)
ap.add_argument("--deg", type=int, default=2, help="Chebyshev degree of the A-block V-cycle (Table 1: 2)")
ap.add_argument("--contrast", type=float, default=1e6)
ap.add_argument("--jump", type=float, default=30.0)
ap.add_argument("--l-eta", type=int, default=-1, help="levels <= l_eta use quadrature-point viscosity (NEXT-2)")
ap.add_argument("--l-min", type=int, default=1, help="coarsest level of the V-cycles (P:661: l_min = 2 on 240 macros)")
ap.add_argument("--coarse-tol", type=float, default=0.0, help="coarse PCG relative tolerance (Table 1: 1e-2; 0: 50 its)")
ap.add_argument("--coarse-iters", type=int, default=50)
ap.add_argument("--tol-vbfbt", type=float, default=1e-1, help="Table 1: 1e-1")
ap.add_argument("--cheap-coarse-iters", type=int, default=None, help="coarse PCG iterations of the A_C hierarchy")
a = ap.parse_args()
L = a.level
M, etas, v0, _, n_dof = build_case(L, 0, contrast=a.contrast, jump=a.jump)
def temp_p2(l):
    keys2 = M.canonical_keys(l, hhg.HHG_P2)
    xyz2 = M.node_coords(l, hhg.HHG_P2)
    xc2 = torch.stack([M.to_canonical(l, hhg.HHG_P2, xyz2[:, c].contiguous()) for c in range(3)], 1)
    return M.from_canonical(l, hhg.HHG_P2, temperature(xc2.cpu().numpy(), keys2))
import math
T2s = {l: temp_p2(l) for l in range(1, a.l_eta + 1)} if a.l_eta >= 1 else None
qeta = (math.log(a.contrast), a.jump, 0.9)
t0 = time.perf_counter()
ck = dict(coarse_tol=a.coarse_tol, coarse_iters=a.coarse_iters)
mg = hhg.MG(M, a.l_min, L, etas, v0, pre=3, post=3, degree=a.deg, T2_per_level=T2s, l_eta=a.l_eta, qeta=qeta, **ck)
v0c = {l: v.clone() for l, v in build_case(L, 0, contrast=a.contrast, jump=a.jump)[2].items()} if a.schur == "vbfbt" else None
ckc = dict(ck) if a.cheap_coarse_iters is None else dict(coarse_tol=0.0, coarse_iters=a.cheap_coarse_iters)
mgc = hhg.MG(M, a.l_min, L, etas, v0c, pre=1, post=1, degree=1, T2_per_level=T2s, l_eta=a.l_eta, qeta=qeta, **ckc) \
    if a.schur == "vbfbt" else None
keys = M.canonical_keys(L, hhg.HHG_P1)
xyz = M.node_coords(L, hhg.HHG_P1)
xc = torch.stack([M.to_canonical(L, hhg.HHG_P1, xyz[:, c].contiguous()) for c in range(3)], 1)
T = M.from_canonical(L, hhg.HHG_P1, temperature(xc.cpu().numpy(), keys))
f = hhg.hhg_buoyancy_load(M, L, T)
rhs = torch.cat([f, M.zeros(L, hhg.HHG_P1)])
S = hhg.StokesSolver(mg, etas[L], GAMMA, restart=a.restart, max_iters=a.max_iters, tol=a.tol, schur=a.schur,
                     mg_cheap=mgc, omega=a.omega, a_l=a.a_l, a_r=a.a_r, uzawa=a.uzawa, tol_A=a.tol_A,
                     tol_vbfbt=a.tol_vbfbt)
torch.cuda.synchronize()
setup = time.perf_counter() - t0
s = torch.cuda.Stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(s):
    e0.record(s)
    x, it, rel = S.solve(rhs, stream=s)
    e1.record(s)
s.synchronize()
ms = e0.elapsed_time(e1)
n_p = M.canonical_len(L, hhg.HHG_P1)
x2, ita, rela = mg.ablock_cg(f, tol=1e-2, max_iters=200)
print(json.dumps({"what": "stokes_solve", "l_eta": a.l_eta, "l_min": a.l_min, "coarse_tol": a.coarse_tol,
                  "tol_vbfbt": a.tol_vbfbt, "cheap_coarse_iters": a.cheap_coarse_iters, "restart": a.restart,
                  "coarse_iters_max": a.coarse_iters, "ablock_cg_iters_tol1e-2": ita, "ablock_rel": rela, "level": L, "schur": a.schur, "omega": a.omega, "a_l": a.a_l, "a_r": a.a_r, "uzawa": a.uzawa, "tol_A": a.tol_A, "velocity_dofs": n_dof, "pressure_dofs": n_p,
                  "fgmres_iters": it, "rel_res": rel, "tol": a.tol, "solve_s": ms / 1e3, "setup_s": setup,
                  "viscosity": f"contrast {a.contrast:g} x {a.jump:g} jump", "rhs": "buoyancy (T - 1/2) x/|x|, g = 0"}))
