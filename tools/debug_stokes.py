"""Compare GPU and oracle Stokes solves for 1..k FGMRES iterations (debug)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2506_04157_b200 as hhg
from oracle.multigrid import Hierarchy
from oracle.stokes import StokesOracle
from tests.harness import BC_SHELL, canon, lib_eta, lib_mesh, lib_p, oracle_case, rel_l2
from workload import icoshell, uniform_vec, uniform_from_keys, GAMMA_TALA
C2 = (1e4, 10.0)
mac = icoshell(3, 2)
discs, v0 = {}, {}
for L in (1, 2):
    lm, d, _ = oracle_case(mac, L, True, BC_SHELL, C2, GAMMA_TALA, build=("A", "B", "C", "M") if L == 2 else ("A",))
    discs[L], v0[L] = d, uniform_vec(lm.p2_keys, 6)
H = Hierarchy(discs, v0)
d = discs[2]
S_o = StokesOracle(H, d, d.M)
rhs_o = np.concatenate([uniform_vec(d.lm.p2_keys, 2), uniform_from_keys(d.lm.p1_keys, 3, 0)])
M = lib_mesh(mac, 2, True, BC_SHELL)
etas = {L: lib_eta(M, L, C2) for L in (1, 2)}
pv = {2: M.from_canonical(2, hhg.HHG_P2VEC, uniform_vec(M.canonical_keys(2, hhg.HHG_P2), 6))}
mg = hhg.MG(M, 1, 2, etas, pv)
ru = M.from_canonical(2, hhg.HHG_P2VEC, uniform_vec(M.canonical_keys(2, hhg.HHG_P2), 2))
rhs = torch.cat([ru, lib_p(M, 2, 3)])
n2 = M.vec_len(2, hhg.HHG_P2VEC)
for k in (1, 2, 3, 5, 10, 40):
    S = hhg.StokesSolver(mg, etas[2], GAMMA_TALA, restart=30, max_iters=k, tol=1e-6)
    x, it, rel = S.solve(rhs)
    torch.cuda.synchronize()
    xc = np.concatenate([canon(M, 2, hhg.HHG_P2VEC, x[:n2].contiguous()), canon(M, 2, hhg.HHG_P1, x[n2:].contiguous())])
    xo, ito, relo = S_o.solve(rhs_o, tol=1e-6, restart=30, max_iters=k)
    nu = 3 * d.lm.n_p2
    print(k, it, rel, ito, relo, "u", rel_l2(xc[:nu], xo[:nu]), "p", rel_l2(xc[nu:], xo[nu:]), flush=True)
