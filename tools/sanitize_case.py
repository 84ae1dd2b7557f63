"""Small cases of every hot-path family through the C-ABI, for compute-sanitizer (memcheck / racecheck /
synccheck) runs: config-1 apply/div/divT, a graph-launched shell V-cycle (L2 -> 1), the same in deterministic
mode, power iteration + Chebyshev, the A-block CG, a Stokes FGMRES solve (mass Schur, device-scalar CG), the
w-BFBT Schur apply, the temperature FGMRES solve and MMOC."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2506_04157_b200 as hhg
from tests.harness import BC_ALL, BC_SHELL, lib_eta, lib_mesh, lib_p, lib_u
from workload import icoshell, reference_tet, uniform_vec, GAMMA_TALA

M1 = lib_mesh(reference_tet(), 2, False, BC_ALL)
u1 = lib_u(M1, 2, 0)
hhg.epsilon_apply(M1, 2, None, u1); hhg.div_apply(M1, 2, 0.0, u1); hhg.divT_apply(M1, 2, lib_p(M1, 2, 1))
mac = icoshell(3, 2)
for det in (False, True):
    M = lib_mesh(mac, 2, True, BC_SHELL)
    if det:
        M.set_deterministic(True)
    etas = {L: lib_eta(M, L, (1e4, 10.0)) for L in (1, 2)}
    pv = {2: M.from_canonical(2, hhg.HHG_P2VEC, uniform_vec(M.canonical_keys(2, hhg.HHG_P2), 6))}
    mg = hhg.MG(M, 1, 2, etas, pv, coarse_iters=10)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        x = mg.vcycle(lib_u(M, 2, 4), stream=s)
        x = mg.vcycle(lib_u(M, 2, 4), stream=s)
    s.synchronize()
    x, it, rel = mg.ablock_cg(lib_u(M, 2, 4), tol=1e-2, max_iters=5)
    yu, yp = hhg.stokes_apply(M, 2, etas[2], GAMMA_TALA, lib_u(M, 2, 2), lib_p(M, 2, 3))
    dinv = 1.0 / hhg.hhg_diag(M, 2, etas[2])
    lam = hhg.hhg_power_iteration(M, 2, etas[2], dinv, 5, lib_u(M, 2, 6))
    hhg.chebyshev_smooth(M, 2, etas[2], dinv, 3, lam / 10, lam, lib_u(M, 2, 4), lib_u(M, 2, 9))
    if not det:
        S = hhg.StokesSolver(mg, etas[2], GAMMA_TALA, restart=5, max_iters=5, tol=1e-6, tol_mass=1e-6,
                             mass_max_iters=20)
        rhs = torch.cat([lib_u(M, 2, 2), lib_p(M, 2, 3)])
        S.solve(rhs)
        del S
        W = hhg.StokesSolver(mg, etas[2], GAMMA_TALA, schur="wbfbt", tol_wbfbt=1e-4, wbfbt_max_iters=5,
                             tol_vmass=1e-2, vmass_max_iters=10)
        W.schur_apply(lib_p(M, 2, 3))
        del W
    del mg
    torch.cuda.synchronize()
M = lib_mesh(mac, 1, True, BC_SHELL)
prm = dict(s=1.0, tau=0.01, kappa=1e-3, beta=0.1, gamma=GAMMA_TALA)
TS = hhg.TempSolver(M, 1, prm, restart=10)
T = M.zeros(1, hhg.HHG_P2) + 0.5
TS.solve(lib_u(M, 1, 2), M.zeros(1, hhg.HHG_P2), T, max_iters=5, cg_max_iters=20)
hhg.hhg_mmoc(M, 1, T, lib_u(M, 1, 2) * 0.01, lib_u(M, 1, 2) * 0.01, 0.1)
torch.cuda.synchronize()
print("sanitize_case ok, kernels launched", hhg.launch_count())
