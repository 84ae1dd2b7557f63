"""--reps stokes_apply calls at BASELINE config 2 (blended shell(3,2), L4, contrast 1e4 x 10, gamma 0.3781)
for ncu captures of the fused A + B^T + (B + C) element kernel."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2506_04157_b200 as hhg
from tests.harness import BC_SHELL, lib_eta, lib_mesh, lib_p, lib_u
from workload import icoshell, GAMMA_TALA
ap = argparse.ArgumentParser()
ap.add_argument("--level", type=int, default=4)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
M = lib_mesh(icoshell(3, 2), a.level, True, BC_SHELL)
eta = lib_eta(M, a.level, (1e4, 10.0))
u, p = lib_u(M, a.level, 2), lib_p(M, a.level, 3)
for _ in range(a.reps):
    yu, yp = hhg.stokes_apply(M, a.level, eta, GAMMA_TALA, u, p)
torch.cuda.synchronize()
print("ok", float(yu.norm()), float(yp.norm()))
