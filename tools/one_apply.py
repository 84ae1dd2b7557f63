"""One warm-up + one profiled epsilon_apply on blended shell(3,2) at --level (for ncu captures)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2506_04157_b200 as hhg
from tests.harness import BC_SHELL, lib_eta, lib_mesh, lib_u
from workload import icoshell

ap = argparse.ArgumentParser()
ap.add_argument("--level", type=int, default=4)
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
M = lib_mesh(icoshell(3, 2), a.level, True, BC_SHELL)
eta = lib_eta(M, a.level, (1e6, 30.0))
u = lib_u(M, a.level, 2)
for _ in range(a.reps):
    y = hhg.epsilon_apply(M, a.level, eta, u)
torch.cuda.synchronize()
print("ok", float(y.norm()))
