"""Time epsilon_apply (and its element kernel share) at a level for the library in HHG_LIB."""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2506_04157_b200 as hhg
from tests.harness import BC_SHELL, lib_eta, lib_mesh, lib_u
from workload import icoshell
ap = argparse.ArgumentParser(); ap.add_argument("--level", type=int, default=5); ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
M = lib_mesh(icoshell(3, 2), a.level, True, BC_SHELL)
eta = lib_eta(M, a.level, (1e6, 30.0)); u = lib_u(M, a.level, 2); y = M.zeros(a.level, hhg.HHG_P2VEC)
for _ in range(3): hhg.epsilon_apply(M, a.level, eta, u, y)
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
torch.cuda.synchronize(); e0.record()
for _ in range(a.reps): hhg.epsilon_apply(M, a.level, eta, u, y)
e1.record(); torch.cuda.synchronize()
print(json.dumps({"lib": os.path.basename(hhg.LIB_PATH), "level": a.level, "ms": e0.elapsed_time(e1) / a.reps, "ynorm": float(y.norm())}))
