"""ORACLE-side probe (test infrastructure, CPU): the config-4 recipe's Stokes solve on the blended shell at
--level (levels 1..L, P1 viscosity of contrast --contrast x --jump, TALA gamma, buoyancy rhs, V-BFBT Schur,
symmetric Uzawa, Table-1 tolerances) by the ORACLE's FGMRES (oracle/stokes.py) -- the residual history to
compare with the GPU's (tools/stokes_bench.py, HHG_STATS=1) on the same recipe.  Prints one JSON line."""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle.multigrid import Hierarchy
from oracle.stokes import StokesOracle
from oracle.operators import node_coords
from tests.harness import BC_SHELL, oracle_case
from workload import icoshell, uniform_vec, GAMMA_TALA, temperature

ap = argparse.ArgumentParser()
ap.add_argument("--level", type=int, default=2)
ap.add_argument("--contrast", type=float, default=1e6)
ap.add_argument("--jump", type=float, default=30.0)
ap.add_argument("--iters", type=int, default=60)
ap.add_argument("--deg", type=int, default=2)
a = ap.parse_args()
mac = icoshell(3, 2)
L = a.level
discs, v0 = {}, {}
for l in range(1, L + 1):
    lm, d, _ = oracle_case(mac, l, True, BC_SHELL, (a.contrast, a.jump), GAMMA_TALA,
                           build=("A", "B", "C", "M") if l == L else ("A",))
    discs[l], v0[l] = d, uniform_vec(lm.p2_keys, 6)
H = Hierarchy(discs, v0, pre=3, post=3, degree=a.deg, power_iters=20, coarse_iters=50)
HC = Hierarchy(discs, v0, pre=1, post=1, degree=1, power_iters=20, coarse_iters=50)
d = discs[L]
S = StokesOracle(H, d, d.M, sigma=1.0, omega=0.3, tol_A=1e-2, schur="vbfbt", HC=HC)
from oracle.operators import buoyancy_load
T = temperature(node_coords(d.lm, "P1", True), d.lm.p1_keys)
f = d.project(buoyancy_load(d.lm, True, T))
rhs = np.concatenate([f, np.zeros(len(d.lm.p1_keys))])
t0 = time.perf_counter()
x, it, rel = S.solve(rhs, tol=1e-8, restart=a.iters, max_iters=a.iters)
print(json.dumps({"what": "oracle_stokes_probe", "level": L, "contrast": a.contrast, "jump": a.jump, "iters": it,
                  "rel": rel, "s": time.perf_counter() - t0, "history": S.history}))
