"""Run-to-run spread of the config-3 V(3,3)-cycle: the same rhs through the same hierarchy --reps times, with the
default element kernels (fp64 REDs on brick borders: summation order varies) and in deterministic mode (brick
colours, no REDs).  Prints one JSON line per (level, mode): max over runs of |x_k - x_0| / |x_0| and whether all
runs were bitwise identical."""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2506_04157_b200 as hhg
from bench import build_case

ap = argparse.ArgumentParser()
ap.add_argument("--levels", default="3,5")
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()
for L in [int(v) for v in a.levels.split(",")]:
    for det in (False, True):
        M, etas, v0, rhs, n_dof = build_case(L, 0)
        if det:
            M.set_deterministic(True)
        mg = hhg.MG(M, 1, L, etas, v0)
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        xs = []
        with torch.cuda.stream(s):
            for _ in range(a.reps):
                x = M.zeros(L, hhg.HHG_P2VEC)
                mg.vcycle(rhs, x, stream=s)
                xs.append(x)
        s.synchronize()
        n0 = float(xs[0].norm())
        spread = max(float((x - xs[0]).norm()) / n0 for x in xs[1:])
        bitwise = all(torch.equal(x, xs[0]) for x in xs[1:])
        print(json.dumps({"level": L, "deterministic": det, "reps": a.reps, "max_rel_spread": spread,
                          "bitwise_identical": bitwise, "velocity_dofs": n_dof}), flush=True)
        del mg, M
