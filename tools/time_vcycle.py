"""Median graph-launched V(3,3)-cycle time of the config-3 case at --level (bench.py's set-up), for A/B
switches given by environment variables (e.g. HHG_NO_FX=1)."""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2506_04157_b200 as hhg
from bench import build_case
ap = argparse.ArgumentParser(); ap.add_argument("--level", type=int, default=5); ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()
M, etas, v0, rhs, n_dof = build_case(a.level, 0)
mg = hhg.MG(M, 1, a.level, etas, v0)
s = torch.cuda.Stream()
x = M.zeros(a.level, hhg.HHG_P2VEC)
ts = []
with torch.cuda.stream(s):
    for i in range(a.reps + 3):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(s); mg.vcycle(rhs, x, stream=s); e1.record(s); e1.synchronize()
        if i >= 3: ts.append(e0.elapsed_time(e1))
ts.sort()
print(json.dumps({"level": a.level, "vcycle_ms_median": ts[len(ts) // 2], "vcycle_ms_min": ts[0],
                  "env": {k: v for k, v in os.environ.items() if k.startswith("HHG_")}, "xnorm": float(x.norm())}))
