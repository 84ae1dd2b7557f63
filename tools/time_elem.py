"""Time the fine-level element kernel (epsilon_apply_partial minus a same-size memset) at --level for
the library in HHG_LIB (A/B experiments).  CUDA events on the launching stream, median of --reps."""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2506_04157_b200 as hhg
from tests.harness import BC_SHELL, lib_eta, lib_mesh, lib_u
from workload import icoshell
ap = argparse.ArgumentParser(); ap.add_argument("--level", type=int, default=5); ap.add_argument("--reps", type=int, default=30)
a = ap.parse_args()
M = lib_mesh(icoshell(3, 2), a.level, True, BC_SHELL)
eta = lib_eta(M, a.level, (1e6, 30.0)); u = lib_u(M, a.level, 2); y = M.zeros(a.level, hhg.HHG_P2VEC)
s = torch.cuda.current_stream()
def t(fn):
    ts = []
    for i in range(a.reps + 3):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(s); fn(); e1.record(s); e1.synchronize()
        if i >= 3: ts.append(e0.elapsed_time(e1))
    ts.sort(); return ts[len(ts) // 2]
t_part = t(lambda: hhg.epsilon_apply_partial(M, a.level, eta, u, y))
t_ms = t(lambda: y.zero_())
t_full = t(lambda: hhg.epsilon_apply(M, a.level, eta, u, y))
print(json.dumps({"lib": os.path.basename(hhg.LIB_PATH), "level": a.level, "elem_ms": t_part - t_ms, "partial_ms": t_part,
                  "memset_ms": t_ms, "apply_ms": t_full, "ynorm": float(y.norm())}))
