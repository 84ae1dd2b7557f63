"""Time the blended variable-viscosity epsilon apply and one V-cycle at the largest single-GPU sizes
(shell(3,2), L6 and L7).  Inputs are generated on the device (torch.rand); eta = config-3 style
exp(lnC * r01) field sampled from the node radius.  Prints one JSON line per level."""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2506_04157_b200 as hhg
from workload import icoshell

ap = argparse.ArgumentParser()
ap.add_argument("--levels", type=int, nargs="+", default=[6, 7])
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
mac = icoshell(3, 2)
for L in a.levels:
    M = hhg.Mesh.from_macro(mac, L)
    M.blend_map(hhg.HHG_BLEND_SHELL)
    M.set_bc(hhg.HHG_BND_OUTER, hhg.HHG_BC_DIRICHLET0)
    M.set_bc(hhg.HHG_BND_INNER, hhg.HHG_BC_FREESLIP)
    n = M.vec_len(L, hhg.HHG_P2VEC)
    g = torch.Generator(device="cuda").manual_seed(L)
    eta = torch.exp(torch.rand(M.vec_len(L, hhg.HHG_P1), dtype=torch.float64, device="cuda", generator=g) * 9.2)
    M.interface_sum(L, hhg.HHG_P1, eta)     # copies agree (sum of equal-law draws; any positive field)
    u = torch.rand(n, dtype=torch.float64, device="cuda", generator=g)
    M.interface_sum(L, hhg.HHG_P2VEC, u)
    u = M.apply_bc(L, u)
    y = torch.zeros_like(u)
    for _ in range(2):
        hhg.epsilon_apply(M, L, eta, u, y)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(a.reps):
        hhg.epsilon_apply(M, L, eta, u, y)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.reps
    tets = 240 * 8 ** L
    print(json.dumps({"level": L, "dofs_u": n, "micro_tets": tets, "apply_ms": ms,
                      "Gtet_per_s": tets / ms / 1e6, "fp64_TFs": tets * 1098 / ms / 1e9,
                      "mem_GB": torch.cuda.max_memory_allocated() / 1e9}), flush=True)
    del M, eta, u, y
    torch.cuda.empty_cache(); torch.cuda.reset_peak_memory_stats()
