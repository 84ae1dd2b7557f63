"""V(3,3)-cycle (config-3 smoother settings) time at levels 5..7 on ONE GPU (SURVEY config 5's single-GPU
points).  Inputs generated on the device: eta = exp(ln(1e6) u), u uniform, interface-summed to make
copies consistent (a positive field with the config's contrast, not the workload recipe, which is
evaluated on the host and too large at L7); rhs uniform, BC-projected; power-iteration start vectors
uniform.  Prints one JSON line per level (time per cycle, GDoF/s, memory)."""
import argparse, json, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2506_04157_b200 as hhg
from workload import icoshell

ap = argparse.ArgumentParser()
ap.add_argument("--levels", type=int, nargs="+", default=[5, 6, 7])
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
mac = icoshell(3, 2)
for L in a.levels:
    try:
        M = hhg.Mesh.from_macro(mac, L)
        M.blend_map(hhg.HHG_BLEND_SHELL)
        M.set_bc(hhg.HHG_BND_OUTER, hhg.HHG_BC_DIRICHLET0)
        M.set_bc(hhg.HHG_BND_INNER, hhg.HHG_BC_FREESLIP)
        g = torch.Generator(device="cuda").manual_seed(L)
        etas, v0 = {}, {}
        for l in range(1, L + 1):
            e = torch.rand(M.vec_len(l, hhg.HHG_P1), dtype=torch.float64, device="cuda", generator=g)
            M.interface_sum(l, hhg.HHG_P1, e)
            etas[l] = torch.exp(math.log(1e6) * (e / 6.0))       # copies summed (<= 6 copies) -> [1, 1e6]
            if l > 1:
                v0[l] = torch.rand(M.vec_len(l, hhg.HHG_P2VEC), dtype=torch.float64, device="cuda", generator=g)
                M.interface_sum(l, hhg.HHG_P2VEC, v0[l])
        mg = hhg.MG(M, 1, L, etas, v0, pre=3, post=3, degree=3, power_iters=20, coarse_iters=50)
        mg._v0 = {}                 # the start vectors are only needed by the power iterations in create
        del v0
        torch.cuda.empty_cache()
        rhs = torch.rand(M.vec_len(L, hhg.HHG_P2VEC), dtype=torch.float64, device="cuda", generator=g)
        M.interface_sum(L, hhg.HHG_P2VEC, rhs)
        rhs = M.apply_bc(L, rhs)
        x = torch.zeros_like(rhs)
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            mg.vcycle(rhs, x, stream=s)
            mg.vcycle(rhs, x, stream=s)
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record(s)
            for _ in range(a.reps):
                mg.vcycle(rhs, x, stream=s)
            e1.record(s)
        s.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        ndof = M.canonical_len(L, hhg.HHG_P2) * 3
        print(json.dumps({"level": L, "velocity_dofs": ndof, "vcycle_ms": ms, "gdofs": ndof / ms / 1e6,
                          "finite": bool(torch.isfinite(x).all()),
                          "mem_GB": torch.cuda.max_memory_allocated() / 1e9}), flush=True)
        del mg, M, etas, rhs, x
        torch.cuda.empty_cache()
        torch.cuda.reset_peak_memory_stats()
    except Exception as ex:  # e.g. HHG_ENOMEM at L7
        print(json.dumps({"level": L, "error": str(ex)[:300]}), flush=True)
        break
