#!/usr/bin/env python
"""bench.py -- one step = one GMG V(3,3)-cycle for the A block (BASELINE config 3: blended
shell(3,2), refinement level 5, viscosity contrast 1e6 x 30 radial jump, Chebyshev degree 3,
lambda_hat from 20 power iterations, P2 transfers down to level 1, 50 Jacobi-PCG coarse
iterations) on a seeded rhs, through the C-ABI (graph-launched).  The per-eta setup (diag(A),
power iterations) runs before the timed region.  Also measured in the same run: the fine-level
epsilon_apply throughput (BASELINE metric's first clause) and the end-to-end V-cycle through
vcycle_host() with pinned host buffers.

Contract: python bench.py --gpus N --steps K --warmup W [--impl reference]; for N>1 launched by
torch.distributed.run, one process per GPU; rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "P2 epsilon-operator apply GDoF/s (fp64) and V-cycle time; % of fp64/HBM roofline"
GAMMA = 0.3781


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--level", type=int, default=5)
    ap.add_argument("--cpu-level", type=int, default=2, help="oracle sample level for cpu_baseline / reference")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--apply-reps", type=int, default=20)
    return ap.parse_args()


def peaks():
    p = {}
    try:
        p = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    return p


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.rows = []
        if self.proc is None:
            return
        time.sleep(0.25)
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=5)
        raw = os.environ.get("HHG_CLOCKS_RAW")
        if raw:
            with open(raw, "a") as fh:
                fh.write(out)
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 7:
                self.rows.append(f)

    def summary(self):
        rows = getattr(self, "rows", [])
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(float(r[0]) for r in rows)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i].strip() == "Active"})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": float(rows[0][1]), "reasons": reasons,
                "samples": len(rows)}


# weak scaling (BASELINE config 5): 240 macros per GPU -- shell(ntan, nrad) by GPU count
SHELL_BY_GPUS = {1: (3, 2), 2: (3, 3), 4: (5, 2), 8: (5, 3)}


def build_case(level, device, world=1, rank=0, comm=None, contrast=1e6, jump=30.0):
    """Library-side set-up of config 3 (mesh, eta per level, power start vectors, rhs).  world > 1:
    shell with 240*world macros partitioned by recursive coordinate bisection, one part per rank."""
    import torch
    import paper_2506_04157_b200 as hhg
    from workload import icoshell, uniform_vec, viscosity
    ntan, nrad = SHELL_BY_GPUS.get(world, (3, 2))
    mac = icoshell(ntan, nrad, 0.55, 1.0)
    if world > 1:
        tr = hhg.partition_rcb(mac.verts, mac.tets, world, radial=True)
        M = hhg.Mesh.from_macro(mac, level, tet_rank=tr, comm=comm)
    else:
        M = hhg.Mesh.from_macro(mac, level)
    M.blend_map(hhg.HHG_BLEND_SHELL)
    M.set_bc(hhg.HHG_BND_OUTER, hhg.HHG_BC_DIRICHLET0)
    M.set_bc(hhg.HHG_BND_INNER, hhg.HHG_BC_FREESLIP)
    etas, v0 = {}, {}
    for L in range(1, level + 1):
        keys1 = M.canonical_keys(L, hhg.HHG_P1)
        xyz = M.node_coords(L, hhg.HHG_P1)
        xc = torch.stack([M.to_canonical(L, hhg.HHG_P1, xyz[:, c].contiguous()) for c in range(3)], 1)
        etas[L] = M.from_canonical(L, hhg.HHG_P1, viscosity(xc.cpu().numpy(), keys1, contrast, jump))
        if L > 1:
            v0[L] = M.from_canonical(L, hhg.HHG_P2VEC, uniform_vec(M.canonical_keys(L, hhg.HHG_P2), 6))
    keysL = M.canonical_keys(level, hhg.HHG_P2)
    rhs = M.apply_bc(level, M.from_canonical(level, hhg.HHG_P2VEC, uniform_vec(keysL, 4)))
    n_dof = 3 * keysL.shape[0]
    return M, etas, v0, rhs, n_dof


def cpu_oracle_vcycle(level, steps=1):
    """The oracle as it stands: config-3 recipe V-cycle on shell(3,2) levels `level`..1 (CPU)."""
    import numpy as np
    from oracle.multigrid import Hierarchy
    from tests.harness import BC_SHELL, oracle_case
    from workload import icoshell, uniform_vec
    mac = icoshell(3, 2)
    t0 = time.perf_counter()
    discs, v0 = {}, {}
    for L in range(1, level + 1):
        lm, d, _ = oracle_case(mac, L, True, BC_SHELL, (1e6, 30.0), 0.0, build=("A",))
        discs[L], v0[L] = d, uniform_vec(lm.p2_keys, 6)
    H = Hierarchy(discs, v0)
    setup = time.perf_counter() - t0
    f = discs[level].project(uniform_vec(discs[level].lm.p2_keys, 4))
    ts = []
    for _ in range(steps):
        t1 = time.perf_counter()
        H.vcycle(f)
        ts.append(time.perf_counter() - t1)
    ndof = 3 * discs[level].lm.n_p2
    return ndof, ts, setup


def run_reference(args, rank, world):
    if rank != 0:
        return
    ndof, ts, setup = cpu_oracle_vcycle(args.cpu_level, args.warmup + args.steps)
    tt = ts[args.warmup:]
    ms = 1e3 * sum(tt) / len(tt)
    val = ndof / (ms * 1e-3) / 1e9
    cores = len(os.sched_getaffinity(0))
    sample = (f"oracle (numpy/scipy CSR) V(3,3)-cycle, shell(3,2) levels {args.cpu_level}->1, config-3 recipe, "
              f"{ndof} dofs; assembly/setup {setup:.1f} s excluded")
    print(json.dumps({"impl": "reference", "metric": METRIC, "value": val, "unit": "GDoF/s", "n_gpus": args.gpus,
                      "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
                      "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                      "config": {"workload": f"config3-sample shell(3,2) L{args.cpu_level} V(3,3)", "level": args.cpu_level},
                      "cpu_baseline": {"value": val, "unit": "GDoF/s", "cores": cores, "kind": "oracle", "sample": sample},
                      "e2e": {"value": val, "unit": "GDoF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)
    import torch
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        # communicator set-up lines (ranks, channels, NVLS) on stderr, so the driver can check nranks
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2506_04157_b200 as hhg

    L = args.level
    comm = hhg.Comm(rank, world, local) if world > 1 else None
    M, etas, v0, rhs, n_dof = build_case(L, local, world, rank, comm)
    t0 = time.perf_counter()
    mg = hhg.MG(M, 1, L, etas, v0, pre=3, post=3, degree=3, power_iters=20, coarse_iters=50)
    setup_s = time.perf_counter() - t0
    s = torch.cuda.Stream()
    x = M.zeros(L, hhg.HHG_P2VEC)

    # kernels per V-cycle (eager count), then graph warm-up
    hhg.launch_count(reset=True)
    mg.profile(True)
    with torch.cuda.stream(s):
        mg.vcycle(rhs, x, stream=s)
    s.synchronize()
    kernels_per_cycle = hhg.launch_count(reset=True)
    # profiled cycles: fine-level element kernel durations measured with CUDA events on s
    mg.profile(True)
    with torch.cuda.stream(s):
        for _ in range(3):
            mg.vcycle(rhs, x, stream=s)
    s.synchronize()
    prof = mg.profile_get()
    mg.profile(False)

    with torch.cuda.stream(s):
        for _ in range(max(3, args.warmup)):
            mg.vcycle(rhs, x, stream=s)
    s.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        with torch.cuda.stream(s):
            e0.record(s)
            for _ in range(args.steps):
                mg.vcycle(rhs, x, stream=s)
            e1.record(s)
        s.synchronize()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    if dist:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = n_dof / (ms * 1e-3) / 1e9          # n_dof: unique velocity dofs of the whole (partitioned) mesh

    # standalone fine-level epsilon_apply (BASELINE metric, first clause)
    y = M.zeros(L, hhg.HHG_P2VEC)
    with torch.cuda.stream(s):
        for _ in range(3):
            hhg.epsilon_apply(M, L, etas[L], rhs, y, stream=s)
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(s)
        for _ in range(args.apply_reps):
            hhg.epsilon_apply(M, L, etas[L], rhs, y, stream=s)
        a1.record(s)
    s.synchronize()
    apply_ms = a0.elapsed_time(a1) / args.apply_reps
    if dist:
        t = torch.tensor([apply_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        apply_ms = float(t.item())

    # end to end: every step copies its rhs from pinned host memory and its solution back, through
    # the public vcycle_host_batch (copies of neighbouring steps overlapped with the compute);
    # two host rhs/x pairs alternate so consecutive steps really move different buffers
    rhs_h = [rhs.cpu().pin_memory() for _ in range(2)]
    x_h = [torch.empty_like(rhs_h[0]).pin_memory() for _ in range(2)]
    with torch.cuda.stream(s):
        mg.vcycle_host_batch([rhs_h[k & 1] for k in range(max(args.warmup, 2))],
                             [x_h[k & 1] for k in range(max(args.warmup, 2))], stream=s)
        s.synchronize()
        h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        h0.record(s)
        mg.vcycle_host_batch([rhs_h[k & 1] for k in range(args.steps)], [x_h[k & 1] for k in range(args.steps)],
                             stream=s)
        h1.record(s)
    s.synchronize()
    e2e_ms = h0.elapsed_time(h1) / args.steps
    if dist:
        t = torch.tensor([e2e_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    nbytes = rhs.numel() * 8

    # roofline of the dominant kernel (fine-level element kernel, fp64 DFMA pipe): flops per micro tet and
    # DRAM bytes per launch from the committed ncu capture, DFMA peak from the committed microbenchmark
    counts = elem_counts()
    n_tets = M.local_macros() * 8 ** L        # this rank's micro tets (the element kernel it times)
    flops_per_tet = counts["epsilon_apply_L5"]["flops_per_tet"]
    traffic = counts["epsilon_apply_L5"]["dram_bytes"] if L == 5 else None
    elem_ms = prof["apply_ms_sum"] / max(1, prof["apply_count"])       # dense + sparse launches of one application
    achieved_op = flops_per_tet * n_tets / (elem_ms * 1e-3) / 1e12
    # the dominant kernel alone: k_elem_fp over the dense bricks (its own tets and flops from the capture's first
    # part, its own CUDA-event duration: an event is recorded between it and the sparse-brick launch)
    parts = counts["epsilon_apply_L5"].get("parts") or []
    dense_ms = prof["dense_ms_sum"] / max(1, prof["apply_count"])
    n_sparse_tets = M.local_macros() * sparse_tets_per_macro(L)
    if parts and L == 5 and dense_ms > 0:
        dense_flops = 2 * parts[0]["dfma"] + parts[0]["dadd"] + parts[0]["dmul"]   # per launch, 240 macros
        dense_flops *= M.local_macros() / 240.0
        traffic = parts[0]["dram_bytes"]
    else:
        dense_flops = flops_per_tet * (n_tets - n_sparse_tets)
    achieved = dense_flops / (dense_ms * 1e-3) / 1e12 if dense_ms > 0 else achieved_op
    pk = peaks()
    fp64 = fp64_peak_measured()
    fp64_peak = pk.get("fp64_tflops") or fp64["fp64_dfma_tflops"]

    # BASELINE config 2: stokes_apply (A + B^T, (B + C)) on shell(3,2) L4, contrast 1e4 x 10, gamma 0.3781
    st = stokes_apply_line(counts, fp64_peak, s, dist) if world == 1 else None
    result = {
        "metric": METRIC, "value": value, "unit": "GDoF/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"config3: V(3,3)-cycle, blended shell{SHELL_BY_GPUS.get(world, (3, 2))} level {L}->1, "
                               "eta contrast 1e6 x30, "
                               "Chebyshev deg 3, 50 PCG coarse its",
                   "level": L, "velocity_dofs": n_dof, "macros": 240 * world,
                   "micro_tets_per_gpu": n_tets, "parallelism": f"macro-partition x{world} (RCB), NCCL interface exchange" if world > 1 else "single GPU",
                   "l2": "inputs larger than L2 (rhs/x/work vectors 276 MB each at level 5)"},
        "apply": {"gdofs": n_dof / (apply_ms * 1e-3) / 1e9, "ms": apply_ms, "level": L,
                  "note": "epsilon_apply (memset + element kernel + interface sum/BC) standalone"},
        "vcycle_ms": ms, "setup_s": setup_s,
        "roofline": {"bound": "alu", "achieved": achieved, "peak": fp64_peak, "unit": "TFLOP/s",
                     "frac": achieved / fp64_peak, "traffic": traffic,
                     "kernel": "k_elem_fp<blend,A,full> over the dense bricks of the fine level (the dominant kernel)",
                     "kernel_ms": dense_ms, "kernel_tets": n_tets - n_sparse_tets,
                     "kernel_flops_per_launch": dense_flops,
                     "operator": {"what": "one epsilon_apply element pass = k_elem_fp (dense bricks) + k_elem_sparse "
                                          "(bricks cut by the macro's slanted face); timed with the two launches in series "
                                          "(profiling mode) -- the timed V-cycle forks the sparse launch onto a side "
                                          "stream", "elem_ms": elem_ms,
                                  "achieved": achieved_op, "frac": achieved_op / fp64_peak,
                                  "traffic": counts["epsilon_apply_L5"]["dram_bytes"] if L == 5 else None},
                     "elem_ms": elem_ms,
                     "flops_per_tet": flops_per_tet,
                     "flops_source": "profiles/r02_elem_counts.json (ncu dfma/dadd/dmul thread instructions per launch "
                                     "/ micro tets, DFMA = 2)",
                     "peak_source": "MEASURED_PEAKS.json fp64_tflops" if pk.get("fp64_tflops") else
                     f"measured DFMA microbenchmark, best of {fp64.get('reps')} launches at "
                     f"{fp64.get('clocks', {}).get('sm_mhz_median_under_load')} MHz (profiles/r02_fp64_peak.json; "
                     "nominal 148 SMs x 64 FP64 lanes x 2 x 1.965 GHz = 37.2 TF/s)",
                     "hbm_gbs_algorithmic": (2 * rhs.numel() + M.local_macros() * ((2 ** L + 1) * (2 ** L + 2)
                                                                                    * (2 ** L + 3) // 6)) * 8
                     / (elem_ms * 1e-3) / 1e9},
        "e2e": {"value": n_dof / (e2e_ms * 1e-3) / 1e9, "unit": "GDoF/s", "ms": e2e_ms,
                "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes,
                "api": "MG.vcycle_host_batch (pinned host rhs -> V-cycle -> pinned host x per step; H2D of step k+1 "
                       "and D2H of step k-1 overlap V-cycle k)"},
        "gpu_launches": kernels_per_cycle * args.steps,
        "clocks": clk.summary(),
    }
    if st:
        result["stokes_apply"] = st
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        ndof_c, ts, setup = cpu_oracle_vcycle(args.cpu_level, 2)
        v = ndof_c / min(ts) / 1e9
        result["cpu_baseline"] = {"value": v, "unit": "GDoF/s", "cores": len(os.sched_getaffinity(0)),
                                  "kind": "oracle",
                                  "sample": f"oracle V(3,3)-cycle shell(3,2) levels {args.cpu_level}->1 "
                                            f"({ndof_c} dofs), best of 2; setup {setup:.1f} s excluded",
                                  "apply": cpu_oracle_apply(3)}
    if rank == 0:
        print(json.dumps(result))
    if dist:
        dist.destroy_process_group()


def sparse_tets_per_macro(L):
    """Micro tets of one macro that lie in sparse bricks (4x4x4-cube bricks with delta = n - (i0+j0+k0) <= 4)."""
    n = 2 ** L
    tot = 0
    for i0 in range(0, n, 4):
        for j0 in range(0, n - i0, 4):
            for k0 in range(0, n - i0 - j0, 4):
                delta = n - (i0 + j0 + k0)
                if delta > 4:
                    continue
                for c in range(64):
                    ts = (c & 3) + ((c >> 2) & 3) + (c >> 4)
                    tot += 6 if ts <= delta - 3 else (5 if ts == delta - 2 else (1 if ts == delta - 1 else 0))
    return tot


def elem_counts():
    """Per-launch ncu counters of the element kernels (tools/ncu_counts.py on the committed captures)."""
    return json.load(open(os.path.join(ROOT, "profiles", "r02_elem_counts.json")))


def fp64_peak_measured():
    """DFMA throughput of this pool's B200 (tools/fp64_peak_clocks.py: 200 launches, clocks sampled)."""
    return json.load(open(os.path.join(ROOT, "profiles", "r02_fp64_peak.json")))


def stokes_apply_line(counts, fp64_peak, s, dist, reps=20):
    """BASELINE config 2: stokes_apply [A u + B^T p ; (B + C) u] on the blended shell(3,2) at level 4,
    viscosity contrast 1e4 x 10, gamma = 0.3781 (whole C-ABI call: zeroing, fused element kernel,
    interface sums + BCs), GDoF/s over the unique (u, p) dofs; roofline of the call against the DFMA peak
    with the fused kernel's flops per micro tet (profiles/r02_elem_counts.json)."""
    import torch
    import paper_2506_04157_b200 as hhg
    from tests.harness import BC_SHELL, lib_eta, lib_mesh, lib_p, lib_u
    from workload import icoshell
    L = 4
    M = lib_mesh(icoshell(3, 2), L, True, BC_SHELL)
    eta = lib_eta(M, L, (1e4, 10.0))
    u, p = lib_u(M, L, 2), lib_p(M, L, 3)
    yu, yp = M.zeros(L, hhg.HHG_P2VEC), M.zeros(L, hhg.HHG_P1)
    n_dof = M.canonical_len(L, hhg.HHG_P2VEC) + M.canonical_len(L, hhg.HHG_P1)
    with torch.cuda.stream(s):
        for _ in range(3):
            hhg.stokes_apply(M, L, eta, GAMMA, u, p, yu, yp, stream=s)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(reps):
            hhg.stokes_apply(M, L, eta, GAMMA, u, p, yu, yp, stream=s)
        e1.record(s)
    s.synchronize()
    ms = e0.elapsed_time(e1) / reps
    c = counts["stokes_apply_L4"]
    achieved = c["flops_per_tet"] * 240 * 8 ** L / (ms * 1e-3) / 1e12
    return {"config": "config2: blended shell(3,2) L4, contrast 1e4 x 10, gamma 0.3781", "ms": ms,
            "gdofs": n_dof / (ms * 1e-3) / 1e9, "dofs_u_p": n_dof,
            "roofline": {"bound": "alu", "achieved": achieved, "peak": fp64_peak, "unit": "TFLOP/s",
                         "frac": achieved / fp64_peak, "flops_per_tet": c["flops_per_tet"],
                         "note": "whole stokes_apply call timed (zeroing + element kernel + interface sums); the fused "
                                 "element kernel alone: %.1f us under ncu" % (1e6 * c["duration_s"])},
            "l2": "level-4 vectors (97 MB) fit in L2"}


def cpu_oracle_apply(level, reps=5):
    """The oracle's epsilon apply: assembled CSR A of shell(3,2) at `level` (config-3 viscosity) times a
    vector, scipy SpMV on the host (assembly excluded), best of `reps`."""
    from tests.harness import BC_SHELL, oracle_case
    from workload import icoshell, uniform_vec
    t0 = time.perf_counter()
    lm, d, _ = oracle_case(icoshell(3, 2), level, True, BC_SHELL, (1e6, 30.0), 0.0, build=("A",))
    Ac = d.Ac()
    setup = time.perf_counter() - t0
    u = d.project(uniform_vec(lm.p2_keys, 2))
    ts = []
    for _ in range(reps):
        t1 = time.perf_counter()
        Ac @ u
        ts.append(time.perf_counter() - t1)
    ndof = 3 * lm.n_p2
    return {"value": ndof / min(ts) / 1e9, "unit": "GDoF/s", "kind": "oracle",
            "sample": f"oracle CSR SpMV (M P_v) A (P_v M) u, shell(3,2) level {level} ({ndof} dofs, nnz {Ac.nnz}), "
                      f"best of {reps}; assembly {setup:.1f} s excluded; scipy (single thread)"}

if __name__ == "__main__":
    main()
