"""Multi-rank execution of the partitioned hot path on ONE GPU (P:689-709 macro-primitive
decomposition).  2, 4 and 8 processes -- one rank each, all on cuda:0 -- run the library's real partitioned
path: each builds its part of the RCB macro partition, every interface sum packs the rank's partial sums
(k_halo_pack), moves them through the host-staged transport (hhg_comm_create_host over a gloo process
group) and adds the neighbours' partials (k_fixup_remote); dots allreduce.  No kernel ever waits on
another rank, so sharing one GPU is safe.  Compared with the 1-rank run of the same case: epsilon_apply,
dots, lambda_hat per level, and one config-3-recipe V(3,3)-cycle with the redundant (gathered) coarse
solve and with the distributed coarse PCG -- all <= 1e-12 relative (the partition changes only the
order of floating-point sums)."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

L = 3
C3 = (1e6, 30.0)


def _case(M, levels):
    import paper_2506_04157_b200 as hhg
    from tests.harness import lib_eta, lib_u
    from workload import uniform_vec
    etas = {l: lib_eta(M, l, C3) for l in levels}
    pv = {l: M.from_canonical(l, hhg.HHG_P2VEC, uniform_vec(M.canonical_keys(l, hhg.HHG_P2), 6)) for l in levels[1:]}
    return etas, pv, lib_u(M, levels[-1], 4)


def _run(M, redundant):
    """-> dict of canonical-order results (+ presence masks) of this rank's part."""
    import paper_2506_04157_b200 as hhg
    from tests.harness import canon
    levels = tuple(range(1, L + 1))
    etas, pv0, rhs = _case(M, levels)
    pv0 = {l: v.clone() for l, v in pv0.items()}
    y = hhg.epsilon_apply(M, L, etas[L], rhs)
    dot = float(hhg.hhg_dot(M, L, hhg.HHG_P2VEC, rhs, y).item())
    out = {"apply": canon(M, L, hhg.HHG_P2VEC, y), "dot": dot,
           "mask": canon(M, L, hhg.HHG_P2VEC, torch.ones_like(rhs))}
    for red in redundant:
        # fresh start vectors: hhg_mg_create's power iterations overwrite them
        pv = {l: v.clone() for l, v in pv0.items()}
        mg = hhg.MG(M, 1, L, etas, pv, pre=3, post=3, degree=3, power_iters=20, coarse_iters=50, coarse_redundant=red)
        x = mg.vcycle(rhs)
        torch.cuda.synchronize()
        out[f"vcycle{int(red)}"] = canon(M, L, hhg.HHG_P2VEC, x)
        out[f"lam{int(red)}"] = [mg.lam(l) for l in levels[1:]]
        del mg
    return out


def _rank_main(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import paper_2506_04157_b200 as hhg
    from tests.harness import BC_SHELL
    from workload import icoshell
    try:
        mac = icoshell(3, 2)
        tr = hhg.partition_rcb(mac.verts, mac.tets, world, radial=True)
        comm = hhg.HostComm()
        M = hhg.Mesh.from_macro(mac, L, tet_rank=tr, comm=comm)
        M.blend_map(hhg.HHG_BLEND_SHELL)
        M.set_bc(hhg.HHG_BND_OUTER, hhg.HHG_BC_DIRICHLET0)
        M.set_bc(hhg.HHG_BND_INNER, hhg.HHG_BC_FREESLIP)
        out = _run(M, (True, False) if world == 2 else (True,))
        out["rank"] = rank
        out["macros"] = M.local_macros()
        q.put(out)
        del M
    except Exception as e:  # pragma: no cover
        q.put({"rank": rank, "error": repr(e)})
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture(scope="module")
def single_rank():
    import paper_2506_04157_b200 as hhg  # noqa: F401
    from tests.harness import BC_SHELL, lib_mesh
    from workload import icoshell
    M = lib_mesh(icoshell(3, 2), L, True, BC_SHELL)
    return _run(M, (True,))


def _merge(outs, key):
    """Combine the ranks' canonical vectors (each node from any rank holding it) and return the largest
    disagreement between ranks on shared nodes."""
    val = np.zeros_like(outs[0][key])
    have = np.zeros(val.shape, dtype=bool)
    spread = 0.0
    for o in outs:
        m = o["mask"] > 0.5
        both = m & have
        if both.any():
            spread = max(spread, float(np.abs(o[key][both] - val[both]).max()))
        val[m & ~have] = o[key][m & ~have]
        have |= m
    assert have.all()
    return val, spread


@pytest.mark.parametrize("world", [2, 4, 8])
def test_partitioned_vcycle_matches_single_rank(single_rank, world):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = [q.get() for _ in range(world)]
    for p in procs:
        p.join(timeout=600)
    errs = [o["error"] for o in outs if "error" in o]
    assert not errs, errs
    assert sum(o["macros"] for o in outs) == 240
    ref = single_rank
    rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
    y, sp = _merge(outs, "apply")
    assert sp <= 1e-13 * np.abs(ref["apply"]).max()
    assert rel(y, ref["apply"]) <= 1e-13
    for o in outs:
        assert abs(o["dot"] - ref["dot"]) <= 1e-12 * abs(ref["dot"])
    for red in ((True, False) if world == 2 else (True,)):
        k = f"vcycle{int(red)}"
        x, sp = _merge(outs, k)
        assert sp <= 1e-12 * np.abs(ref["vcycle1"]).max(), (k, sp)
        err = rel(x, ref["vcycle1"])
        print(f"world {world} coarse_redundant={red}: V-cycle rel_l2 vs 1 rank {err:.2e}")
        assert err <= 1e-12, (k, err)
        for o in outs:
            for a, b in zip(o[f"lam{int(red)}"], ref["lam1"]):
                assert abs(a - b) <= 1e-12 * b
