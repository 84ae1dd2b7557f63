"""GPU robustness: stream safety of solver objects, the deterministic (atomic-free) mode, lifetime
guards and argument checks of the binding.

* Two hhg_mg objects on ONE mesh run V-cycles concurrently on two non-blocking streams: each owns its
  reduction scratch (fused-dot partials + arrival counter), so the results equal the sequential ones.
* hhg_set_deterministic: element kernels per brick colour without fp64 REDs -> repeated V-cycles are
  bitwise identical, and agree with the oracle within the V-cycle tolerance (north star: 1e-9).
* blend_map / hhg_set_bc / hhg_set_deterministic are refused while a solver object uses the mesh.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2506_04157_b200 as hhg  # noqa: E402
from tests.harness import BC_SHELL, canon, lib_eta, lib_mesh, lib_u, oracle_case, rel_l2  # noqa: E402
from workload import icoshell, uniform_vec  # noqa: E402

C3 = (1e6, 30.0)


def _mg(M, levels, seed=6, **kw):
    etas = {L: lib_eta(M, L, C3) for L in levels}
    pv = {L: M.from_canonical(L, hhg.HHG_P2VEC, uniform_vec(M.canonical_keys(L, hhg.HHG_P2), seed))
          for L in levels[1:]}
    return hhg.MG(M, levels[0], levels[-1], etas, pv, pre=3, post=3, degree=3, power_iters=20, coarse_iters=50,
                  **kw), etas


def test_two_solver_objects_on_two_streams():
    M = lib_mesh(icoshell(3, 2), 3, True, BC_SHELL)
    mg1, _ = _mg(M, (1, 2, 3))
    mg2, _ = _mg(M, (1, 2, 3))
    f1, f2 = lib_u(M, 3, 4), lib_u(M, 3, 7)
    ref1, ref2 = mg1.vcycle(f1).clone(), mg2.vcycle(f2).clone()
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    xs = []
    for _ in range(3):
        x1, x2 = M.zeros(3, hhg.HHG_P2VEC), M.zeros(3, hhg.HHG_P2VEC)
        with torch.cuda.stream(s1):
            mg1.vcycle(f1, x1, stream=s1)
        with torch.cuda.stream(s2):
            mg2.vcycle(f2, x2, stream=s2)
        xs.append((x1, x2))
    torch.cuda.synchronize()
    for x1, x2 in xs:
        assert float((x1 - ref1).norm()) <= 1e-12 * float(ref1.norm())
        assert float((x2 - ref2).norm()) <= 1e-12 * float(ref2.norm())


def test_profiled_serial_vcycle_equals_forked_graph_vcycle_and_times_the_dense_kernel():
    """The element launcher forks the sparse-brick launch onto a side stream (parallel graph branches); with
    hhg_mg_profile on, the launches stay serial and the dense-brick kernel is timed alone.  Both orders give the
    same V-cycle up to the rounding order of the border REDs, and 0 < dense time <= element time."""
    M = lib_mesh(icoshell(3, 2), 3, True, BC_SHELL)
    mg, _ = _mg(M, (1, 2, 3))
    f = lib_u(M, 3, 4)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        x_graph = mg.vcycle(f, stream=s).clone()
    s.synchronize()
    mg.profile(True)
    with torch.cuda.stream(s):
        x_prof = mg.vcycle(f, stream=s).clone()
    s.synchronize()
    p = mg.profile_get()
    mg.profile(False)
    assert float((x_prof - x_graph).norm()) <= 1e-12 * float(x_graph.norm())
    assert p["apply_count"] > 0 and p["cycle_count"] == 1
    assert 0.0 < p["dense_ms_sum"] <= p["apply_ms_sum"] <= p["cycle_ms_sum"]


def test_deterministic_mode_is_bitwise_reproducible_and_matches_oracle():
    from oracle.multigrid import Hierarchy
    mac = icoshell(3, 2)
    levels = (1, 2, 3)
    M = lib_mesh(mac, 3, True, BC_SHELL)
    M.set_deterministic(True)
    mg, etas = _mg(M, levels)
    f = lib_u(M, 3, 4)
    s = torch.cuda.Stream()
    outs = []
    with torch.cuda.stream(s):
        for _ in range(4):
            outs.append(mg.vcycle(f, stream=s).clone())
    s.synchronize()
    for x in outs[1:]:
        assert torch.equal(x, outs[0])
    # element-kernel outputs of the two modes agree to rounding (only the border summation order differs)
    u = lib_u(M, 3, 2)
    y_det = hhg.epsilon_apply(M, 3, etas[3], u)
    y_det2 = hhg.epsilon_apply(M, 3, etas[3], u)
    assert torch.equal(y_det, y_det2)
    M2 = lib_mesh(mac, 3, True, BC_SHELL)
    y_at = hhg.epsilon_apply(M2, 3, lib_eta(M2, 3, C3), lib_u(M2, 3, 2))
    assert float((y_det - y_at).norm()) <= 1e-13 * float(y_at.norm())
    # and the deterministic V-cycle against the oracle
    discs, v0 = {}, {}
    for L in levels:
        lm, d, _ = oracle_case(mac, L, True, BC_SHELL, C3, 0.0, build=("A",))
        discs[L], v0[L] = d, uniform_vec(lm.p2_keys, 6)
    H = Hierarchy(discs, v0, pre=3, post=3, degree=3, power_iters=20, coarse_iters=50)
    x_o = H.vcycle(discs[3].project(uniform_vec(discs[3].lm.p2_keys, 4)))
    assert rel_l2(canon(M, 3, hhg.HHG_P2VEC, outs[0]), x_o) <= 1e-9


def test_mesh_changes_refused_while_solver_alive():
    M = lib_mesh(icoshell(3, 2), 2, True, BC_SHELL)
    mg, _ = _mg(M, (1, 2))
    with pytest.raises(hhg.HHGError, match="HHG_EINVAL"):
        M.set_bc(hhg.HHG_BND_OUTER, hhg.HHG_BC_FREESLIP)
    with pytest.raises(hhg.HHGError, match="HHG_EINVAL"):
        M.blend_map(hhg.HHG_BLEND_IDENTITY)
    with pytest.raises(hhg.HHGError, match="HHG_EINVAL"):
        M.set_deterministic(True)
    del mg
    import gc
    gc.collect()
    M.set_bc(hhg.HHG_BND_OUTER, hhg.HHG_BC_DIRICHLET0)   # allowed again


def test_host_vcycle_argument_checks():
    M = lib_mesh(icoshell(3, 2), 2, True, BC_SHELL)
    mg, _ = _mg(M, (1, 2))
    n = M.vec_len(2, hhg.HHG_P2VEC)
    good = torch.zeros(n, dtype=torch.float64).pin_memory()
    for bad in (torch.zeros(n, dtype=torch.float32).pin_memory(), torch.zeros(n - 1, dtype=torch.float64).pin_memory(),
                torch.zeros(n, dtype=torch.float64, device="cuda")):
        with pytest.raises(hhg.HHGError):
            mg.vcycle_host_batch([bad], [good])
        with pytest.raises(hhg.HHGError):
            mg.vcycle_host(bad, good)
    with pytest.raises(hhg.HHGError):
        mg.vcycle_host_batch([good], [torch.zeros(n, dtype=torch.float64)])   # not pinned
    rhs = lib_u(M, 2, 4)
    ref = mg.vcycle(rhs).cpu()
    xh = torch.zeros(n, dtype=torch.float64).pin_memory()
    mg.vcycle_host(rhs.cpu().pin_memory(), xh)
    torch.cuda.synchronize()
    assert float((xh - ref).norm()) <= 1e-12 * float(ref.norm())
