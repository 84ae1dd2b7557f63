"""GPU: the cluster-resident coarse Jacobi-PCG (hhg_coarse.cu, one kernel per coarse solve) against the oracle
and against the library's generic coarse path (element kernel + interface sum + dots + updates, selected with
HHG_NO_CCL=1 at hierarchy creation).  P:441-443 (coarse grid: Jacobi-preconditioned CG, fixed iteration count).

* The bare coarse solve (l_min = l_max = 1: the V-cycle IS the 50-iteration PCG) equals the oracle's PCG on the
  assembled operator and the generic path, for the config-3 viscosity on the blended shell, the unblended
  shell with the simplified form, and the quadrature-point viscosity tier.
* It is deterministic: no atomics, fixed-order sums -> repeated solves are bitwise identical.
* Inside the config-3 V(3,3) hierarchy (levels 3 -> 1) the V-cycle equals the generic-path V-cycle.
"""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2506_04157_b200 as hhg  # noqa: E402
from tests.harness import BC_SHELL, canon, lib_eta, lib_mesh, lib_u, rel_l2  # noqa: E402
from workload import icoshell, uniform_vec  # noqa: E402

C3 = (1e6, 30.0)


def _with_env(var, make):
    os.environ[var] = "1"
    try:
        return make()
    finally:
        del os.environ[var]


def _pair(make):
    """(cluster-kernel object, generic-path object) built by make()"""
    return make(), _with_env("HHG_NO_CCL", make)


@pytest.mark.parametrize("blend,form,level", [(True, hhg.HHG_VISC_FULL, 1), (False, hhg.HHG_VISC_EPS, 1),
                                              (True, hhg.HHG_VISC_FULL, 2)])
def test_coarse_pcg_matches_oracle_and_generic_path(blend, form, level):
    from oracle.multigrid import Hierarchy
    from oracle.operators import FORM_EPS, FORM_FULL, Discretisation, node_coords
    from oracle.refine import build_level
    from tests.harness import oracle_bc
    from workload import viscosity
    mac = icoshell(3, 2)
    lm = build_level(mac.verts, mac.tets, mac.vtag, level)
    eta_o = viscosity(node_coords(lm, "P1", blend), lm.p1_keys, *C3)
    d = Discretisation(lm, blend, eta_o, 0.0, oracle_bc(BC_SHELL), build=("A",),
                       form=FORM_FULL if form == hhg.HHG_VISC_FULL else FORM_EPS)
    H = Hierarchy({1: d}, {}, coarse_iters=50)
    f_o = d.project(uniform_vec(lm.p2_keys, 4))
    x_o = H.vcycle(f_o)
    M = lib_mesh(mac, level, blend, BC_SHELL)
    eta = {level: lib_eta(M, level, C3)}
    mk = lambda: hhg.MG(M, level, level, eta, {}, coarse_iters=50, form=form)  # noqa: E731
    mg, mg_ref = _pair(mk)
    mg_gl = _with_env("HHG_CCL_GLOBAL", mk)  # the global-memory variant of the cluster kernel
    assert mg.coarse_iterations() == 0  # the cluster kernel serves this level (the generic path raises)
    f = lib_u(M, level, 4)
    x, x_ref, x_gl = mg.vcycle(f), mg_ref.vcycle(f), mg_gl.vcycle(f)
    x2 = mg.vcycle(f)
    torch.cuda.synchronize()
    assert mg.coarse_iterations() == 50
    e_o = rel_l2(canon(M, level, hhg.HHG_P2VEC, x), x_o)
    e_g = float((x - x_ref).norm() / x_ref.norm())
    print(f"coarse PCG level {level} blend={blend} form={form}: vs oracle {e_o:.2e}, vs generic path {e_g:.2e}, "
          f"shared-memory vs global variant {float((x - x_gl).norm() / x_ref.norm()):.2e}")
    assert e_o <= 1e-9 and e_g <= 1e-9
    assert torch.equal(x, x2), "cluster coarse PCG must be bitwise reproducible"
    # the two objects' D^-1 come from the (RED-summed) diag kernel, so they agree to rounding, not bitwise
    assert float((x - x_gl).norm() / x_ref.norm()) <= 1e-14


def test_coarse_pcg_quadrature_point_viscosity():
    from tests.test_gpu_parity import _temperature_p2
    mac = icoshell(3, 2)
    M = lib_mesh(mac, 1, True, BC_SHELL)
    qeta = (np.log(1e6), 30.0, 0.9)
    mk = lambda: hhg.MG(M, 1, 1, {1: lib_eta(M, 1, C3)}, {}, coarse_iters=50, T2_per_level={1: _temperature_p2(M, 1)},  # noqa: E731
                        l_eta=1, qeta=qeta)
    mg, mg_ref = _pair(mk)
    f = lib_u(M, 1, 4)
    x, x_ref = mg.vcycle(f), mg_ref.vcycle(f)
    torch.cuda.synchronize()
    e_g = float((x - x_ref).norm() / x_ref.norm())
    print(f"coarse PCG, quadrature-point viscosity: vs generic path {e_g:.2e}")
    assert e_g <= 1e-8  # the 50-iteration PCG on this operator amplifies rounding to ~1e-9


def test_config3_vcycle_cluster_coarse_equals_generic():
    M = lib_mesh(icoshell(3, 2), 3, True, BC_SHELL)
    levels = (1, 2, 3)
    etas = {L: lib_eta(M, L, C3) for L in levels}

    def mk():  # fresh power-iteration start vectors per hierarchy (hhg_mg_create overwrites them)
        pv = {L: M.from_canonical(L, hhg.HHG_P2VEC, uniform_vec(M.canonical_keys(L, hhg.HHG_P2), 6)) for L in levels[1:]}
        return hhg.MG(M, 1, 3, etas, pv, pre=3, post=3, degree=3, power_iters=20, coarse_iters=50)
    mg, mg_ref = _pair(mk)
    f = lib_u(M, 3, 4)
    x_ref = mg_ref.vcycle(f)  # eager launches, generic coarse path
    x_eager = mg.vcycle(f)    # eager launches, cluster coarse kernel
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):  # graph-captured V-cycles
        x = mg.vcycle(f, stream=s)
        x_ref_g = mg_ref.vcycle(f, stream=s)
    s.synchronize()
    e_eager = float((x_eager - x_ref).norm() / x_ref.norm())
    e = float((x - x_ref).norm() / x_ref.norm())
    e_g = float((x_ref_g - x_ref).norm() / x_ref.norm())
    print(f"config-3 V(3,3) L3->1: cluster coarse vs generic: eager {e_eager:.2e}, graph {e:.2e} (generic graph vs "
          f"eager {e_g:.2e})")
    assert e_eager <= 1e-11 and e <= 1e-11 and e_g <= 1e-11


@pytest.mark.parametrize("tol,level", [(1e-2, 1), (1e-6, 1), (1e-2, 2)])
def test_coarse_pcg_relative_tolerance_matches_oracle(tol, level):
    """coarse_tol (Table 1 tol_coarse = 1e-2): stop at sqrt(r.z) <= tol sqrt(r0.z0) -- same iteration count
    as the oracle's PCG and the same iterate."""
    from oracle.multigrid import pcg
    from tests.harness import oracle_case
    mac = icoshell(3, 2)
    lm, d, _ = oracle_case(mac, level, True, BC_SHELL, C3, 0.0, build=("A",))
    f_o = d.project(uniform_vec(lm.p2_keys, 4))
    x_o, it_o = pcg(d.Ac(), 1.0 / d.diagA(), d.Pm, f_o, 5000, tol=tol, count=True)
    M = lib_mesh(mac, level, True, BC_SHELL)
    mg = hhg.MG(M, level, level, {level: lib_eta(M, level, C3)}, {}, coarse_iters=5000, coarse_tol=tol)
    x = mg.vcycle(lib_u(M, level, 4))
    it = mg.coarse_iterations()
    e = rel_l2(canon(M, level, hhg.HHG_P2VEC, x), x_o)
    # the method's own rounding sensitivity after `it` iterations on this operator: the oracle's PCG on a rhs
    # perturbed by 1e-16 relative (fixed iteration count) -- two correct implementations differ by about that much
    rng = np.random.default_rng(0)
    f_p = d.project(f_o * (1.0 + 1e-16 * rng.standard_normal(f_o.shape)))
    floor = rel_l2(pcg(d.Ac(), 1.0 / d.diagA(), d.Pm, f_p, it_o), x_o)
    print(f"coarse PCG level {level} tol {tol:g}: {it} iterations (oracle {it_o}), vs oracle {e:.2e}, oracle rounding floor "
          f"{floor:.2e}")
    assert it == it_o and 0 < it < 5000
    assert e <= max(1e-9, 10.0 * floor), (e, floor)
