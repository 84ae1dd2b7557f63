"""GPU parity of the temperature operator of eq:WeakTemp (SURVEY §8(f) NEXT-4 without MMOC)
and its FGMRES/CG solve against oracle/temperature.py: blended shell(3,2), seeded velocity,
TALA-like rho coupling."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2506_04157_b200 as hhg  # noqa: E402
from tests.harness import BC_SHELL, canon, lib_mesh, rel_l2  # noqa: E402
from workload import icoshell, uniform_vec, uniform_from_keys, GAMMA_TALA  # noqa: E402

PRM = dict(s=1.5, tau=0.05, kappa=1.0, beta=0.5, gamma=GAMMA_TALA)


def _case(L, blended=True):
    from oracle.refine import build_level
    mac = icoshell(3, 2)
    lm = build_level(mac.verts, mac.tets, mac.vtag, L)
    M = lib_mesh(mac, L, blended, BC_SHELL)
    u_o = 0.5 * uniform_vec(lm.p2_keys, 2)
    u = M.from_canonical(L, hhg.HHG_P2VEC, 0.5 * uniform_vec(M.canonical_keys(L, hhg.HHG_P2), 2))
    return lm, M, u_o, u


@pytest.mark.parametrize("blended", [True, False])
def test_temperature_operator_apply(blended):
    from oracle.temperature import assemble_temperature
    L = 2
    lm, M, u_o, u = _case(L, blended)
    Lo, Po = assemble_temperature(lm, blended, u_o, **PRM)
    T_o = uniform_from_keys(lm.p2_keys, 3, 0)
    T = M.from_canonical(L, hhg.HHG_P2, uniform_from_keys(M.canonical_keys(L, hhg.HHG_P2), 3, 0))
    for which, ref in ((0, Lo @ T_o), (1, Po @ T_o), (2, Po.diagonal())):
        y = hhg.hhg_temp_apply(M, L, PRM, u, T, which=which)
        assert rel_l2(canon(M, L, hhg.HHG_P2, y), ref) <= 1e-11, which


def test_temperature_solve_matches_direct_solve():
    """FGMRES + CG(P) to 1e-12 reproduces the oracle's direct Dirichlet solve."""
    from oracle.temperature import assemble_temperature, boundary_mask, solve_temperature
    L = 2
    lm, M, u_o, u = _case(L)
    Lo, _ = assemble_temperature(lm, True, u_o, **PRM)
    mask = boundary_mask(lm)
    TD_o = uniform_from_keys(lm.p2_keys, 9, 0)
    b_o = uniform_from_keys(lm.p2_keys, 4, 0)
    T_ref = solve_temperature(Lo, b_o, TD_o, mask)
    keys = M.canonical_keys(L, hhg.HHG_P2)
    T = M.from_canonical(L, hhg.HHG_P2, uniform_from_keys(keys, 9, 0))
    b = M.from_canonical(L, hhg.HHG_P2, uniform_from_keys(keys, 4, 0))
    S = hhg.TempSolver(M, L, PRM, restart=50)
    T, it, rel = S.solve(u, b, T, tol=1e-12, max_iters=100)
    assert rel <= 1e-12 and it < 30, (it, rel)
    assert rel_l2(canon(M, L, hhg.HHG_P2, T), T_ref) <= 1e-9


@pytest.mark.parametrize("L,scale", [(1, 0.3), (2, 0.3)])
def test_mmoc_matches_oracle(L, scale):
    """MMOC on the blended shell: seeded u_new, u_old (displacements ~ a micro-tet size),
    seeded T; every P2 node against the oracle's RK4 back-tracking with brute-force point location."""
    from oracle.mmoc import mmoc
    lm, M, u_o, u = _case(L)
    keys = M.canonical_keys(L, hhg.HHG_P2)
    un_o = scale * uniform_vec(lm.p2_keys, 2)
    uo_o = scale * uniform_vec(lm.p2_keys, 5)
    T_o = uniform_from_keys(lm.p2_keys, 3, 0)
    tau = 0.1
    ref = mmoc(lm, True, T_o, un_o, uo_o, tau)
    un = M.from_canonical(L, hhg.HHG_P2VEC, scale * uniform_vec(keys, 2))
    uo = M.from_canonical(L, hhg.HHG_P2VEC, scale * uniform_vec(keys, 5))
    T = M.from_canonical(L, hhg.HHG_P2, uniform_from_keys(keys, 3, 0))
    Th = hhg.hhg_mmoc(M, L, T, un, uo, tau)
    got = canon(M, L, hhg.HHG_P2, Th)
    assert np.abs(got - ref).max() <= 1e-11 * np.abs(ref).max()
    z = torch.zeros_like(un)
    assert torch.equal(hhg.hhg_mmoc(M, L, T, z, z, tau), T) or \
        float((hhg.hhg_mmoc(M, L, T, z, z, tau) - T).abs().max()) <= 1e-13
