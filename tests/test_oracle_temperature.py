"""Pins of oracle/temperature.py (the eq:WeakTemp operator) against closed forms: the mass
part integrates 1 to |Omega|; the diffusion part (gamma = 0) annihilates constants, integrates
|grad(c.x)|^2 exactly and has zero interior rows for linear T; with gamma != 0 the interior rows for
linear T are int kappa c . grad(phi_a / rho) = 0 up to the quadrature error, which vanishes under
refinement (a transposed coupling term would not); the advection part for constant u and linear T
is (u . c) int phi_a; the adiabatic term for T = 1 and the radial field u = x/|x| sums to beta |Omega|; the direct
solve honours the Dirichlet values and the interior equations."""
import numpy as np
import pytest

from oracle.refine import build_level
from oracle.temperature import assemble_temperature, boundary_mask, solve_temperature
from workload import icoshell, reference_tet, uniform_from_keys


def _vol(X):
    E = X[:, 1:] - X[:, :1]
    return np.abs(np.linalg.det(E)) / 6.0


@pytest.fixture(scope="module")
def flat_shell():
    m = icoshell(3, 2)
    return m, build_level(m.verts, m.tets, m.vtag, 1)


def test_mass_and_diffusion_closed_forms(flat_shell):
    m, lm = flat_shell
    zero_u = np.zeros(3 * lm.n_p2)
    vol = float(_vol(lm.X).sum())
    Lm, _ = assemble_temperature(lm, False, zero_u, s=1.0, tau=0.0)
    one = np.ones(lm.n_p2)
    assert abs(one @ Lm @ one - vol) < 1e-13 * vol
    Kd, Ps = assemble_temperature(lm, False, zero_u, s=0.0, tau=1.0, kappa=1.0, beta=0.0, gamma=0.0)
    assert np.abs(Kd @ one).max() < 1e-13
    assert abs(Kd - Kd.T).max() < 1e-14 and abs(Kd - Ps).max() < 1e-14     # gamma = 0: L = P
    c = np.array([0.4, -0.9, 1.3])
    T = lm.p2_xt @ c
    assert abs(T @ Kd @ T - c @ c * vol) < 1e-12 * vol
    interior = lm.p2_keys[:, 0] == 3
    assert np.abs((Kd @ T)[interior]).max() < 1e-13


def test_rho_coupling_interior_rows_vanish_under_refinement():
    """gamma != 0 on the blended shell: rows of L T for linear T at interior nodes approximate
    int kappa c . grad(phi_a / rho) = 0; the error decays with h (>= 4x per level), while the row scale
    |int kappa/rho c . grad phi_a| does not vanish that fast."""
    m = icoshell(3, 2)
    errs = []
    for L in (1, 2):
        lm = build_level(m.verts, m.tets, m.vtag, L)
        Kd, Ps = assemble_temperature(lm, True, np.zeros(3 * lm.n_p2), s=0.0, tau=1.0, kappa=1.0, beta=0.0, gamma=2.0)
        c = np.array([0.4, -0.9, 1.3])
        from oracle.operators import node_coords
        T = node_coords(lm, "P2", True) @ c
        interior = lm.p2_keys[:, 0] == 3
        e = np.abs((Kd @ T)[interior]).max()
        scale = np.abs((Ps @ T)[interior]).max()
        errs.append(e)
        assert e < 0.2 * scale          # the symmetric part alone leaves an O(1) fraction: the coupling cancels it
    assert errs[1] < errs[0] / 4.0


def test_advection_and_adiabatic_terms(flat_shell):
    m, lm = flat_shell
    u = np.tile([0.3, -0.2, 0.5], lm.n_p2)
    c = np.array([0.4, -0.9, 1.3])
    T = lm.p2_xt @ c
    vol = float(_vol(lm.X).sum())
    La, _ = assemble_temperature(lm, False, u, s=0.0, tau=1.0, kappa=0.0, beta=0.0, gamma=0.0)
    # (u . c) int phi_a: summed over a it is (u . c) |Omega|; per row it equals (u.c) M 1
    Mm, _ = assemble_temperature(lm, False, np.zeros(3 * lm.n_p2), s=1.0, tau=0.0)
    uc = float(np.array([0.3, -0.2, 0.5]) @ c)
    assert np.abs(La @ T - uc * (Mm @ np.ones(lm.n_p2))).max() < 1e-14
    assert abs((La @ T).sum() - uc * vol) < 1e-12 * vol
    # adiabatic term: -beta int (u . g) phi_a for T = 1; with the radial field u = x/|x| (P2-interpolated)
    # u . g = -1 up to interpolation error, so the rows sum to beta |Omega| (and vanish for beta = 0)
    xr = lm.p2_xt / np.linalg.norm(lm.p2_xt, axis=1, keepdims=True)
    Lb, _ = assemble_temperature(lm, False, xr.ravel(), s=0.0, tau=1.0, kappa=0.0, beta=2.0, gamma=0.0)
    La0, _ = assemble_temperature(lm, False, xr.ravel(), s=0.0, tau=1.0, kappa=0.0, beta=0.0, gamma=0.0)
    one = np.ones(lm.n_p2)
    adi = (Lb - La0) @ one
    assert abs(adi.sum() - 2.0 * vol) < 2e-3 * 2.0 * vol
    assert np.abs(La0 @ one).max() < 1e-14       # advection of a constant vanishes


def test_direct_solve_honours_dirichlet_and_interior_equations(flat_shell):
    m, lm = flat_shell
    u = 0.1 * uniform_from_keys(np.repeat(lm.p2_keys, 1, axis=0), 2, 0)
    u = np.tile(u[:, None], (1, 3)).ravel()
    Lm, _ = assemble_temperature(lm, False, u, s=1.5, tau=0.01, kappa=1.0, beta=0.5, gamma=0.3)
    mask = boundary_mask(lm)
    r = np.linalg.norm(lm.p2_xt, axis=1)
    assert mask.sum() > 0 and (~mask).sum() > 0
    TD = np.where(r > 0.8, 0.0, 1.0)
    b = uniform_from_keys(lm.p2_keys, 4, 0)
    T = solve_temperature(Lm, b, TD, mask)
    assert np.array_equal(T[mask], TD[mask])
    assert np.abs((Lm @ T - b)[~mask]).max() < 1e-12 * np.abs(b).max()
