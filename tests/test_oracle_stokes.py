"""Pins of oracle/stokes.py (FGMRES + symmetric Uzawa): on the isoviscous
unblended reference tet the preconditioned solve reaches the solution of the saddle-point system
computed by a direct sparse solve (pressure fixed by a mean-zero Lagrange multiplier), stops at the
requested relative residual, and the mass-matrix CG solves M_{1/eta} z = r."""
import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as sla

from oracle.multigrid import Hierarchy
from oracle.operators import Discretisation
from oracle.refine import build_level, BC_DIRICHLET
from oracle.stokes import StokesOracle, mass_cg
from workload import reference_tet, uniform_vec, uniform_from_keys


@pytest.fixture(scope="module")
def tet_case():
    m = reference_tet()
    discs, v0 = {}, {}
    for L in (1, 2):
        lm = build_level(m.verts, m.tets, m.vtag, L)
        discs[L] = Discretisation(lm, False, None, 0.0, {"all": BC_DIRICHLET}, build=("A", "B", "C", "M"))
        v0[L] = uniform_vec(lm.p2_keys, 6)
    H = Hierarchy(discs, v0, pre=3, post=3, degree=3)
    return discs, H


def test_mass_cg_solves_mass_system(tet_case):
    discs, _ = tet_case
    M = discs[2].M
    r = uniform_from_keys(discs[2].lm.p1_keys, 5, 0)
    z = mass_cg(M, r, tol=1e-13, max_iters=500)
    assert np.linalg.norm(M @ z - r) <= 1e-12 * np.linalg.norm(r)


def test_fgmres_uzawa_recovers_a_manufactured_solution(tet_case):
    """rhs = P K P x* for a seeded x* (velocity constrained, pressure mean zero): the solve recovers
    the velocity (unique) to the tolerance-implied accuracy, and P K P (x - x*) = 0 (pressure is
    only unique up to the kernel of P B^T: constants and, on this all-Dirichlet macro, corner modes)."""
    discs, H = tet_case
    d = discs[2]
    S = StokesOracle(H, d, d.M, tol_A=1e-2)
    n2 = 3 * d.lm.n_p2
    xs = np.concatenate([d.project(uniform_vec(d.lm.p2_keys, 2)), uniform_from_keys(d.lm.p1_keys, 3, 0)])
    xs[n2:] -= xs[n2:].mean()
    rhs = S.op(xs)
    x, it, rel = S.solve(rhs, tol=1e-11, restart=40, max_iters=200)
    assert rel <= 1e-11
    assert np.linalg.norm(x[:n2] - xs[:n2]) <= 1e-9 * np.linalg.norm(xs[:n2])
    assert np.linalg.norm(S.op(x - xs)) <= 1e-10 * np.linalg.norm(rhs)
    assert abs(x[n2:].mean()) <= 1e-13 * np.abs(x[n2:]).max()
    # the velocity also solves A u = f - B^T p of the direct reduced system for the returned pressure
    f = rhs[:n2] - d.Pm @ (d.B.T @ x[n2:])
    Areg = (H.Ac[2] + sp.identity(n2) - d.Pm).tocsc()
    assert np.linalg.norm(sla.spsolve(Areg, f) - x[:n2]) <= 1e-9 * np.linalg.norm(x[:n2])
    # a loose tolerance stops earlier and still meets it
    x2, it2, rel2 = S.solve(rhs, tol=1e-3, restart=40, max_iters=200)
    assert rel2 <= 1e-3 and it2 < it


def test_fgmres_uzawa_vbfbt_recovers_a_manufactured_solution(tet_case):
    """Same manufactured solve with the V-cycle BFBT Schur approximation (eq:schurV, A_C = V(1,1) with
    degree-1 Chebyshev, B A_C^-1 B^T by M_{1/eta}-preconditioned CG to 0.1)."""
    discs, H = tet_case
    d = discs[2]
    v0 = {L: uniform_vec(discs[L].lm.p2_keys, 6) for L in (1, 2)}
    HC = Hierarchy(discs, v0, pre=1, post=1, degree=1)
    S = StokesOracle(H, d, d.M, tol_A=1e-2, schur="vbfbt", HC=HC, tol_vbfbt=1e-1)
    n2 = 3 * d.lm.n_p2
    xs = np.concatenate([d.project(uniform_vec(d.lm.p2_keys, 2)), uniform_from_keys(d.lm.p1_keys, 3, 0)])
    xs[n2:] -= xs[n2:].mean()
    rhs = S.op(xs)
    x, it, rel = S.solve(rhs, tol=1e-10, restart=60, max_iters=200)
    assert rel <= 1e-10
    assert np.linalg.norm(x[:n2] - xs[:n2]) <= 1e-8 * np.linalg.norm(xs[:n2])
    assert np.linalg.norm(S.op(x - xs)) <= 1e-9 * np.linalg.norm(rhs)


@pytest.mark.parametrize("uzawa", ["inexact", "adjoint"])
def test_uzawa_variants_recover_a_manufactured_solution(tet_case, uzawa):
    """Inexact (eq:InexactUzawaStep1) and adjoint inexact (eq:AdjointInexactUzawaStep1) Uzawa as
    FGMRES preconditioners also reach the manufactured velocity."""
    discs, H = tet_case
    d = discs[2]
    S = StokesOracle(H, d, d.M, tol_A=1e-2, uzawa=uzawa)
    n2 = 3 * d.lm.n_p2
    xs = np.concatenate([d.project(uniform_vec(d.lm.p2_keys, 2)), uniform_from_keys(d.lm.p1_keys, 3, 0)])
    xs[n2:] -= xs[n2:].mean()
    rhs = S.op(xs)
    x, it, rel = S.solve(rhs, tol=1e-10, restart=80, max_iters=200)
    assert rel <= 1e-10
    assert np.linalg.norm(x[:n2] - xs[:n2]) <= 1e-7 * np.linalg.norm(xs[:n2])  # residual 1e-10 x conditioning

