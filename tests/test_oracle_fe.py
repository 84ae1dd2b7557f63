"""Pins of oracle/fe.py and the oracle's element matrices against mathematics that does not
depend on the oracle: exact monomial integrals, exact rational element matrices (Fractions),
finite differences, the nodal property of the Lagrange basis, the exact shell volume."""
import math

import numpy as np
import pytest

from oracle import fe
from oracle.refine import build_level
from oracle.operators import Discretisation, FORM_FULL, FORM_EPS, quad_geometry, macro_blend
from tests import exact_poly as ep
from workload import reference_tet, icoshell


def test_q4_exact_to_degree_2_and_not_3():
    xi, w = fe.q4_rule()
    assert abs(w.sum() - 1.0 / 6.0) < 1e-16
    for a in range(4):
        for b in range(4 - a):
            for c in range(4 - a - b):
                q = float(np.sum(w * xi[:, 0] ** a * xi[:, 1] ** b * xi[:, 2] ** c))
                exact = float(ep.mono_integral(a, b, c))
                if a + b + c <= 2:
                    assert abs(q - exact) < 1e-16, (a, b, c)
    # degree 3 is not integrated exactly (so the rule is exactly degree 2)
    assert abs(np.sum(w * xi[:, 0] ** 3) - float(ep.mono_integral(3, 0, 0))) > 1e-6


def test_p2_basis_nodal_property_and_partition_of_unity():
    nodes = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1],
                      [.5, 0, 0], [0, .5, 0], [0, 0, .5], [.5, .5, 0], [.5, 0, .5], [0, .5, .5]])
    assert np.allclose(fe.p2_basis(nodes), np.eye(10), atol=1e-15)
    pts = np.random.default_rng(0).dirichlet(np.ones(4), size=50)[:, 1:]
    assert np.allclose(fe.p2_basis(pts).sum(axis=1), 1.0, atol=1e-14)
    assert np.allclose(fe.p2_grad(pts).sum(axis=1), 0.0, atol=1e-13)


def test_p2_gradient_matches_central_differences():
    pts = np.random.default_rng(1).dirichlet(np.ones(4), size=20)[:, 1:]
    g = fe.p2_grad(pts)
    h = 1e-6
    for d in range(3):
        e = np.zeros(3)
        e[d] = h
        fd = (fe.p2_basis(pts + e) - fe.p2_basis(pts - e)) / (2 * h)
        assert np.abs(fd - g[:, :, d]).max() < 1e-8


@pytest.mark.parametrize("form", [FORM_FULL, FORM_EPS])
def test_reference_element_matrices_equal_exact_rationals(form):
    """eta = 1, level 0 reference tet: Q4 is exact for the degree-2 integrand, so the oracle's
    element matrices must equal the exact rational integrals (computed here with Fractions)."""
    m = reference_tet()
    lm = build_level(m.verts, m.tets, m.vtag, 0)
    d = Discretisation(lm, False, None, 0.0, {}, form=form)
    Aex, Bex = ep.reference_element_matrices(form_full=(form == FORM_FULL))
    Aex = np.array([[float(v) for v in r] for r in Aex])
    Bex = np.array([[float(v) for v in r] for r in Bex])
    assert np.abs(d.A.toarray() - Aex).max() < 1e-14
    assert np.abs(d.B.toarray() - Bex).max() < 1e-15
    # a few of the printed-by-hand values
    if form == FORM_FULL:
        assert abs(Aex[0, 0] - 1 / 3) < 1e-15 and abs(np.trace(Aex) - 46 / 3) < 1e-13
        assert abs(Bex[0, 0] - 1 / 40) < 1e-16
    else:
        assert abs(Aex[0, 0] - 2 / 5) < 1e-15 and abs(np.trace(Aex) - 92 / 5) < 1e-13


def _shell_lm(level, ntan=3, nrad=2):
    m = icoshell(ntan, nrad)
    return m, build_level(m.verts, m.tets, m.vtag, level)


def test_blend_jacobian_matches_finite_differences():
    m, lm = _shell_lm(0)
    nhat, c = macro_blend(lm)
    rng = np.random.default_rng(2)
    X = lm.macro_verts[lm.macro_tets]
    lam = rng.dirichlet(np.ones(4), size=len(X))
    x = np.einsum("tv,tvd->td", lam, X)
    J = fe.blend_jacobian(x, nhat, c)
    h = 1e-6
    for d in range(3):
        e = np.zeros(3)
        e[d] = h
        fd = (fe.blend(x + e, nhat, c) - fe.blend(x - e, nhat, c)) / (2 * h)
        assert np.abs(fd - J[:, :, d]).max() < 1e-8


def test_blend_fixes_macro_vertices_maps_layers_to_spheres_and_is_continuous():
    m, lm = _shell_lm(0, 3, 3)
    nhat, c = macro_blend(lm)
    X = lm.macro_verts[lm.macro_tets]                      # (T,4,3)
    for v in range(4):
        assert np.abs(fe.blend(X[:, v], nhat, c) - X[:, v]).max() < 1e-14
    # points on a layer triangle (3 vertices of one radius) go to that sphere
    rng = np.random.default_rng(3)
    r = np.linalg.norm(X, axis=2)
    for t in range(len(X)):
        for skip in range(4):
            idx = [i for i in range(4) if i != skip]
            if np.ptp(r[t, idx]) < 1e-12:
                lam = rng.dirichlet(np.ones(3))
                p = lam @ X[t, idx]
                b = fe.blend(p[None], nhat[t:t + 1], c[t:t + 1])[0]
                assert abs(np.linalg.norm(b) - r[t, idx[0]]) < 1e-14
    # continuity: every interior macro face maps identically from both sides
    faces = {}
    for t, tet in enumerate(lm.macro_tets):
        for skip in range(4):
            f = tuple(int(v) for i, v in enumerate(tet) if i != skip)
            faces.setdefault(f, []).append(t)
    worst = 0.0
    for f, ts in faces.items():
        if len(ts) != 2:
            continue
        lam = rng.dirichlet(np.ones(3))
        p = lam @ lm.macro_verts[list(f)]
        b0 = fe.blend(p[None], nhat[ts[0]:ts[0] + 1], c[ts[0]:ts[0] + 1])
        b1 = fe.blend(p[None], nhat[ts[1]:ts[1] + 1], c[ts[1]:ts[1] + 1])
        worst = max(worst, np.abs(b0 - b1).max())
    assert worst < 1e-14


def test_blended_volume_converges_to_exact_shell_volume():
    """sum_q w_q |det J_F||det J_B| -> 4 pi/3 (1 - 0.55^3); Q4 error shrinks fast with level."""
    exact = 4.0 * math.pi / 3.0 * (1.0 - 0.55 ** 3)
    errs = []
    for L in (0, 1, 2):
        m, lm = _shell_lm(L)
        W, _, _ = quad_geometry(lm, np.arange(lm.n_tets), True, macro_blend(lm))
        errs.append(abs(W.sum() - exact) / exact)
    assert errs[2] < 1e-6
    assert errs[0] / errs[1] > 20 and errs[1] / errs[2] > 20
