"""Pins of oracle/operators.py against properties fixed by the mathematics: symmetry and
positive semi-definiteness of A, its exact kernels (rigid motions, dilation, special
conformal fields), divergence identities of B, the integral that C approximates, and
optimal P2 convergence for a manufactured solution."""
import math

import numpy as np
import pytest
import scipy.sparse.linalg as sla
import sympy as sy

from oracle import fe
from oracle.refine import build_level, BC_DIRICHLET, BC_FREESLIP
from oracle.operators import Discretisation, FORM_FULL, FORM_EPS, quad_geometry
from workload import reference_tet, icoshell, MacroMesh


def collapsed_gauss(n=8):
    """Stroud conical product rule on the reference tet (cube -> tet, Duffy), exact to degree 2n-3."""
    g, w = np.polynomial.legendre.leggauss(n)
    g = 0.5 * (g + 1.0)
    w = 0.5 * w
    U, V, W = np.meshgrid(g, g, g, indexing="ij")
    WU, WV, WW = np.meshgrid(w, w, w, indexing="ij")
    x = U
    y = V * (1 - U)
    z = W * (1 - U) * (1 - V)
    jac = (1 - U) ** 2 * (1 - V)
    return np.stack([x.ravel(), y.ravel(), z.ravel()], 1), (WU * WV * WW * jac).ravel()


def test_collapsed_gauss_rule():
    xi, w = collapsed_gauss(6)
    assert abs(w.sum() - 1 / 6) < 1e-15
    assert abs(np.sum(w * xi[:, 0] ** 3 * xi[:, 1] ** 2 * xi[:, 2] ** 2) - 6 * 2 * 2 / math.factorial(10)) < 1e-16


def _reftet_disc(L, eta_fn=None, form=FORM_FULL, bc=None):
    m = reference_tet()
    lm = build_level(m.verts, m.tets, m.vtag, L)
    eta = None if eta_fn is None else eta_fn(lm.p1_xt)
    return Discretisation(lm, False, eta, 0.0, bc or {}, form=form)


def _interp(lm, fn):
    return fn(lm.p2_xt).reshape(-1)


def test_A_symmetric_psd_variable_eta_blended():
    m = icoshell(3, 2)
    lm = build_level(m.verts, m.tets, m.vtag, 0)
    eta = 1.0 + np.abs(lm.p1_xt[:, 0]) + lm.p1_xt[:, 1] ** 2
    d = Discretisation(lm, True, eta, 0.3781, {2: BC_DIRICHLET, 1: BC_FREESLIP})
    A = d.A.toarray()
    assert np.abs(A - A.T).max() <= 1e-14 * np.abs(A).max()
    ev = np.linalg.eigvalsh(A)
    assert ev.min() >= -1e-13 * ev.max()
    Ac = d.Ac().toarray()
    assert np.abs(Ac - Ac.T).max() <= 1e-14 * np.abs(A).max()
    assert np.linalg.eigvalsh(Ac).min() >= -1e-13 * ev.max()
    # blended: only translations stay in the kernel (dim 3), rotations do not
    nker = int(np.sum(np.abs(ev) < 1e-10 * ev.max()))
    assert nker == 3
    for c in range(3):
        t = np.zeros((lm.n_p2, 3))
        t[:, c] = 1.0
        assert np.abs(A @ t.ravel()).max() < 1e-12 * ev.max()
    rot = lambda x: np.stack([-x[:, 1], x[:, 0], 0 * x[:, 0]], 1)
    assert np.abs(A @ _interp(lm, rot)).max() > 1e-6


@pytest.mark.parametrize("form,dim_ker", [(FORM_FULL, 10), (FORM_EPS, 6)])
def test_A_kernel_unblended(form, dim_ker):
    d = _reftet_disc(1, lambda x: 1.0 + x[:, 0] + 2.0 * x[:, 1], form)
    A = d.A.toarray()
    ev = np.linalg.eigvalsh(A)
    assert int(np.sum(np.abs(ev) < 1e-10 * ev.max())) == dim_ker
    lm = d.lm
    fields = [lambda x, c=c: np.eye(3)[c][None, :] + 0 * x for c in range(3)]
    for (i, j) in [(0, 1), (0, 2), (1, 2)]:
        def rot(x, i=i, j=j):
            v = np.zeros_like(x)
            v[:, i] = -x[:, j]
            v[:, j] = x[:, i]
            return v
        fields.append(rot)
    if form == FORM_FULL:
        fields.append(lambda x: x.copy())                       # dilation
        for b in np.eye(3):
            fields.append(lambda x, b=b: 2 * (x @ b)[:, None] * x - (x * x).sum(1)[:, None] * b[None])
    for f in fields:
        assert np.abs(A @ _interp(lm, f)).max() < 1e-12 * ev.max()


def test_B_divergence_identities():
    # constant field is divergence free (also blended); Σ_i (B x)_i = -3 |Ω| unblended
    d = _reftet_disc(2)
    lm = d.lm
    B = d.B
    for c in range(3):
        t = np.zeros((lm.n_p2, 3))
        t[:, c] = 1.0
        assert np.abs(B @ t.ravel()).max() < 1e-15
    assert abs((B @ _interp(lm, lambda x: x.copy())).sum() + 3.0 / 6.0) < 1e-14
    # B^T 1 = 0 on interior rows (unblended): -∫ div phi_j = 0 for interior j
    bt1 = B.T @ np.ones(lm.n_p1)
    interior = np.repeat(lm.p2_keys[:, 0] == 3, 3)
    assert np.abs(bt1[interior]).max() < 1e-15
    m = icoshell(3, 2)
    lmb = build_level(m.verts, m.tets, m.vtag, 1)
    db = Discretisation(lmb, True, None, 0.0, {}, build=("B",))
    for c in range(3):
        t = np.zeros((lmb.n_p2, 3))
        t[:, c] = 1.0
        assert np.abs(db.B @ t.ravel()).max() < 1e-15


def test_C_is_linear_in_gamma_and_converges_to_its_integral():
    """p=1, u=e_x: p^T C u = -∫ grad ln rho . e_x = gamma ∫ x/|x| dx over a shifted tet."""
    shift = np.array([0.3, 0.4, 0.5])
    m = MacroMesh(reference_tet().verts + shift, reference_tet().tets, reference_tet().vtag)
    xi, w = collapsed_gauss(24)
    x = xi + shift
    exact = 0.7 * float(np.sum(w * x[:, 0] / np.linalg.norm(x, axis=1)))
    errs = []
    for L in range(4):
        lm = build_level(m.verts, m.tets, m.vtag, L)
        u = np.zeros((lm.n_p2, 3))
        u[:, 0] = 1.0
        d1 = Discretisation(lm, False, None, 0.7, {}, build=("C",))
        d2 = Discretisation(lm, False, None, 1.4, {}, build=("C",))
        v1 = d1.C @ u.ravel()
        assert np.abs(d2.C @ u.ravel() - 2 * v1).max() < 1e-15
        errs.append(abs(v1.sum() - exact))
    assert errs[-1] < 1e-7, errs
    # composite degree-2 rule on a smooth integrand: asymptotically O(h^4) (ratios -> 16)
    assert errs[0] > errs[1] and all(errs[i] / errs[i + 1] > 10 for i in (1, 2)), errs


def test_blended_C_against_closed_forms_on_the_shell():
    """Blended C (-(grad ln rho . u, q) with grad ln rho = -gamma x/|x|, i.e. q^T C u = gamma ∫ (d.u) q on
    the shell mapped exactly by the blending) against integrals known in closed form:
    u = x/|x| (d.u = 1):  1^T C u -> gamma |Omega| = gamma 4/3 pi (r_o^3 - r_i^3),  r^T C u -> gamma pi (r_o^4 - r_i^4);
    u = e_z x x (tangential, d.u = 0): C u -> 0.  Errors fall like O(h^4) (composite degree-2 rule, smooth
    integrands); a missing |det J_B|, a wrong sign or a transposed J_B in the blended path fails the limits."""
    from oracle.operators import node_coords
    m = icoshell(3, 2)
    ri, ro, g = 0.55, 1.0, 0.7
    vol, rint = 4.0 / 3.0 * math.pi * (ro**3 - ri**3), math.pi * (ro**4 - ri**4)
    e_vol, e_r, e_tan = [], [], []
    for L in range(3):
        lm = build_level(m.verts, m.tets, m.vtag, L)
        d = Discretisation(lm, True, None, g, {}, build=("C",))
        x2, x1 = node_coords(lm, "P2", True), node_coords(lm, "P1", True)
        v = d.C @ (x2 / np.linalg.norm(x2, axis=1)[:, None]).ravel()
        e_vol.append(abs(v.sum() / (g * vol) - 1.0))
        e_r.append(abs(np.linalg.norm(x1, axis=1) @ v / (g * rint) - 1.0))
        ut = np.stack([-x2[:, 1], x2[:, 0], np.zeros(x2.shape[0])], 1)
        e_tan.append(np.abs(d.C @ ut.ravel()).max() / np.abs(v).max())
    assert e_vol[-1] < 2e-5 and e_r[-1] < 2e-5 and e_tan[-1] < 1e-3, (e_vol, e_r, e_tan)
    for e in (e_vol, e_r):
        assert all(e[i] / e[i + 1] > 8 for i in (0, 1)), e
    assert e_tan[0] > e_tan[1] > e_tan[2], e_tan


def _manufactured():
    X, Y, Z = sy.symbols("x y z")
    b = X * Y * Z * (1 - X - Y - Z)
    u = sy.Matrix([b * sy.sin(X + 2 * Y), 2 * b, -b * sy.cos(Z)])
    eta = 1 + X + 2 * Y
    grad = u.jacobian([X, Y, Z])
    eps = (grad + grad.T) / 2
    dev = eps - sy.eye(3) * (grad.trace() / 3)
    tau = 2 * eta * dev
    f = -sy.Matrix([sum(sy.diff(tau[i, j], v) for j, v in enumerate((X, Y, Z))) for i in range(3)])
    fu = sy.lambdify((X, Y, Z), list(u), "numpy")
    ff = sy.lambdify((X, Y, Z), list(f), "numpy")
    return lambda x: np.stack(np.broadcast_arrays(*fu(x[:, 0], x[:, 1], x[:, 2])), 1), \
        lambda x: np.stack(np.broadcast_arrays(*ff(x[:, 0], x[:, 1], x[:, 2])), 1)


def test_manufactured_solution_converges_at_order_3_in_L2():
    """-div(2 eta dev eps(u*)) = f on the reference tet, u* = 0 on the boundary:
    the oracle's A (Q4, P1 eta) must give optimal O(h^3) L2 error for P2."""
    u_ex, f_ex = _manufactured()
    xi, w = collapsed_gauss(7)
    phi = fe.p2_basis(xi)
    errs = []
    for L in (1, 2, 3):
        d = _reftet_disc(L, lambda x: 1.0 + x[:, 0] + 2.0 * x[:, 1], FORM_FULL, {"all": BC_DIRICHLET})
        lm = d.lm
        X = lm.X
        JF = np.stack([X[:, 1] - X[:, 0], X[:, 2] - X[:, 0], X[:, 3] - X[:, 0]], axis=2)
        det = np.abs(np.linalg.det(JF))
        xq = X[:, 0][:, None, :] + np.einsum("tij,qj->tqi", JF, xi)       # (T,Q,3)
        fq = f_ex(xq.reshape(-1, 3)).reshape(xq.shape)
        F = np.zeros((lm.n_p2, 3))
        contrib = np.einsum("q,t,tqc,qa->tac", w, det, fq, phi)
        np.add.at(F, lm.tet_p2, contrib)
        F = d.project(F.ravel())
        A = d.Ac()
        free = d.free_dofs()
        uh = np.zeros(3 * lm.n_p2)
        uh[free] = sla.spsolve(A[free][:, free].tocsc(), F[free])
        uq = np.einsum("qa,tac->tqc", phi, uh.reshape(-1, 3)[lm.tet_p2])
        e2 = np.einsum("q,t,tq->", w, det, ((uq - u_ex(xq.reshape(-1, 3)).reshape(xq.shape)) ** 2).sum(2))
        errs.append(math.sqrt(e2))
    rates = [math.log2(errs[i] / errs[i + 1]) for i in range(2)]
    assert rates[1] >= 2.8, (errs, rates)


def test_pressure_mass_closed_forms():
    """M_{1/eta} (eq:schurMass): with eta = 1, 1^T M 1 = |Omega| (reference tet: 1/6); element matrix
    |K|/20 (1 + delta_pr) (degree-2 rule is exact for P1 x P1); scaling eta -> c eta gives M / c;
    symmetric positive definite."""
    import scipy.sparse.linalg as sla
    from oracle.refine import build_level
    from oracle.operators import Discretisation
    from workload import reference_tet
    m = reference_tet()
    lm = build_level(m.verts, m.tets, m.vtag, 1)
    d = Discretisation(lm, False, None, 0.0, {}, build=("M",))
    one = np.ones(lm.n_p1)
    assert abs(one @ d.M @ one - 1.0 / 6.0) < 1e-15
    lm0 = build_level(m.verts, m.tets, m.vtag, 0)
    M0 = Discretisation(lm0, False, None, 0.0, {}, build=("M",)).M.toarray()
    assert np.abs(M0 - (1.0 / 6.0) / 20.0 * (np.ones((4, 4)) + np.eye(4))).max() < 1e-16
    d3 = Discretisation(lm, False, 3.0 * np.ones(lm.n_p1), 0.0, {}, build=("M",))
    assert abs(d3.M - d.M / 3.0).max() < 1e-17
    assert abs(d.M - d.M.T).max() < 1e-18
    assert sla.eigsh(d.M, k=1, which="SA")[0][0] > 0


def test_buoyancy_load_closed_forms():
    """Config-4 buoyancy load: linear in (T - 1/2); T = 1/2 gives 0; a uniform T = 3/2 gives
    b . e = int (x/|x|) . e over the domain for the constant field e (partition of unity of P2),
    which for the blended shell and e = e_z vanishes by symmetry and for the radial test field
    v = x (nodal interpolation) equals int |x| = pi (r1^4 - r0^4) up to the quadrature error."""
    from oracle.refine import build_level
    from oracle.operators import buoyancy_load, node_coords
    from workload import icoshell
    m = icoshell(3, 2)
    lm = build_level(m.verts, m.tets, m.vtag, 2)
    half = np.full(lm.n_p1, 0.5)
    assert np.abs(buoyancy_load(lm, True, half)).max() == 0.0
    b = buoyancy_load(lm, True, np.full(lm.n_p1, 1.5))
    ez = np.zeros(3 * lm.n_p2)
    ez[2::3] = 1.0
    x2 = node_coords(lm, "P2", True).ravel()
    radial = b @ x2
    assert abs(radial - np.pi * (1.0 - 0.55 ** 4)) < 1e-4 * np.pi
    assert abs(b @ ez) < 1e-5 * radial          # zero for the exact shell; discretisation-level here
    rng = np.random.default_rng(0)
    T1, T2 = rng.uniform(0, 1, lm.n_p1), rng.uniform(0, 1, lm.n_p1)
    lin = buoyancy_load(lm, True, 2 * T1 - T2)
    assert np.abs(lin - (2 * buoyancy_load(lm, True, T1) - buoyancy_load(lm, True, T2) - buoyancy_load(lm, True, half))).max() < 1e-14


def test_quadrature_point_viscosity_tier_special_cases():
    """NEXT-2 tier: with a constant temperature T = t0 and no jump the quadrature-point
    viscosity is the constant exp(lnC (1/2 - t0)), so A equals the P1-eta operator with that constant;
    a jump radius beyond the domain multiplies A by the jump factor."""
    from oracle.refine import build_level
    from oracle.operators import Discretisation
    from workload import icoshell
    m = icoshell(3, 2)
    lm = build_level(m.verts, m.tets, m.vtag, 1)
    lnC, t0 = np.log(1e4), 0.3
    T = np.full(lm.n_p2, t0)
    dq = Discretisation(lm, True, None, 0.0, {}, build=("A",), T_p2=T, qeta=(lnC, 1.0, 0.0))
    e = np.exp(lnC * (0.5 - t0))
    dp = Discretisation(lm, True, np.full(lm.n_p1, e), 0.0, {}, build=("A",))
    assert abs(dq.A - dp.A).max() <= 1e-13 * abs(dp.A).max()
    dj = Discretisation(lm, True, None, 0.0, {}, build=("A",), T_p2=T, qeta=(lnC, 30.0, 2.0))
    assert abs(dj.A - 30.0 * dq.A).max() <= 1e-13 * abs(dj.A).max()


def test_sampled_rows_equal_assembled_rows_shell_level2():
    """Pin of sampled_rows (the checker of every full-size parity test): on the blended shell at L2 with
    the TALA term (gamma = 0.3781), config-2 viscosity and constraints, its rows at nodes sampled on macro
    vertices, edges, faces and cells equal the rows of the fully assembled Discretisation."""
    from oracle.refine import build_level, node_bc
    from oracle.operators import Discretisation, node_coords, sampled_rows
    from workload import icoshell, uniform_vec, uniform_from_keys, viscosity, GAMMA_TALA
    mac = icoshell(3, 2)
    lm = build_level(mac.verts, mac.tets, mac.vtag, 2)
    bc_tags = {2: 1, 1: 2}
    eta = viscosity(node_coords(lm, "P1", True), lm.p1_keys, 1e4, 10.0)
    d = Discretisation(lm, True, eta, GAMMA_TALA, bc_tags)
    u = d.project(uniform_vec(lm.p2_keys, 2))
    p = uniform_from_keys(lm.p1_keys, 3, 0)
    yu_full = d.apply_A(u) + d.apply_BT(p)
    yp_full = d.apply_Bbar(u)
    rng = np.random.default_rng(3)
    s2 = np.unique(np.concatenate([np.nonzero(lm.p2_keys[:, 0] == dim)[0][rng.integers(0, 10**9, 25) %
                                   np.count_nonzero(lm.p2_keys[:, 0] == dim)] for dim in range(4)]))
    s1 = np.unique(np.concatenate([np.nonzero(lm.p1_keys[:, 0] == dim)[0][rng.integers(0, 10**9, 15) %
                                   np.count_nonzero(lm.p1_keys[:, 0] == dim)] for dim in range(4)]))
    assert {int(k) for k in lm.p2_keys[s2, 0]} == {0, 1, 2, 3}
    bc = node_bc(lm.p2_keys, lm.macro_tets, lm.macro_vtag, bc_tags)
    yu_s, yp_s = sampled_rows(lm, True, eta, GAMMA_TALA, u, p, s2, s1, bc)
    r2 = (3 * s2[:, None] + np.arange(3)).ravel()
    assert np.linalg.norm(yu_s[r2] - yu_full[r2]) <= 1e-13 * np.linalg.norm(yu_full[r2])
    assert np.linalg.norm(yp_s[s1] - yp_full[s1]) <= 1e-13 * np.linalg.norm(yp_full[s1])
