"""Pins of the weighted-BFBT pieces of the oracle (eq:schurWBFBT and its a_l / a_r variant):
P1 prolongation (linear interpolation), the weighted P1 Laplacian K_{1/sqrt(eta)} and the weighted
vector mass M_{sqrt(eta)} against closed forms, the D_eta surface scaling against volumes computed
from the macro geometry, and the w-BFBT Stokes solve against a manufactured solution."""
import numpy as np
import pytest

from oracle.multigrid import Hierarchy, p1_prolongation
from oracle.operators import Discretisation
from oracle.refine import build_level, BC_DIRICHLET
from oracle.stokes import StokesOracle, neumann_solve
from workload import icoshell, reference_tet, uniform_vec, uniform_from_keys


def _vol(X):
    """Volumes of tets X (T,4,3) from the triple product."""
    E = X[:, 1:] - X[:, :1]
    return np.abs(np.linalg.det(E)) / 6.0


def _surface_volume(lm, outer_tag=2):
    """|D_eta|: micro tets with a vertex on the surface -- a micro vertex is on the outer sphere iff all
    macro vertices carrying a nonzero weight of it are outer-tagged (single radial layer: such vertex
    sets span outer faces, edges or vertices), from the integer macro weights, not from node keys."""
    mt = lm.macro_tets[lm.tet_macro]                       # (T,4) macro vertex ids
    outer = (lm.macro_vtag[mt] == outer_tag)[:, None, :]   # (T,1,4)
    on = ((lm.tet_w == 0) | outer).all(axis=2)             # (T,4 micro vertices)
    hit = on.any(axis=1)
    return float(_vol(lm.X[hit]).sum()), hit


def test_p1_prolongation_exact_on_linears():
    m = icoshell(3, 2)
    l0 = build_level(m.verts, m.tets, m.vtag, 1)
    l1 = build_level(m.verts, m.tets, m.vtag, 2)
    P = p1_prolongation(l0, l1)
    g = lambda x: x @ np.array([1.0, -2.0, 0.5]) + 3.0
    assert np.abs(P @ g(l0.p1_xt) - g(l1.p1_xt)).max() < 1e-13
    assert np.abs(P @ np.ones(l0.n_p1) - 1.0).max() < 1e-15
    assert set(np.round(P.data, 15)) <= {1.0, 0.5}
    # every fine node is a coarse node (one weight 1) or a coarse edge midpoint (two weights 1/2)
    nnz = np.diff(P.indptr)
    assert set(nnz) == {1, 2} and (nnz == 1).sum() == l0.n_p1


@pytest.mark.parametrize("a", [1.0, 3.0])
def test_weighted_laplacian_closed_forms(a):
    """Unblended shell(3,2), L2: K e = 0; for p = c.x (exact in P1) p^T K p = |c|^2 int omega with
    omega = 1 off D_eta and 1/a on it (eta = 1), and (K p)_i = 0 at interior nodes (int grad lam_i = 0);
    constant eta0 scales K by 1/sqrt(eta0); K symmetric positive semidefinite."""
    m = icoshell(3, 2)
    lm = build_level(m.verts, m.tets, m.vtag, 2)
    d = Discretisation(lm, False, None, 0.0, {}, build=("K",), surf_a=a)
    K = d.K
    assert abs(K - K.T).max() < 1e-15
    assert np.abs(K @ np.ones(lm.n_p1)).max() < 1e-13
    c = np.array([0.3, -1.1, 0.7])
    p = lm.p1_xt @ c
    vol = float(_vol(lm.X).sum())
    vD, hit = _surface_volume(lm)
    assert 0 < vD < vol and hit.sum() > 0
    assert abs(p @ K @ p - c @ c * (vol - vD + vD / a)) < 1e-12 * vol
    interior = lm.p1_keys[:, 0] == 3
    if a != 1.0:      # omega is constant on the support of nodes that touch no D_eta tet
        inD = np.zeros(lm.n_p1, dtype=bool)
        inD[lm.tet_p1[hit].ravel()] = True
        interior &= ~inD
    assert interior.sum() > 0 and np.abs((K @ p)[interior]).max() < 1e-13
    d4 = Discretisation(lm, False, np.full(lm.n_p1, 4.0), 0.0, {}, build=("K",), surf_a=a)
    assert abs(d4.K - 0.5 * K).max() < 1e-15
    w = np.linalg.eigvalsh(K.toarray())
    assert w.min() > -1e-12 and (w < 1e-10).sum() == 1      # one-dimensional kernel: constants


def test_weighted_vector_mass_closed_forms():
    """Reference tet, L1, eta = 1: 1^T VM_c 1 = |Omega| = 1/6 per component, no coupling between
    components; for f = c.x in one component f^T VM f = sum_T |T|/20 (sum f_i^2 + (sum f_i)^2) over the
    micro tets' vertices (the degree-2 rule is exact); constant eta0 scales VM by sqrt(eta0)."""
    m = reference_tet()
    lm = build_level(m.verts, m.tets, m.vtag, 1)
    d = Discretisation(lm, False, None, 0.0, {}, build=("VM",))
    VM = d.VM
    n2 = lm.n_p2
    for comp in range(3):
        e = np.zeros(3 * n2)
        e[comp::3] = 1.0
        assert abs(e @ VM @ e - 1.0 / 6.0) < 1e-15
        o = np.zeros(3 * n2)
        o[(comp + 1) % 3::3] = 1.0
        assert abs(e @ VM @ o) < 1e-16
    c = np.array([0.3, -1.1, 0.7])
    f = np.zeros(3 * n2)
    f[1::3] = lm.p2_xt @ c
    fv = lm.X @ c                                           # (T,4) vertex values
    exact = float((_vol(lm.X) / 20.0 * ((fv ** 2).sum(1) + fv.sum(1) ** 2)).sum())
    assert abs(f @ VM @ f - exact) < 1e-15
    d9 = Discretisation(lm, False, np.full(lm.n_p1, 9.0), 0.0, {}, build=("VM",))
    assert abs(d9.VM - 3.0 * VM).max() < 1e-15


def test_surface_scaling_of_vector_mass():
    """VM(a) - VM(1) = (a - 1) VM restricted to D_eta: summed over one component of the constant field
    it is (a - 1) |D_eta| (unblended shell, eta = 1)."""
    m = icoshell(3, 2)
    lm = build_level(m.verts, m.tets, m.vtag, 1)
    d1 = Discretisation(lm, False, None, 0.0, {}, build=("VM",), surf_a=1.0)
    d3 = Discretisation(lm, False, None, 0.0, {}, build=("VM",), surf_a=3.0)
    e = np.zeros(3 * lm.n_p2)
    e[0::3] = 1.0
    vD, _ = _surface_volume(lm)
    assert abs(e @ (d3.VM - d1.VM) @ e - 2.0 * vD) < 1e-13


@pytest.fixture(scope="module")
def shell_case():
    m = icoshell(3, 2)
    discs, v0 = {}, {}
    for L in (0, 1):
        lm = build_level(m.verts, m.tets, m.vtag, L)
        eta = 1.0 + 0.5 * (uniform_from_keys(lm.p1_keys, 5, 0) + 1.0)
        discs[L] = Discretisation(lm, True, eta, 0.0, {2: BC_DIRICHLET, 1: 2},
                                  build=("A", "B", "C", "M", "K", "VM"))
        v0[L] = uniform_vec(lm.p2_keys, 6)
    return discs, Hierarchy(discs, v0, pre=3, post=3, degree=3)


def test_wbfbt_symmetry_and_viscosity_scaling(shell_case):
    """With a_l = a_r the w-BFBT operator is symmetric on mean-zero vectors; eta -> 4 eta (all pieces
    rebuilt) multiplies S_w^-1 by 4 (K^-1 ~ eta^1/2, VM^-1 ~ eta^-1/2, A ~ eta)."""
    discs, H = shell_case
    d = discs[1]
    S = StokesOracle(H, d, d.M, schur="wbfbt", wbfbt_ops=(d.K, d.K, d.VM, d.VM))
    t = uniform_from_keys(d.lm.p1_keys, 3, 0)
    s = uniform_from_keys(d.lm.p1_keys, 4, 0)
    t, s = t - t.mean(), s - s.mean()
    zt, zs = S.wbfbt(t), S.wbfbt(s)
    assert abs(s @ zt - t @ zs) <= 1e-10 * abs(s @ zt)
    assert t @ zt > 0
    d4 = Discretisation(d.lm, True, 4.0 * d.eta_p1, 0.0, {2: BC_DIRICHLET, 1: 2}, build=("A", "B", "C", "M", "K", "VM"))
    S4 = StokesOracle(H, d4, d4.M, schur="wbfbt", wbfbt_ops=(d4.K, d4.K, d4.VM, d4.VM))
    S4.A = d4.Ac()
    assert np.linalg.norm(S4.wbfbt(t) - 4.0 * zt) <= 1e-10 * np.linalg.norm(zt)
    # K solve: mean zero, exact
    y = neumann_solve(d.K, t)
    assert abs(y.sum()) < 1e-12 * np.abs(y).max() and np.linalg.norm(d.K @ y - t) < 1e-11 * np.linalg.norm(t)


@pytest.mark.parametrize("a", [(1.0, 1.0), (2.0, 0.5)])
def test_fgmres_wbfbt_recovers_a_manufactured_solution(shell_case, a):
    """Blended shell L1, variable eta: FGMRES + symmetric Uzawa with S_w (a_l, a_r) reaches the
    manufactured solution of the projected system."""
    discs, H = shell_case
    d = discs[1]
    lm = d.lm
    if a == (1.0, 1.0):
        ops = (d.K, d.K, d.VM, d.VM)
    else:
        dl = Discretisation(lm, True, d.eta_p1, 0.0, {2: BC_DIRICHLET, 1: 2}, build=("K", "VM"), surf_a=a[0])
        dr = Discretisation(lm, True, d.eta_p1, 0.0, {2: BC_DIRICHLET, 1: 2}, build=("K", "VM"), surf_a=a[1])
        ops = (dl.K, dr.K, dl.VM, dr.VM)
    S = StokesOracle(H, d, d.M, tol_A=1e-2, schur="wbfbt", wbfbt_ops=ops)
    n2 = 3 * lm.n_p2
    xs = np.concatenate([d.project(uniform_vec(lm.p2_keys, 2)), uniform_from_keys(lm.p1_keys, 3, 0)])
    xs[n2:] -= xs[n2:].mean()
    rhs = S.op(xs)
    x, it, rel = S.solve(rhs, tol=1e-9, restart=60, max_iters=200)
    assert rel <= 1e-9
    assert np.linalg.norm(x[:n2] - xs[:n2]) <= 1e-7 * np.linalg.norm(xs[:n2])


def _k_levels(a, levels=(1, 2)):
    from workload import viscosity
    from oracle.operators import node_coords
    m = icoshell(3, 2)
    out = {}
    for L in levels:
        lm = build_level(m.verts, m.tets, m.vtag, L)
        eta = viscosity(node_coords(lm, "P1", True), lm.p1_keys, 1e4, 10.0)
        out[L] = (lm, Discretisation(lm, True, eta, 0.0, {2: BC_DIRICHLET, 1: 2}, build=("K", "VM"), surf_a=a))
    return out


@pytest.mark.parametrize("a", [1.0, 3.0])
def test_kmg_cg_converges_to_the_direct_neumann_solution(a):
    """oracle.kmg (reading R23) pinned to the direct mean-zero solve: the GMG-preconditioned CG driven to
    1e-13 reproduces neumann_solve to 1e-10, in few (level-robust multigrid) iterations; the power
    iteration's lambda_hat lies within 5% below the dense lambda_max(D^-1 K) of the finest level."""
    from oracle.kmg import KHierarchy, K_POWER_SEED, mean0
    lv = _k_levels(a)
    KH = KHierarchy({L: d.K for L, (lm, d) in lv.items()}, {L: lm for L, (lm, d) in lv.items()},
                    {L: uniform_from_keys(lm.p1_keys, K_POWER_SEED, 0) for L, (lm, d) in lv.items()})
    lm, d = lv[2]
    t = mean0(uniform_from_keys(lm.p1_keys, 3, 0))
    y, it, rel = KH.solve(t, 1e-13, 0.0, 100)
    y_d = neumann_solve(d.K, t)
    assert rel <= 1e-13 and it <= 30
    assert np.linalg.norm(y - y_d) <= 1e-10 * np.linalg.norm(y_d)
    Kd = d.K.toarray()
    dinv = 1.0 / np.diag(Kd)
    lmax = float(np.max(np.real(np.linalg.eigvals(dinv[:, None] * Kd))))
    assert 0.95 * lmax <= KH.lam[2] <= lmax * (1 + 1e-12)


def test_vmass_cg_converges_to_the_direct_constrained_solution():
    """oracle.kmg.vmass_solve (reading R24) pinned to the direct constrained solve at tight tolerance."""
    from oracle.kmg import vmass_solve
    from oracle.stokes import constrained_solve
    lm, d = _k_levels(2.0, levels=(1,))[1]
    from oracle.refine import node_bc
    from oracle.operators import constraint_matrix
    Pm = constraint_matrix(lm.p2_xt, node_bc(lm.p2_keys, lm.macro_tets, lm.macro_vtag, {2: BC_DIRICHLET, 1: 2}))
    v = Pm @ uniform_vec(lm.p2_keys, 5)
    x, it, rel = vmass_solve(d.VM, Pm, v, 1e-14, 2000)
    x_d = constrained_solve(d.VM, Pm, v)
    assert rel <= 1e-14
    assert np.linalg.norm(x - x_d) <= 1e-9 * np.linalg.norm(x_d)
