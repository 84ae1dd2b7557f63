"""ORACLE (test infrastructure only): assembled P2-P1 operators from the weak forms.

Definitions followed:
  A_ij = int 2 eta [ eps(phi_j) : eps(phi_i) - (1/dim) div phi_j div phi_i ]  (P:277-278,
         with eta on BOTH terms -- reading R1: P:278 drops eta from the div-div
         term, contradicted by tau := 2 eta eps_dot, the appendix
         and "A symmetric positive semidefinite").  The factor 2/dim of
         P:278 multiplies div.div with the eps:eps term weighted 2 -> 2 eta (1/3).
  B_ij = - int (div phi_j^u) phi_i^p
  C_ij = - int grad(ln rho) . phi_j^u phi_i^p,  grad ln rho = -gamma x/|x|
  Pull-back to the reference tet through F and the blending B:
      grad_x phi = (J_B^-1)^T (J_F^-1)^T grad_xi phi,  dx = |det J_B||det J_F| dxi
  Viscosity as a P1 function interpolated at quadrature points.
  Constraints: zero Dirichlet rows (surface) by block-row modification,
  free-slip projection P_v at CMB nodes, u <- u - (u.n) n;
  the constrained operator is (M P_v) A (P_v M).  diag(A) WITHOUT P_v.

Weighted-BFBT pieces (eq:schurWBFBT and the a_l / a_r variant):
  K_ij = int omega grad(lam_j) . grad(lam_i),  omega = 1/sqrt(eta_a)  (P1, Neumann: no constraints)
  VM_(a,c),(b,d) = delta_cd int sqrt(eta_a) phi_a phi_b                (P2 vector mass)
  eta_a = a^2 eta on D_eta (micro tets with a vertex on the surface, the outer boundary), else eta.

The element matrices are computed one quadrature point at a time from these
formulas (numpy) and summed into scipy CSR matrices (assembly = the plain
definition of the matrix-free apply).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from . import fe
from .refine import LevelMesh, node_bc, BC_DIRICHLET, BC_FREESLIP

FORM_FULL, FORM_EPS = 0, 1


def macro_blend(lm: LevelMesh):
    """(nhat, c) of every macro tet (computed from macro vertices, reading R3)."""
    return fe.shell_blend_params(lm.macro_verts[lm.macro_tets])


def quad_geometry(lm: LevelMesh, tets: np.ndarray, blended: bool, blend_params=None, p1_grads=False):
    """For the micro tets `tets`: per quadrature point the weight w_q |det J|, the physical
    P2 gradients (T,Q,10,3), the blended point x_q (T,Q,3) [, the physical P1 gradients (T,Q,4,3)]."""
    xi, w = fe.q4_rule()
    X = lm.X[tets]                                          # (T,4,3)
    JF = np.stack([X[:, 1] - X[:, 0], X[:, 2] - X[:, 0], X[:, 3] - X[:, 0]], axis=2)  # columns
    G = fe.p2_grad(xi)                                      # (Q,10,3)
    T, Q = len(tets), len(w)
    W = np.empty((T, Q))
    grads = np.empty((T, Q, 10, 3))
    g1 = np.empty((T, Q, 4, 3))
    DL = np.array([[-1.0, -1.0, -1.0], [1.0, 0.0, 0.0], [0.0, 1.0, 0.0], [0.0, 0.0, 1.0]])
    xq_all = np.empty((T, Q, 3))
    if blended:
        nhat_m, c_m = blend_params
        mac = lm.tet_macro[tets]
        nhat, c = nhat_m[mac], c_m[mac]
    for q in range(Q):
        xq = X[:, 0] + np.einsum("tij,j->ti", JF, xi[q])
        if blended:
            JB = fe.blend_jacobian(xq, nhat, c)
            J = JB @ JF
            xq_all[:, q] = fe.blend(xq, nhat, c)
        else:
            J = JF
            xq_all[:, q] = xq
        Jinv = np.linalg.inv(J)
        W[:, q] = w[q] * np.abs(np.linalg.det(J))
        # grad_x phi (row) = grad_xi phi (row) J^-1
        grads[:, q] = np.einsum("am,tmd->tad", G[q], Jinv)
        g1[:, q] = np.einsum("am,tmd->tad", DL, Jinv)
    if p1_grads:
        return W, grads, xq_all, g1
    return W, grads, xq_all


def element_A(W, grads, eta_q, form=FORM_FULL):
    """(T,30,30) element matrices, local dof = 3*a + c (a = local node, c = component)."""
    T, Q = W.shape
    Ae = np.zeros((T, 30, 30))
    eye = np.eye(3)
    for q in range(Q):
        g = grads[:, q]                                     # (T,10,3)
        # grad of vector basis (a,c): Gr[i,j] = delta_ic g_a[j]
        Gr = np.einsum("ci,taj->tacij", eye, g)             # (T,10,3,3,3)
        eps = 0.5 * (Gr + Gr.transpose(0, 1, 2, 4, 3))
        E = eps.reshape(T, 30, 9)
        K = E @ E.transpose(0, 2, 1)                        # eps(phi_i):eps(phi_j)
        if form == FORM_FULL:
            # div(phi_a e_c) = d_c phi_a = g[a, c] -> flat index 3a+c
            div = g.reshape(T, 30)
            K = K - (1.0 / 3.0) * div[:, :, None] * div[:, None, :]
        Ae += (2.0 * eta_q[:, q] * W[:, q])[:, None, None] * K
    return Ae


def element_B(W, grads):
    """(T,4,30): B_K[p,(b,d)] = - sum_q W lam_p(xi_q) d_d phi_b."""
    xi, _ = fe.q4_rule()
    lam = fe.p1_basis(xi)                                   # (Q,4)
    T, Q = W.shape
    div = grads.reshape(T, Q, 30)
    return -np.einsum("tq,qp,tqj->tpj", W, lam, div)


def element_C(W, xq, gamma):
    """(T,4,30): C_K[p,(b,d)] = - sum_q W lam_p (grad ln rho)_d phi_b,  grad ln rho = -gamma x/|x|."""
    xi, _ = fe.q4_rule()
    lam = fe.p1_basis(xi)
    phi = fe.p2_basis(xi)                                   # (Q,10)
    glr = -gamma * xq / np.linalg.norm(xq, axis=2, keepdims=True)   # (T,Q,3)
    vals = np.einsum("qb,tqd->tqbd", phi, glr).reshape(xq.shape[0], xq.shape[1], 30)
    return -np.einsum("tq,qp,tqj->tpj", W, lam, vals)


def element_M(W, eta_q):
    """(T,4,4): pressure mass weighted by 1/eta, M_K[p,r] = sum_q W/eta_q lam_p lam_r
    (Schur complement approximation M_{1/eta}, eq:schurMass)."""
    xi, _ = fe.q4_rule()
    lam = fe.p1_basis(xi)                                   # (Q,4)
    return np.einsum("tq,qp,qr->tpr", W / eta_q, lam, lam)


def element_K(W, g1, omega_q):
    """(T,4,4): K_K[p,r] = sum_q W omega_q grad lam_p . grad lam_r (P1 Laplacian weighted by omega)."""
    return np.einsum("tq,tqpd,tqrd->tpr", W * omega_q, g1, g1)


def element_VM(W, omega_q):
    """(T,30,30): vector mass weighted by omega, VM[(a,c),(b,d)] = delta_cd sum_q W omega_q phi_a phi_b."""
    xi, _ = fe.q4_rule()
    phi = fe.p2_basis(xi)                                   # (Q,10)
    Ms = np.einsum("tq,qa,qb->tab", W * omega_q, phi, phi)  # (T,10,10)
    return np.einsum("tab,cd->tacbd", Ms, np.eye(3)).reshape(W.shape[0], 30, 30)


def surface_tets(lm: LevelMesh, outer_tag=2) -> np.ndarray:
    """D_eta of P:474-478: micro tets with at least one vertex on the surface (boundary faces tagged
    `outer_tag`), by node keys (a node is on the surface iff its primitive lies in such a face)."""
    on = node_bc(lm.p1_keys, lm.macro_tets, lm.macro_vtag, {outer_tag: BC_DIRICHLET}) != 0
    return on[lm.tet_p1].any(axis=1)


def p2vec_dofs(tet_p2: np.ndarray) -> np.ndarray:
    return (3 * tet_p2[:, :, None] + np.arange(3)[None, None, :]).reshape(tet_p2.shape[0], 30)


class Discretisation:
    """Assembled operators of one level.  eta_p1: nodal P1 viscosity (canonical order) or None (=1)."""

    def __init__(self, lm: LevelMesh, blended: bool, eta_p1=None, gamma=0.0,
                 bc_by_tag=None, form=FORM_FULL, chunk=20000, build=("A", "B", "C"), T_p2=None, qeta=None,
                 surf_a=1.0):
        """T_p2 + qeta = (lnC, jump, r_jump): A uses eta at the quadrature points,
        eta_q = exp(lnC (1/2 - T_q)) (jump if |x_q| < r_jump else 1), T_q = P2 interpolant of the nodal
        temperature (the quadrature-point tier of P:451-453, R22); else the P1 eta.
        build "K" / "VM": the w-BFBT operators with eta_a = surf_a^2 eta on D_eta."""
        self.lm = lm
        self.blended = blended
        self.blend_params = macro_blend(lm) if blended else None
        self.gamma = gamma
        self.form = form
        n2, n1 = lm.n_p2, lm.n_p1
        eta_p1 = np.ones(n1) if eta_p1 is None else np.asarray(eta_p1, dtype=np.float64)
        self.eta_p1 = eta_p1
        mats = {k: [] for k in build}
        dsurf = surface_tets(lm) if ("K" in build or "VM" in build) else None
        for s in range(0, lm.n_tets, chunk):
            tets = np.arange(s, min(s + chunk, lm.n_tets))
            W, grads, xq, g1 = quad_geometry(lm, tets, blended, self.blend_params, p1_grads=True)
            vd = p2vec_dofs(lm.tet_p2[tets])
            pd = lm.tet_p1[tets]
            if "A" in build:
                xi, _ = fe.q4_rule()
                if T_p2 is not None:
                    lnC, jump, r_jump = qeta
                    Tq = np.asarray(T_p2)[lm.tet_p2[tets]] @ fe.p2_basis(xi).T     # (T,Q)
                    rq = np.linalg.norm(xq, axis=2)
                    eta_q = np.exp(lnC * (0.5 - Tq)) * np.where(rq < r_jump, jump, 1.0)
                else:
                    eta_q = eta_p1[pd] @ fe.p1_basis(xi).T   # (T,Q) P1 interpolation
                Ae = element_A(W, grads, eta_q, form)
                M = _coo(Ae, vd, vd, 3 * n2, 3 * n2)
                mats["A"].append(M)
            if "B" in build:
                Be = element_B(W, grads)
                M = _coo(Be, pd, vd, n1, 3 * n2)
                mats["B"].append(M)
            if "C" in build:
                Ce = element_C(W, xq, gamma) if gamma != 0.0 else np.zeros((len(tets), 4, 30))
                M = _coo(Ce, pd, vd, n1, 3 * n2)
                mats["C"].append(M)
            if "M" in build:
                xi, _ = fe.q4_rule()
                eta_q = eta_p1[pd] @ fe.p1_basis(xi).T
                M = _coo(element_M(W, eta_q), pd, pd, n1, n1)
                mats["M"].append(M)
            if "K" in build or "VM" in build:
                xi, _ = fe.q4_rule()
                eta_a = (eta_p1[pd] @ fe.p1_basis(xi).T) * np.where(dsurf[tets], surf_a ** 2, 1.0)[:, None]
                if "K" in build:
                    M = _coo(element_K(W, g1, 1.0 / np.sqrt(eta_a)), pd, pd, n1, n1)
                    mats["K"].append(M)
                if "VM" in build:
                    M = _coo(element_VM(W, np.sqrt(eta_a)), vd, vd, 3 * n2, 3 * n2)
                    mats["VM"].append(M)
        mats = {k: _tree_sum(v) for k, v in mats.items()}
        self.A = mats.get("A")
        self.B = mats.get("B")
        self.C = mats.get("C")
        self.M = mats.get("M")
        self.K = mats.get("K")
        self.VM = mats.get("VM")
        # constraints
        self.bc = node_bc(lm.p2_keys, lm.macro_tets, lm.macro_vtag, bc_by_tag or {})
        self.Pm = constraint_matrix(lm.p2_xt, self.bc)

    # constrained operators -------------------------------------------------
    def Ac(self):
        return (self.Pm @ self.A @ self.Pm).tocsr()

    def diagA(self):
        """diag(A) from the unprojected A; Dirichlet dofs keep their raw value."""
        return self.A.diagonal().copy()

    def project(self, u):
        """P_v M u."""
        return self.Pm @ u

    def apply_A(self, u):
        return self.Pm @ (self.A @ (self.Pm @ u))

    def apply_BT(self, p):
        return self.Pm @ (self.B.T @ p)

    def apply_Bbar(self, u):
        return (self.B + self.C) @ (self.Pm @ u)

    def free_dofs(self):
        m = np.ones(3 * self.lm.n_p2, dtype=bool)
        d = np.nonzero(self.bc == BC_DIRICHLET)[0]
        for c in range(3):
            m[3 * d + c] = False
        return m


def buoyancy_load(lm: LevelMesh, blended: bool, T_p1, chunk=20000) -> np.ndarray:
    """Config-4 buoyancy right-hand side (P:282 with rho' = -alpha (T - 1/2), alpha = 1, g = -x/|x|;
    DESIGN.md R21): b_(a,c) = sum_K sum_q w_q |det J| (T_q - 1/2) (x_q/|x_q|)_c phi_a(xi_q), T the P1
    interpolant of the nodal temperature.  Unconstrained (apply Pm for the constrained rhs)."""
    xi, _ = fe.q4_rule()
    lam = fe.p1_basis(xi)
    phi = fe.p2_basis(xi)                                   # (Q,10)
    bp = macro_blend(lm) if blended else None
    b = np.zeros(3 * lm.n_p2)
    for s in range(0, lm.n_tets, chunk):
        tets = np.arange(s, min(s + chunk, lm.n_tets))
        W, _, xq = quad_geometry(lm, tets, blended, bp)
        Tq = np.asarray(T_p1)[lm.tet_p1[tets]] @ lam.T      # (T,Q)
        dq = xq / np.linalg.norm(xq, axis=2, keepdims=True)
        Be = np.einsum("tq,qa,tqc->tac", W * (Tq - 0.5), phi, dq).reshape(len(tets), 30)
        np.add.at(b, p2vec_dofs(lm.tet_p2[tets]).ravel(), Be.ravel())
    return b


def node_coords(lm: LevelMesh, space: str, blended: bool) -> np.ndarray:
    """Physical (blended) coordinates of the canonical nodes: B(x~) evaluated with the blending
    parameters of one macro containing the node (B is C^0 across macros)."""
    xt = lm.p2_xt if space == "P2" else lm.p1_xt
    if not blended:
        return xt.copy()
    tet_nodes = lm.tet_p2 if space == "P2" else lm.tet_p1
    first_tet = np.full(xt.shape[0], -1, dtype=np.int64)
    flat = tet_nodes.ravel()
    order = np.arange(flat.size)[::-1]
    first_tet[flat[order]] = order // tet_nodes.shape[1]
    nhat, c = macro_blend(lm)
    mac = lm.tet_macro[first_tet]
    return fe.blend(xt, nhat[mac], c[mac])


def sampled_rows(lm: LevelMesh, blended, eta_p1, gamma, u, p, nodes_p2, nodes_p1, bc, form=FORM_FULL):
    """Rows of y_u = (M P_v)(A u + B^T p) at P2 nodes `nodes_p2` and of y_p = (B + C) u at P1 nodes
    `nodes_p1`, from the element matrices of only the micro tets touching them (same definitions
    as Discretisation; u must already be constraint-consistent, canonical numbering of lm)."""
    bp = macro_blend(lm) if blended else None
    want2 = np.zeros(lm.n_p2, dtype=bool)
    want2[nodes_p2] = True
    want1 = np.zeros(lm.n_p1, dtype=bool)
    want1[nodes_p1] = True
    tets = np.nonzero(want2[lm.tet_p2].any(axis=1) | want1[lm.tet_p1].any(axis=1))[0]
    yu = np.zeros(3 * lm.n_p2)
    yp = np.zeros(lm.n_p1)
    xi, _ = fe.q4_rule()
    for s in range(0, len(tets), 20000):
        tt = tets[s:s + 20000]
        W, grads, xq = quad_geometry(lm, tt, blended, bp)
        vd = p2vec_dofs(lm.tet_p2[tt])
        pd = lm.tet_p1[tt]
        eta_q = eta_p1[pd] @ fe.p1_basis(xi).T
        Ae = element_A(W, grads, eta_q, form)
        Be = element_B(W, grads)
        Ce = element_C(W, xq, gamma) if gamma != 0.0 else 0.0 * Be
        ue = u[vd]
        np.add.at(yu, vd, np.einsum("tij,tj->ti", Ae, ue) + np.einsum("tpi,tp->ti", Be, p[pd]))
        np.add.at(yp, pd, np.einsum("tpj,tj->tp", Be + Ce, ue))
    Pm = constraint_matrix(lm.p2_xt, bc)
    return Pm @ yu, yp


def _tree_sum(parts):
    """Sum of the per-chunk assembled matrices, pairwise (the entries are those of the element-by-element
    definition; only the order in which duplicate entries are added differs from a running sum)."""
    if not parts:
        return None
    while len(parts) > 1:
        parts = [parts[i] + parts[i + 1] if i + 1 < len(parts) else parts[i] for i in range(0, len(parts), 2)]
    return parts[0]


def _coo(E, rows, cols, nr, nc):
    T, a, b = E.shape
    r = np.broadcast_to(rows[:, :, None], (T, a, b))
    c = np.broadcast_to(cols[:, None, :], (T, a, b))
    return sp.coo_matrix((E.ravel(), (r.ravel(), c.ravel())), shape=(nr, nc)).tocsr()


def constraint_matrix(xt: np.ndarray, bc: np.ndarray) -> sp.csr_matrix:
    """P_v M as a sparse block-diagonal matrix: 0 on Dirichlet nodes, I - n n^T on free-slip
    nodes with n = x/|x| (the blending preserves directions), I elsewhere."""
    n = xt.shape[0]
    rows, cols, vals = [], [], []
    free = np.nonzero(bc == 0)[0]
    for c in range(3):
        rows.append(3 * free + c)
        cols.append(3 * free + c)
        vals.append(np.ones(len(free)))
    fs = np.nonzero(bc == BC_FREESLIP)[0]
    if len(fs):
        nv = xt[fs] / np.linalg.norm(xt[fs], axis=1, keepdims=True)
        for i in range(3):
            for j in range(3):
                rows.append(3 * fs + i)
                cols.append(3 * fs + j)
                vals.append((1.0 if i == j else 0.0) - nv[:, i] * nv[:, j])
    return sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                         shape=(3 * n, 3 * n)).tocsr()
