"""ORACLE (test infrastructure only): the discrete temperature (advection-diffusion) operator of
eq:WeakTemp and its solve, SURVEY §8(f) NEXT-4 without the MMOC advection step.

Left-hand side of eq:WeakTemp for a trial T and test w (both P2 scalar on the blended mesh):
    L(T, w) = s int T w + tau [ int (u . grad T) w + int kappa grad T . grad(w / rho)
                                - int beta T (u . g) w ]
with s = s^{n+1}, tau = tau^{n+1}, kappa = k / (Pe C_p), beta = Di alpha / C_p (constants, reading
R26), u = u_*^{n+1} (P2 vector), g = -x/|x| (unit gravity), rho = exp(gamma (1 - |x|)) so that
grad ln rho = -gamma x/|x| (reading R9), hence grad(w / rho) = (grad w + gamma w x/|x|) / rho.
The preconditioner of the FGMRES solve is CG on "the symmetric, positive semidefinite mass and
diffusion part": P(T, w) = s int T w + tau int (kappa / rho) grad T . grad w (reading R27).
Dirichlet values on the surface and the CMB: rows/columns of boundary nodes are replaced by
the identity (T = T_D there).  Element integrals use the Q4 rule of every other operator (R6).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from . import fe
from .operators import quad_geometry, macro_blend, _coo
from .refine import LevelMesh, node_bc, BC_DIRICHLET


def element_T(W, grads, xq, u_q, s, tau, kappa, beta, gamma):
    """(T,10,10) element matrices of L, row a = test function, column b = trial function."""
    xi, _ = fe.q4_rule()
    phi = fe.p2_basis(xi)                                      # (Q,10)
    r = np.linalg.norm(xq, axis=2)                             # (T,Q)
    xh = xq / r[:, :, None]
    rho = np.exp(gamma * (1.0 - r))
    adv = np.einsum("tqd,tqbd->tqb", u_q, grads)               # u . grad phi_b
    ug = -np.einsum("tqd,tqd->tq", u_q, xh)                    # u . g
    gw = grads + gamma * phi[None, :, :, None] * xh[:, :, None, :]   # grad w + gamma w x^  (test a)
    E = s * np.einsum("tq,qa,qb->tab", W, phi, phi)
    E += tau * np.einsum("tq,qa,tqb->tab", W, phi, adv)
    E += tau * np.einsum("tq,tqad,tqbd->tab", W * kappa / rho, gw, grads)
    E -= tau * beta * np.einsum("tq,qa,qb->tab", W * ug, phi, phi)
    return E


def element_Tsym(W, grads, xq, s, tau, kappa, gamma):
    """(T,10,10): s int phi_a phi_b + tau int (kappa / rho) grad phi_a . grad phi_b."""
    xi, _ = fe.q4_rule()
    phi = fe.p2_basis(xi)
    rho = np.exp(gamma * (1.0 - np.linalg.norm(xq, axis=2)))
    return (s * np.einsum("tq,qa,qb->tab", W, phi, phi)
            + tau * np.einsum("tq,tqad,tqbd->tab", W * kappa / rho, grads, grads))


def assemble_temperature(lm: LevelMesh, blended: bool, u_vec, s=1.5, tau=1e-3, kappa=1.0, beta=0.5,
                         gamma=0.0, chunk=20000):
    """(L, P) as CSR over the canonical P2 nodes; u_vec: P2 vector (node-major xyz), canonical order."""
    xi, _ = fe.q4_rule()
    phi = fe.p2_basis(xi)
    bp = macro_blend(lm) if blended else None
    u3 = np.asarray(u_vec, dtype=np.float64).reshape(-1, 3)
    Lm = Pm = None
    for s0 in range(0, lm.n_tets, chunk):
        tets = np.arange(s0, min(s0 + chunk, lm.n_tets))
        W, grads, xq = quad_geometry(lm, tets, blended, bp)
        nd = lm.tet_p2[tets]
        u_q = np.einsum("qa,tad->tqd", phi, u3[nd])
        A = _coo(element_T(W, grads, xq, u_q, s, tau, kappa, beta, gamma), nd, nd, lm.n_p2, lm.n_p2)
        B = _coo(element_Tsym(W, grads, xq, s, tau, kappa, gamma), nd, nd, lm.n_p2, lm.n_p2)
        Lm = A if Lm is None else Lm + A
        Pm = B if Pm is None else Pm + B
    return Lm.tocsr(), Pm.tocsr()


def boundary_mask(lm: LevelMesh) -> np.ndarray:
    """True at P2 nodes on the surface or the CMB (every boundary face)."""
    return node_bc(lm.p2_keys, lm.macro_tets, lm.macro_vtag, {"all": BC_DIRICHLET}) != 0


def constrain(Lm, mask):
    """Identity rows and columns at Dirichlet nodes, the rest unchanged: D L D + (I - D)."""
    D = sp.diags((~mask).astype(np.float64))
    return (D @ Lm @ D + sp.diags(mask.astype(np.float64))).tocsr()


def solve_temperature(Lm, b, T_D, mask):
    """T with T = T_D on the boundary and (L T)_i = b_i at interior nodes (direct sparse solve):
    interior unknowns from D L D x = D (b - L T_D)."""
    Td = np.where(mask, T_D, 0.0)
    rhs = np.where(mask, 0.0, b - Lm @ Td)
    x = spla.spsolve(constrain(Lm, mask).tocsc(), rhs)
    return np.where(mask, T_D, x)
