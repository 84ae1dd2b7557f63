"""ORACLE (test infrastructure only): P2 transfers, Chebyshev smoother, power iteration,
coarse Jacobi-PCG and the GMG V-cycle for the A block.

Paper: P:441 (CG preconditioned by a GMG V-cycle; m_A pre/post Chebyshev steps of
degree deg_A preconditioned by the inverse diagonal of A; diag(A) without P_v),
P:443 (coarse-grid CG), P:445-450 (fig:ASolverStructure, the V-cycle)
(projections applied in prolongation, restriction and smoother).

Readings: R12 Chebyshev recurrence and interval [b/10, b], b = 1.1 lambda_hat;
R13 power iteration (20 its on D^-1 A from a seeded vector); R14 prolongation =
nodal P2 interpolation, restriction = its transpose, each followed by P_v M;
R15 coarse solve = exactly 50 Jacobi-PCG iterations from x = 0 (BASELINE config 3,
replacing the paper's AMG-CG).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from . import fe
from .refine import LevelMesh, keys_from_weights


def lookup_keys(table: np.ndarray, queries: np.ndarray) -> np.ndarray:
    """Row index in `table` of every row of `queries` (all must exist)."""
    n = table.shape[0]
    uniq, inv = np.unique(np.vstack([table, queries]), axis=0, return_inverse=True)
    inv = inv.ravel()
    pos = np.full(uniq.shape[0], -1, dtype=np.int64)
    pos[inv[:n]] = np.arange(n)
    out = pos[inv[n:]]
    if np.any(out < 0):
        raise KeyError("query key not in table")
    return out


def p2_prolongation(coarse: LevelMesh, fine: LevelMesh) -> sp.csr_matrix:
    """Scalar P2 prolongation P[f, c] = phi_c^coarse(x_f): nodal interpolation of the coarse
    P2 function at the fine P2 nodes (the exact embedding of nested P2 spaces)."""
    nc = 2 ** coarse.level
    beta = np.array([(a, b, c, 4 - a - b - c) for a in range(5) for b in range(5 - a)
                     for c in range(5 - a - b)], dtype=np.int64)       # (35,4) over coarse-tet vertices
    xi = beta[:, 1:].astype(np.float64) / 4.0                          # reference coords
    phi = fe.p2_basis(xi)                                             # (35,10)
    T = coarse.n_tets
    # fine-node macro weights = sum_v beta_v W_v  at res 4 nc = 2 n_fine
    w = np.einsum("pv,tvm->tpm", beta, coarse.tet_w)                  # (T,35,4)
    mids = coarse.macro_tets[coarse.tet_macro]
    keys = keys_from_weights(w.reshape(-1, 4), 4 * nc, np.repeat(mids, 35, axis=0))
    frow = lookup_keys(fine.p2_keys, keys).reshape(T, 35)
    rows = np.broadcast_to(frow[:, :, None], (T, 35, 10)).ravel()
    cols = np.broadcast_to(coarse.tet_p2[:, None, :], (T, 35, 10)).ravel()
    vals = np.broadcast_to(phi[None], (T, 35, 10)).ravel()
    keep = np.abs(vals) > 0
    rc = np.stack([rows[keep], cols[keep]], axis=1)
    rc_u, first = np.unique(rc, axis=0, return_index=True)
    P = sp.coo_matrix((vals[keep][first], (rc_u[:, 0], rc_u[:, 1])),
                      shape=(fine.n_p2, coarse.n_p2)).tocsr()
    return P


def p1_prolongation(coarse: LevelMesh, fine: LevelMesh) -> sp.csr_matrix:
    """Scalar P1 prolongation P[f, c] = lam_c^coarse(x_f): nodal (linear) interpolation of the coarse
    P1 function at the fine P1 nodes (nested P1 spaces; the K_{1/sqrt(eta)} multigrid of P:470)."""
    nc = 2 ** coarse.level
    beta = np.array([(a, b, c, 2 - a - b - c) for a in range(3) for b in range(3 - a)
                     for c in range(3 - a - b)], dtype=np.int64)       # (10,4) over coarse-tet vertices
    lam = beta.astype(np.float64) / 2.0                                # barycentric coordinates
    T = coarse.n_tets
    w = np.einsum("pv,tvm->tpm", beta, coarse.tet_w)                  # fine-node weights at res 2 nc
    mids = coarse.macro_tets[coarse.tet_macro]
    keys = keys_from_weights(w.reshape(-1, 4), 2 * nc, np.repeat(mids, 10, axis=0))
    frow = lookup_keys(fine.p1_keys, keys).reshape(T, 10)
    rows = np.broadcast_to(frow[:, :, None], (T, 10, 4)).ravel()
    cols = np.broadcast_to(coarse.tet_p1[:, None, :], (T, 10, 4)).ravel()
    vals = np.broadcast_to(lam[None], (T, 10, 4)).ravel()
    keep = vals > 0
    rc = np.stack([rows[keep], cols[keep]], axis=1)
    rc_u, first = np.unique(rc, axis=0, return_index=True)
    return sp.coo_matrix((vals[keep][first], (rc_u[:, 0], rc_u[:, 1])),
                         shape=(fine.n_p1, coarse.n_p1)).tocsr()


def vec_prolongation(Ps: sp.csr_matrix) -> sp.csr_matrix:
    """Componentwise (node-major, xyz interleaved) version of the scalar prolongation."""
    return sp.kron(Ps, sp.identity(3), format="csr")


def chebyshev(Ac, dinv, Pm, f, x, degree, lam_hi):
    """Degree-`degree` Chebyshev iteration on D^-1 A over [b/10, b] (b = lam_hi).
    theta=(b+a)/2, delta=(b-a)/2, sigma=theta/delta, rho=1/sigma; r=f-Ax; d=PM D^-1 r/theta;
    for k=1..deg: x+=d; if k<deg: r-=A d; rho'=1/(2 sigma-rho); d=rho' rho d+(2 rho'/delta) PM D^-1 r."""
    b = lam_hi
    a = b / 10.0
    theta, delta = 0.5 * (b + a), 0.5 * (b - a)
    sigma = theta / delta
    rho = 1.0 / sigma
    x = x.copy()
    r = f - Ac @ x
    d = Pm @ (dinv * r) / theta
    for k in range(1, degree + 1):
        x = x + d
        if k < degree:
            r = r - Ac @ d
            rho_n = 1.0 / (2.0 * sigma - rho)
            d = rho_n * rho * d + (2.0 * rho_n / delta) * (Pm @ (dinv * r))
            rho = rho_n
    return x


def power_iteration(Ac, dinv, Pm, v0, iters=20):
    """w = PM D^-1 A v ; lambda = |w|_2 ; v = w / lambda  (iters times) -> last lambda."""
    v = Pm @ v0
    lam = 0.0
    for _ in range(iters):
        w = Pm @ (dinv * (Ac @ v))
        lam = float(np.linalg.norm(w))
        if lam == 0.0:
            raise ZeroDivisionError("power iteration on a zero operator")
        v = w / lam
    return lam


def pcg(Ac, dinv, Pm, f, iters=50, tol=0.0, count=False):
    """Jacobi-preconditioned CG from x = 0: exactly `iters` iterations (stop early only if r.z <= 1e-300), or,
    with tol > 0, until sqrt(r.z) <= tol sqrt(r0.z0), at most `iters` -- the coarse solve "up to a relative
    tolerance tol_coarse" of P:443 (Table 1: 1e-2; R29).  count=True also returns the iterations."""
    x = np.zeros_like(f)
    r = f.copy()
    z = Pm @ (dinv * r)
    p = z.copy()
    rz = float(r @ z)
    rz0 = rz
    it = 0
    for it in range(iters + 1):
        if it == iters or rz <= 1e-300 or (tol > 0 and rz <= tol * tol * rz0):
            break
        q = Ac @ p
        alpha = rz / float(p @ q)
        x = x + alpha * p
        r = r - alpha * q
        z = Pm @ (dinv * r)
        rz_new = float(r @ z)
        beta = rz_new / rz
        p = z + beta * p
        rz = rz_new
    return (x, it) if count else x


class Hierarchy:
    """Per-level constrained operators Ac, D^-1, P_v M, lambda_hat, and transfers between levels."""

    def __init__(self, discs: dict, power_v0: dict, pre=3, post=3, degree=3, power_iters=20,
                 coarse_iters=50, hi_factor=1.1, coarse_tol=0.0):
        self.coarse_tol = coarse_tol
        self.levels = sorted(discs)
        self.lmin, self.lmax = self.levels[0], self.levels[-1]
        self.pre, self.post, self.degree, self.coarse_iters = pre, post, degree, coarse_iters
        self.Ac, self.dinv, self.Pm, self.lam = {}, {}, {}, {}
        for l in self.levels:
            d = discs[l]
            self.Ac[l] = d.Ac()
            self.dinv[l] = 1.0 / d.diagA()
            self.Pm[l] = d.Pm
            if l > self.lmin:
                self.lam[l] = power_iteration(self.Ac[l], self.dinv[l], self.Pm[l], power_v0[l], power_iters)
        self.P = {}
        for l in self.levels[1:]:
            Pv = vec_prolongation(p2_prolongation(discs[l - 1].lm, discs[l].lm))
            self.P[l] = Pv
        self.hi_factor = hi_factor

    def prolong(self, l, xc):
        """fine += P_v M P xc."""
        return self.Pm[l] @ (self.P[l] @ xc)

    def restrict(self, l, rf):
        """coarse = P_v M P^T rf."""
        return self.Pm[l - 1] @ (self.P[l].T @ rf)

    def vcycle(self, f, l=None):
        """fig:ASolverStructure from x = 0."""
        l = self.lmax if l is None else l
        if l == self.lmin:
            return pcg(self.Ac[l], self.dinv[l], self.Pm[l], f, self.coarse_iters, self.coarse_tol)
        b = self.hi_factor * self.lam[l]
        x = np.zeros_like(f)
        for _ in range(self.pre):
            x = chebyshev(self.Ac[l], self.dinv[l], self.Pm[l], f, x, self.degree, b)
        r = f - self.Ac[l] @ x
        xc = self.vcycle(self.restrict(l, r), l - 1)
        x = x + self.prolong(l, xc)
        for _ in range(self.post):
            x = chebyshev(self.Ac[l], self.dinv[l], self.Pm[l], f, x, self.degree, b)
        return x


def ablock_cg(H: Hierarchy, f, tol=1e-2, max_iters=100):
    """A-block solver: CG preconditioned by one V-cycle of H per iteration, from x = 0,
    until |r|_2 <= tol |f|_2 or max_iters -> (x, iterations, relative residual)."""
    A = H.Ac[H.lmax]
    x = np.zeros_like(f)
    r = f.copy()
    r0 = float(np.linalg.norm(r))
    if r0 == 0.0:
        return x, 0, 0.0
    z = H.vcycle(r)
    p = z.copy()
    rz = float(r @ z)
    it, rel = 0, 1.0
    while it < max_iters:
        it += 1
        q = A @ p
        pq = float(p @ q)
        alpha = rz / pq if pq != 0.0 else 0.0
        x = x + alpha * p
        r = r - alpha * q
        rel = float(np.linalg.norm(r)) / r0
        if rel <= tol:
            break
        z = H.vcycle(r)
        rz_new = float(r @ z)
        beta = rz_new / rz if rz != 0.0 else 0.0
        p = z + beta * p
        rz = rz_new
    return x, it, rel

