"""ORACLE (test infrastructure only): the iterative inner solves of the weighted BFBT Schur approximation
(eq:schurWBFBT with the a_l / a_r surface scaling), step by step as the method specifies them:

  K_{1/sqrt(eta_a)}^-1 : "an inverse viscosity scaled Poisson problem with Neumann boundary conditions ...
      solved ... using a CG solver preconditioned by a GMG approach".  Reading R23:
      P1 hierarchy on the A hierarchy's levels with the A smoother settings (m pre/post Chebyshev sweeps
      of degree deg on D^-1 K over [b/10, b], b = 1.1 lambda_hat, lambda_hat from `power_iters` power
      iterations from a start vector keyed by node identity, seed 7), linear
      interpolation and its transpose, coarsest level a fixed number of Jacobi-PCG iterations on the
      mean-zero-projected rhs; the outer CG works on arithmetic-mean-zero vectors and stops at the
      relative OR absolute tolerance (Table 1 tol_wBFBT, "whichever applies first").
  M_{sqrt(eta_a)}^-1 : "solved ... using a CG solver".  Reading R24: Jacobi-preconditioned CG on
      the constrained velocity space to the relative tolerance tol_VM (Table 1: 1e-4).

No blocking, no fusion: plain sparse matrix-vector products with the assembled operators of
oracle/operators.py, the P1 prolongation of oracle/multigrid.py, numpy dot products in canonical order.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .multigrid import chebyshev, power_iteration, p1_prolongation

K_POWER_SEED = 7    # start vector of the K power iterations (keyed by node identity)


def mean0(v):
    return v - v.mean()


def cg(op, prec, proj, rhs, tol, tol_abs, max_iters):
    """CG from x = 0 with preconditioner `prec` and optional projection `proj` of the residual, the
    preconditioned residual and the result; stops when |r| <= tol |r0| or |r| <= tol_abs
    -> (x, iterations, relative residual)."""
    x = np.zeros_like(rhs)
    r = rhs.copy()
    if proj is not None:
        r = proj(r)
    r0 = float(np.linalg.norm(r))
    it, rel = 0, (1.0 if r0 > 0 else 0.0)
    if r0 > 0 and r0 > tol_abs:
        z = prec(r)
        if proj is not None:
            z = proj(z)
        p = z.copy()
        rz = float(r @ z)
        while it < max_iters:
            it += 1
            q = op(p)
            pq = float(p @ q)
            alpha = rz / pq if pq != 0.0 else 0.0
            x = x + alpha * p
            r = r - alpha * q
            rn = float(np.linalg.norm(r))
            rel = rn / r0
            if rel <= tol or rn <= tol_abs:
                break
            z = prec(r)
            if proj is not None:
                z = proj(z)
            rz_new = float(r @ z)
            beta = rz_new / rz if rz != 0.0 else 0.0
            p = z + beta * p
            rz = rz_new
    if proj is not None:
        x = proj(x)
    return x, it, rel


class KHierarchy:
    """GMG-preconditioned CG for K_{1/sqrt(eta_a)} (Neumann, constants in the kernel), reading R23.
    Ks[l]: assembled K on level l (oracle.operators, build "K"); lms[l]: the LevelMesh of level l;
    v0[l]: power-iteration start vector (canonical P1 order) for l > l_min."""

    def __init__(self, Ks: dict, lms: dict, v0: dict, pre=3, post=3, degree=3, power_iters=20, coarse_iters=50,
                 hi_factor=1.1):
        self.levels = sorted(Ks)
        self.lmin, self.lmax = self.levels[0], self.levels[-1]
        self.K = Ks
        self.pre, self.post, self.degree, self.coarse_iters, self.hi = pre, post, degree, coarse_iters, hi_factor
        self.dinv = {l: 1.0 / Ks[l].diagonal() for l in self.levels}
        self.I = {l: sp.identity(Ks[l].shape[0], format="csr") for l in self.levels}
        self.lam = {l: power_iteration(Ks[l], self.dinv[l], self.I[l], v0[l], power_iters)
                    for l in self.levels if l > self.lmin}
        self.P = {l: p1_prolongation(lms[l - 1], lms[l]) for l in self.levels[1:]}

    def coarse(self, f):
        """Exactly coarse_iters Jacobi-PCG iterations from 0 on the mean-zero rhs (zero-rhs guard 1e-300)."""
        l = self.lmin
        K, dinv = self.K[l], self.dinv[l]
        x = np.zeros_like(f)
        r = mean0(f)
        z = dinv * r
        p = z.copy()
        rz = float(r @ z)
        for _ in range(self.coarse_iters):
            q = K @ p
            pq = float(p @ q)
            alpha = rz / pq if (rz > 1e-300 and pq != 0.0) else 0.0
            x = x + alpha * p
            r = r - alpha * q
            z = dinv * r
            rz_new = float(r @ z)
            beta = rz_new / rz if rz > 1e-300 else 0.0
            p = z + beta * p
            rz = rz_new
        return x

    def cycle(self, f, l=None):
        """One V-cycle (fig:ASolverStructure's structure on the P1 hierarchy) from x = 0."""
        l = self.lmax if l is None else l
        if l == self.lmin:
            return self.coarse(f)
        K, dinv, I = self.K[l], self.dinv[l], self.I[l]
        b = self.hi * self.lam[l]
        x = np.zeros_like(f)
        for _ in range(self.pre):
            x = chebyshev(K, dinv, I, f, x, self.degree, b)
        r = f - K @ x
        x = x + self.P[l] @ self.cycle(self.P[l].T @ r, l - 1)
        for _ in range(self.post):
            x = chebyshev(K, dinv, I, f, x, self.degree, b)
        return x

    def solve(self, rhs, tol, tol_abs, max_iters):
        """CG on the mean-zero space preconditioned by one V-cycle -> (x, iterations, relative residual)."""
        K = self.K[self.lmax]
        return cg(lambda v: K @ v, self.cycle, mean0, rhs, tol, tol_abs, max_iters)


def vmass_solve(VM, Pm, v, tol, max_iters):
    """x = M_{sqrt(eta_a)}^-1 v on the constrained velocity space: Jacobi-preconditioned CG with the
    operator P_v M VM and the preconditioner P_v M D^-1 (reading R24) -> (x, iterations, rel. residual)."""
    dinv = 1.0 / VM.diagonal()
    return cg(lambda u: Pm @ (VM @ u), lambda r: Pm @ (dinv * r), None, v, tol, 0.0, max_iters)
