"""ORACLE (test infrastructure only): the preconditioned Stokes solve, step by step in the paper's
order.

  FGMRES (Saad 1993), right-preconditioned, restarted, modified Gram-Schmidt + Givens,
  for the projected system P K P x = P b, K = [[A, B^T], [B + C, 0]] (eq:SaddlePointStructure,
  P:284-287), P = diag(P_v M, P_p) with P_p = arithmetic mean zero.
  Preconditioner: one symmetric Uzawa step from (0, 0) (eq:SymmetricUzawaStep1) with
  B -> B + C in the pressure update:
      u_hat = sigma A^-1 r_u ; p = -omega S^-1 (r_p - (B+C) u_hat) ; u = u_hat + sigma A^-1 (r_u - A u_hat - B^T p)
  A^-1: CG preconditioned by the V-cycle to tol_A (multigrid.ablock_cg);
  S^-1: M_{1/eta}^-1 by Jacobi-preconditioned CG to tol_mass (eq:schurMass).
  schur="wbfbt": the weighted BFBT with the a_l / a_r surface scaling (eq:schurWBFBT),
      S_w^-1 = K_l^-1 (B VM_l^-1 A VM_r^-1 B^T) K_r^-1,
  K = K_{1/sqrt(eta_a)} (Neumann, mean-zero space), VM = M_{sqrt(eta_a)} (constrained velocity space),
  either solved exactly (direct factorisations: pins of the approximation itself) or -- wbfbt_iter --
  iteratively as the method prescribes (oracle/kmg.py: GMG-preconditioned CG for K to tol_wBFBT,
  Jacobi CG for VM to tol_VM, Table 1; readings R23, R24).
Readings (R17-R19): P_p applied to the rhs, to every operator output and to the
preconditioned pressure; relative residual stopping; Table 1 defaults (sigma 1, omega 0.3,
tol_A 1e-2, tol_mass 1e-10).
"""
from __future__ import annotations

import numpy as np

from .multigrid import Hierarchy, ablock_cg


def mean0(p):
    return p - p.mean()


_LU = {}


def _lu(key, refs, build):
    """Sparse LU factorisation, computed once per (matrix, system) and reused for every solve.  The
    cache holds the matrices themselves so that their ids (the key) cannot be recycled."""
    import scipy.sparse.linalg as spla
    if key not in _LU:
        _LU[key] = (refs, spla.splu(build()))
    return _LU[key][1]


def neumann_solve(K, t):
    """y with K y = t and sum(y) = 0 (t must sum to zero): the augmented system [[K, e], [e^T, 0]]."""
    import scipy.sparse as sp
    n = K.shape[0]
    e = sp.csr_matrix(np.ones((n, 1)))
    lu = _lu(("K", id(K)), (K,), lambda: sp.bmat([[K, e], [e.T, None]], format="csc"))
    return lu.solve(np.concatenate([t, [0.0]]))[:n]


def constrained_solve(VM, Pm, v):
    """x = (P VM P)^-1 P v on the constrained velocity space (regularised by I - P)."""
    import scipy.sparse as sp
    n = VM.shape[0]
    lu = _lu(("VM", id(VM), id(Pm)), (VM, Pm), lambda: (Pm @ VM @ Pm + (sp.identity(n) - Pm)).tocsc())
    return Pm @ lu.solve(Pm @ v)


def mass_cg(M, r, tol=1e-10, max_iters=500):
    """Jacobi-preconditioned CG on the SPD pressure mass from 0 to |r_k| <= tol |r|."""
    dinv = 1.0 / M.diagonal()
    z = np.zeros_like(r)
    res = r.copy()
    r0 = float(np.linalg.norm(res))
    if not r0 > 0:
        return z
    s = dinv * res
    p = s.copy()
    rz = float(res @ s)
    for _ in range(max_iters):
        q = M @ p
        pq = float(p @ q)
        alpha = rz / pq if pq != 0.0 else 0.0
        z = z + alpha * p
        res = res - alpha * q
        if float(np.linalg.norm(res)) <= tol * r0:
            break
        s = dinv * res
        rzn = float(res @ s)
        p = s + (rzn / rz) * p
        rz = rzn
    return z


class StokesOracle:
    """schur="mass": S^-1 = M_{1/eta}^-1 (eq:schurMass); schur="vbfbt": the V-cycle BFBT of eq:schurV
    (P:483-489), S_V^-1 = (B A_C^-1 B^T)^-1 (B A_C^-1 A A_C^-1 B^T) (B A_C^-1 B^T)^-1 with A_C^-1 one
    V-cycle of the cheap hierarchy HC and (B A_C^-1 B^T)^-1 by M_{1/eta}-preconditioned CG to tol_vbfbt."""

    def __init__(self, H: Hierarchy, disc, Mmass, sigma=1.0, omega=0.3, tol_A=1e-2, ablock_max_iters=200,
                 tol_mass=1e-10, mass_max_iters=500, schur="mass", HC: Hierarchy = None, tol_vbfbt=1e-1,
                 vbfbt_max_iters=100, uzawa="symmetric", wbfbt_ops=None, wbfbt_iter=None):
        """wbfbt_ops = (K_l, K_r, VM_l, VM_r) for schur="wbfbt" (direct inner solves); wbfbt_iter = dict(Kl, Kr
        (oracle.kmg.KHierarchy), VMl, VMr, tol_wbfbt, tol_wbfbt_abs, wbfbt_max_iters, tol_vmass,
        vmass_max_iters) for the iterative inner solves of the method."""
        self.wb = wbfbt_ops
        self.wbi = wbfbt_iter
        self.schur, self.HC, self.tol_vbfbt, self.vbfbt_max_iters = schur, HC, tol_vbfbt, vbfbt_max_iters
        self.uzawa = uzawa
        self.H, self.d = H, disc
        self.A = H.Ac[H.lmax]
        self.Pm = disc.Pm
        self.B, self.Bbar = disc.B, disc.B + disc.C
        self.M = Mmass
        self.sigma, self.omega, self.tol_A, self.ablock_max_iters = sigma, omega, tol_A, ablock_max_iters
        self.tol_mass, self.mass_max_iters = tol_mass, mass_max_iters
        self.n2 = self.A.shape[0]

    def op(self, x):
        """P K x."""
        u, p = x[:self.n2], x[self.n2:]
        yu = self.A @ u + self.Pm @ (self.B.T @ p)
        yp = mean0(self.Bbar @ (self.Pm @ u))
        return np.concatenate([yu, yp])

    def bacbt(self, y):
        """P_p B A_C^-1 B^T y (B, not B + C: the Schur complement of the symmetric system)."""
        return mean0(self.B @ (self.Pm @ self.HC.vcycle(self.Pm @ (self.B.T @ y))))

    def bacbt_solve(self, t):
        """CG for (B A_C^-1 B^T) y = t, preconditioned by M_{1/eta}^-1 (mass CG), to tol_vbfbt."""
        y = np.zeros_like(t)
        r = t.copy()
        r0 = float(np.linalg.norm(r))
        if not r0 > 0:
            return y
        z = mean0(mass_cg(self.M, r, self.tol_mass, self.mass_max_iters))
        p = z.copy()
        rz = float(r @ z)
        for _ in range(self.vbfbt_max_iters):
            q = self.bacbt(p)
            pq = float(p @ q)
            alpha = rz / pq if pq != 0.0 else 0.0
            y = y + alpha * p
            r = r - alpha * q
            if float(np.linalg.norm(r)) <= self.tol_vbfbt * r0:
                break
            z = mean0(mass_cg(self.M, r, self.tol_mass, self.mass_max_iters))
            rzn = float(r @ z)
            p = z + (rzn / rz) * p
            rz = rzn
        return mean0(y)

    def vbfbt(self, t):
        y1 = self.bacbt_solve(t)
        w = self.HC.vcycle(self.Pm @ (self.B.T @ y1))
        w = self.HC.vcycle(self.A @ w)
        y2 = mean0(self.B @ (self.Pm @ w))
        return self.bacbt_solve(y2)

    def wbfbt(self, t):
        """S_w^-1 t = K_l^-1 (B VM_l^-1 A VM_r^-1 B^T) K_r^-1 t."""
        if self.wbi is not None:
            from .kmg import vmass_solve
            w = self.wbi
            y = w["Kr"].solve(mean0(t), w["tol_wbfbt"], w["tol_wbfbt_abs"], w["wbfbt_max_iters"])[0]
            v = vmass_solve(w["VMr"], self.Pm, self.Pm @ (self.B.T @ y), w["tol_vmass"], w["vmass_max_iters"])[0]
            v = vmass_solve(w["VMl"], self.Pm, self.A @ v, w["tol_vmass"], w["vmass_max_iters"])[0]
            return w["Kl"].solve(mean0(self.B @ (self.Pm @ v)), w["tol_wbfbt"], w["tol_wbfbt_abs"],
                                 w["wbfbt_max_iters"])[0]
        Kl, Kr, VMl, VMr = self.wb
        y = neumann_solve(Kr, mean0(t))
        w = constrained_solve(VMr, self.Pm, self.Pm @ (self.B.T @ y))
        w = constrained_solve(VMl, self.Pm, self.A @ w)
        return neumann_solve(Kl, mean0(self.B @ (self.Pm @ w)))

    def schur_step(self, t):
        if self.schur == "vbfbt":
            sinv = self.vbfbt(t)
        elif self.schur == "wbfbt":
            sinv = self.wbfbt(t)
        else:
            sinv = mass_cg(self.M, t, self.tol_mass, self.mass_max_iters)
        return mean0(-self.omega * sinv)

    def prec(self, r):
        """One Uzawa step from (0, 0): symmetric (eq:SymmetricUzawaStep1), inexact
        (eq:InexactUzawaStep1) or adjoint inexact (eq:AdjointInexactUzawaStep1)."""
        ru, rp = r[:self.n2], r[self.n2:]
        if self.uzawa == "adjoint":
            p = self.schur_step(mean0(rp))
            u = self.sigma * ablock_cg(self.H, ru - self.Pm @ (self.B.T @ p), self.tol_A, self.ablock_max_iters)[0]
            return np.concatenate([u, p])
        uh = self.sigma * ablock_cg(self.H, ru, self.tol_A, self.ablock_max_iters)[0]
        tp = mean0(rp - self.Bbar @ (self.Pm @ uh))
        p = self.schur_step(tp)
        if self.uzawa == "inexact":
            return np.concatenate([uh, p])
        tu = ru - (self.A @ uh + self.Pm @ (self.B.T @ p))
        u = uh + self.sigma * ablock_cg(self.H, tu, self.tol_A, self.ablock_max_iters)[0]
        return np.concatenate([u, p])

    def solve(self, rhs, tol=1e-8, restart=30, max_iters=100):
        """FGMRES from x = 0 -> (x, iterations, relative residual of the projected system); the residual estimate
        of every iteration is appended to self.history."""
        self.history = []
        b = np.concatenate([self.Pm @ rhs[:self.n2], mean0(rhs[self.n2:])])
        bn = float(np.linalg.norm(b))
        x = np.zeros_like(b)
        total, rel = 0, 1.0 if bn > 0 else 0.0
        while bn > 0 and total < max_iters and rel > tol:
            r = b - self.op(x)
            beta = float(np.linalg.norm(r))
            rel = beta / bn
            if rel <= tol:
                break
            m = restart
            V, Z = [r / beta], []
            H = np.zeros((m + 1, m))
            cs, sn = np.zeros(m), np.zeros(m)
            g = np.zeros(m + 1)
            g[0] = beta
            j = 0
            while j < m and total < max_iters:
                total += 1
                Z.append(self.prec(V[j]))
                w = self.op(Z[j])
                for i in range(j + 1):                     # modified Gram-Schmidt
                    H[i, j] = float(w @ V[i])
                    w = w - H[i, j] * V[i]
                hn = float(np.linalg.norm(w))
                H[j + 1, j] = hn
                V.append(w / hn if hn > 0 else w)
                for i in range(j):                         # previous Givens rotations
                    h0, h1 = H[i, j], H[i + 1, j]
                    H[i, j], H[i + 1, j] = cs[i] * h0 + sn[i] * h1, -sn[i] * h0 + cs[i] * h1
                h0, h1 = H[j, j], H[j + 1, j]
                dd = float(np.hypot(h0, h1))
                cs[j], sn[j] = (h0 / dd, h1 / dd) if dd > 0 else (1.0, 0.0)
                H[j, j], H[j + 1, j] = dd, 0.0
                g[j + 1] = -sn[j] * g[j]
                g[j] = cs[j] * g[j]
                rel = abs(g[j + 1]) / bn
                self.history.append(rel)
                j += 1
                if rel <= tol or hn == 0.0:
                    break
            y = np.zeros(j)
            for i in range(j - 1, -1, -1):
                y[i] = (g[i] - H[i, i + 1:j] @ y[i + 1:j]) / H[i, i]
            for i in range(j):
                x = x + y[i] * Z[i]
        if bn > 0:
            rel = float(np.linalg.norm(b - self.op(x))) / bn
        return x, total, rel
