"""ORACLE (test infrastructure only): the particle-based modified method of characteristics (MMOC) of
P:500-512: "tracks particles backwards in time along a linear interpolation
between u^{n+1} and u^n using the classical Runge-Kutta method and evaluates T^n at the calculated
positions".

For every P2 node x (blended position) with u(y, theta) = (1 - theta) u^{n+1}(y) + theta u^n(y) at
time t^{n+1} - theta tau:
    k1 = u(x, 0), k2 = u(x - tau/2 k1, 1/2), k3 = u(x - tau/2 k2, 1/2), k4 = u(x - tau k3, 1),
    X = x - tau/6 (k1 + 2 k2 + 2 k3 + k4),   T_hat(x) = T^n(X).
Fields are evaluated at a physical point y by locating it: inverse blending per macro (the blending
keeps directions, B(x) = c x (n.x)/|x|, so x = s y/|y| with s = |y| / (c n.y/|y|)), the macro's
barycentric coordinates, then the micro tet among that macro's micro tets (brute force), and the P2
basis there.  Points outside the shell are moved radially onto it (reading R28).  Plain and slow.
"""
from __future__ import annotations

import numpy as np

from . import fe
from .operators import macro_blend, node_coords
from .refine import LevelMesh

TOL = 1e-12


class Locator:
    def __init__(self, lm: LevelMesh, blended: bool):
        self.lm, self.blended = lm, blended
        self.bp = macro_blend(lm) if blended else None
        mv = lm.macro_verts[lm.macro_tets]                    # (M,4,3)
        self.X0 = mv[:, 0]
        self.Jinv = np.linalg.inv(np.stack([mv[:, 1] - mv[:, 0], mv[:, 2] - mv[:, 0], mv[:, 3] - mv[:, 0]], axis=2))
        r = np.linalg.norm(lm.macro_verts, axis=1)
        self.r_min, self.r_max = r.min(), r.max()
        self.tets_of = [np.nonzero(lm.tet_macro == m)[0] for m in range(len(lm.macro_tets))]
        X = lm.X
        self.tX0 = X[:, 0]
        self.tJinv = np.linalg.inv(np.stack([X[:, 1] - X[:, 0], X[:, 2] - X[:, 0], X[:, 3] - X[:, 0]], axis=2))

    def clamp(self, y):
        r = np.linalg.norm(y)
        if self.blended and r > self.r_max:
            return y * (self.r_max / r)
        if self.blended and r < self.r_min:
            return y * (self.r_min / r)
        return y

    def locate(self, y):
        """(micro tet index, its barycentric coordinates (4,)) of the physical point y: the first macro
        (by id) whose inverse-blended point has barycentric coordinates in [-TOL, 1 + TOL], then the
        micro tet of that macro containing it (largest minimum barycentric coordinate)."""
        if self.blended:
            nh, c = self.bp
            ry = np.linalg.norm(y)
            d = y / ry
            den = c * (nh @ d)                                  # (M,)
            with np.errstate(divide="ignore", invalid="ignore"):
                X = (ry / den)[:, None] * d[None, :]
        else:
            den = np.ones(len(self.X0))
            X = np.broadcast_to(y, (len(self.X0), 3))
        lam = np.einsum("mij,mj->mi", self.Jinv, X - self.X0)
        inside = (den > 0) & (lam.min(axis=1) >= -TOL) & (lam.sum(axis=1) <= 1 + TOL)
        for m in np.nonzero(inside)[0]:
            x = X[m]
            ts = self.tets_of[m]
            mu = np.einsum("tij,tj->ti", self.tJinv[ts], x - self.tX0[ts])
            mu4 = np.concatenate([1.0 - mu.sum(1, keepdims=True), mu], axis=1)
            k = int(np.argmax(mu4.min(axis=1)))
            if mu4[k].min() >= -1e-10:
                return ts[k], mu4[k]
        raise ValueError(f"point {y} not in the mesh")

    def evaluate(self, field, y):
        """P2 field (n_p2,) or (n_p2, 3) at the physical point y."""
        t, lam = self.locate(y)
        phi = fe.p2_basis(lam[None, 1:])[0]                   # (10,)
        return phi @ np.asarray(field)[self.lm.tet_p2[t]]


def mmoc(lm: LevelMesh, blended: bool, T, u_new, u_old, tau, nodes=None):
    """T_hat at the P2 nodes `nodes` (default: all, canonical order); u_* as (n_p2, 3) or flat."""
    loc = Locator(lm, blended)
    xs = node_coords(lm, "P2", blended)
    un, uo = np.asarray(u_new).reshape(-1, 3), np.asarray(u_old).reshape(-1, 3)
    nodes = np.arange(lm.n_p2) if nodes is None else np.asarray(nodes)
    out = np.empty(len(nodes))

    def vel(y, th):
        y = loc.clamp(y)
        return (1.0 - th) * loc.evaluate(un, y) + th * loc.evaluate(uo, y)

    for i, x in enumerate(xs[nodes]):
        k1 = vel(x, 0.0)
        k2 = vel(x - 0.5 * tau * k1, 0.5)
        k3 = vel(x - 0.5 * tau * k2, 0.5)
        k4 = vel(x - tau * k3, 1.0)
        X = loc.clamp(x - tau / 6.0 * (k1 + 2.0 * k2 + 2.0 * k3 + k4))
        out[i] = loc.evaluate(T, X)
    return out
