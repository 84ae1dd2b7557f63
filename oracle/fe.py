"""ORACLE (test infrastructure only): reference-element data and the blending map.

* P2 / P1 Lagrange bases on the reference tet xi in {xi_i >= 0, sum <= 1}
  ("nodal basis functions associated with the Lagrange interpolation
  points of order 1 and 2").  Local P2 order: vertices 0..3, edges 01,02,03,12,13,23.
* Q4 quadrature (reading R6): the 4-point degree-2 rule with
  barycentric points (a,b,b,b) (and permutations), a=(5+3 sqrt5)/20,
  b=(5-sqrt5)/20, weights 1/24.  The paper does not state its rule.
* Shell blending map (reading R3): B(x) = c_K x (n_K . x)/|x| (C^0
  globally, C^1 per macro), derivative J_B by differentiating that formula.
"""
from __future__ import annotations

import math

import numpy as np

SQ5 = math.sqrt(5.0)
Q4_A = (5.0 + 3.0 * SQ5) / 20.0
Q4_B = (5.0 - SQ5) / 20.0


def q4_rule():
    """Points as xi = (lambda1, lambda2, lambda3) with lambda0 = 1 - sum; weights sum to 1/6."""
    lam = np.full((4, 4), Q4_B)
    np.fill_diagonal(lam, Q4_A)
    return lam[:, 1:].copy(), np.full(4, 1.0 / 24.0)


def barycentric(xi: np.ndarray) -> np.ndarray:
    xi = np.atleast_2d(xi)
    return np.concatenate([1.0 - xi.sum(axis=1, keepdims=True), xi], axis=1)


# gradients of the barycentric coordinates w.r.t. xi
DLAM = np.array([[-1.0, -1.0, -1.0], [1.0, 0.0, 0.0], [0.0, 1.0, 0.0], [0.0, 0.0, 1.0]])
EDGES = [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)]


def p2_basis(xi: np.ndarray) -> np.ndarray:
    """phi_m = lam_m (2 lam_m - 1) for vertices, phi_ij = 4 lam_i lam_j for edges. -> (P,10)"""
    lam = barycentric(xi)
    out = np.empty((lam.shape[0], 10))
    for m in range(4):
        out[:, m] = lam[:, m] * (2.0 * lam[:, m] - 1.0)
    for e, (i, j) in enumerate(EDGES):
        out[:, 4 + e] = 4.0 * lam[:, i] * lam[:, j]
    return out


def p2_grad(xi: np.ndarray) -> np.ndarray:
    """Reference gradients d phi / d xi -> (P,10,3)."""
    lam = barycentric(xi)
    out = np.empty((lam.shape[0], 10, 3))
    for m in range(4):
        out[:, m, :] = (4.0 * lam[:, m] - 1.0)[:, None] * DLAM[m][None, :]
    for e, (i, j) in enumerate(EDGES):
        out[:, 4 + e, :] = 4.0 * (lam[:, i][:, None] * DLAM[j][None, :] + lam[:, j][:, None] * DLAM[i][None, :])
    return out


def p1_basis(xi: np.ndarray) -> np.ndarray:
    return barycentric(xi)


# ---------------------------------------------------------------- blending

def shell_blend_params(X4: np.ndarray):
    """Per macro tet (4 vertices on layer spheres with 3 distinct directions):
    n_K = outward unit normal of the plane through the 3 unit directions, c_K = 1/(n_K . p).
    X4: (M,4,3) -> (nhat (M,3), c (M,))."""
    M = X4.shape[0]
    nhat = np.empty((M, 3))
    c = np.empty(M)
    for t in range(M):
        dirs = []
        for v in X4[t]:
            d = v / np.linalg.norm(v)
            if not any(np.linalg.norm(d - e) < 1e-10 for e in dirs):
                dirs.append(d)
        if len(dirs) != 3:
            raise ValueError("shell blending needs exactly 3 distinct vertex directions per macro tet")
        p, q, r = dirs
        nv = np.cross(q - p, r - p)
        nv /= np.linalg.norm(nv)
        if nv @ p < 0:
            nv = -nv
        nhat[t] = nv
        c[t] = 1.0 / (nv @ p)
    return nhat, c


def blend(x: np.ndarray, nhat: np.ndarray, c: np.ndarray) -> np.ndarray:
    """B(x) = c x (n . x)/|x|   (x, nhat: (N,3); c: (N,))."""
    r = np.linalg.norm(x, axis=1)
    return (c * np.einsum("nd,nd->n", nhat, x) / r)[:, None] * x


def blend_jacobian(x: np.ndarray, nhat: np.ndarray, c: np.ndarray) -> np.ndarray:
    """J_B = dB/dx = c [ phi I + x (grad phi)^T ],  phi = (n . x)/|x|,
    grad phi = n/|x| - (n . x) x / |x|^3.   -> (N,3,3), J[i,j] = dB_i/dx_j."""
    r = np.linalg.norm(x, axis=1)
    nx = np.einsum("nd,nd->n", nhat, x)
    phi = nx / r
    gphi = nhat / r[:, None] - (nx / r ** 3)[:, None] * x
    J = phi[:, None, None] * np.eye(3)[None] + x[:, :, None] * gphi[:, None, :]
    return c[:, None, None] * J
