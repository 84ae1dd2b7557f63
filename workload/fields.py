"""Seeded synthetic workload: temperature / viscosity fields and the BASELINE configs.

Input generation only.  The paper's geodynamic inputs (plate reconstructions
P:109, the 500 Myr temperature checkpoint P:676, the eta_base profile that is
only a figure) are not available; these synthetic fields stand in
for them with the paper's shapes: a Frank-Kamenetskii-type exponential of a
temperature field (eq:ViscosityDef) with a radial jump, contrast
>= 1e4 (BASELINE.json configs 2-5).

Reading (R8): Y_4^2 is the unnormalised P_4^2(cos theta) cos(2 phi)
with P_4^2(t) = (15/2)(7t^2-1)(1-t^2) (max ~9.64) and T is clipped to [0,1],
so that eta spans exactly C (from T) times J (radial jump).
"""
from __future__ import annotations

import math

import numpy as np

from .seeded import uniform_from_keys

NOISE_SEED = 5


def temperature(xyz: np.ndarray, keys: np.ndarray, noise_seed: int = NOISE_SEED) -> np.ndarray:
    """T(x) = 0.5 + 0.1 sin(4 pi r) Y_4^2(theta, phi) + 0.01 xi, clipped to [0, 1]."""
    x, y, z = xyz[:, 0], xyz[:, 1], xyz[:, 2]
    r = np.sqrt(x * x + y * y + z * z)
    t = np.clip(z / r, -1.0, 1.0)           # cos(theta), theta = polar angle from +z
    phi = np.arctan2(y, x)
    p42 = 7.5 * (7.0 * t * t - 1.0) * (1.0 - t * t)
    ylm = p42 * np.cos(2.0 * phi)
    xi = uniform_from_keys(keys, noise_seed, 0)
    T = 0.5 + 0.1 * np.sin(4.0 * math.pi * r) * ylm + 0.01 * xi
    return np.clip(T, 0.0, 1.0)


def viscosity(xyz: np.ndarray, keys: np.ndarray, contrast: float, jump: float,
              r_jump: float = 0.9, noise_seed: int = NOISE_SEED) -> np.ndarray:
    """eta = exp(ln(contrast) (0.5 - T)) * (jump if r < r_jump else 1)."""
    T = temperature(xyz, keys, noise_seed)
    r = np.linalg.norm(xyz, axis=1)
    eta = np.exp(math.log(contrast) * (0.5 - T))
    return np.where(r < r_jump, jump * eta, eta)


# BASELINE.json configs as concrete synthetic recipes
CONFIGS = {
    1: dict(mesh="reftet", level=3, blend=False, eta=None, gamma=0.0, bc="all_dirichlet",
            seed_u=0, seed_p=1),
    2: dict(mesh=("icoshell", 3, 2, 0.55, 1.0), level=4, blend=True, eta=(1e4, 10.0),
            gamma=0.3781, bc="noslip_outer_freeslip_inner", seed_u=2, seed_p=3),
    3: dict(mesh=("icoshell", 3, 2, 0.55, 1.0), level=5, blend=True, eta=(1e6, 30.0),
            gamma=0.3781, bc="noslip_outer_freeslip_inner", seed_rhs=4, seed_power=6,
            pre=3, post=3, degree=3, power_iters=20, coarse_iters=50, l_min=1),
}
GAMMA_TALA = 0.3781   # Di / Gamma_0, table of nondimensional numbers
