"""Seeded synthetic workload: counter-based random values keyed by node identity.

Input generation only -- none of the method's arithmetic lives here.  Both the
CUDA path and the oracle obtain their random vectors from these functions,
each passing node keys that IT computed (library export vs. oracle numbering).

Node key (one int64 row of width 10):
    [dim, id0, id1, id2, id3, w0, w1, w2, w3, res]
dim = dimension of the macro primitive whose relative interior holds the node
(0 vertex, 1 edge, 2 face, 3 cell); id* = ascending global macro-vertex ids of
that primitive (-1 padded); w* = positive integer barycentric weights of the
node w.r.t. those vertices at lattice resolution ``res`` (0 padded).

The hash reduces (weights, res) by their largest common power of two first, so
the key is a property of the POINT (identical on every level and in the P1 and
P2 spaces), hence nested coarse nodes draw the same values as on finer levels.
"""
from __future__ import annotations

import numpy as np

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(z: np.ndarray) -> np.ndarray:
    """Vectorised splitmix64 finaliser (uint64 arithmetic wraps mod 2^64)."""
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = z + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def reduce_keys(keys: np.ndarray) -> np.ndarray:
    """Divide weights and res by their largest common power of two (level-independent key)."""
    keys = np.array(keys, dtype=np.int64, copy=True)
    w = keys[:, 5:10]
    while True:
        even = np.all((w % 2) == 0, axis=1) & (w[:, 4] > 1)
        if not even.any():
            break
        w[even] //= 2
    keys[:, 5:10] = w
    return keys


def hash_keys(keys: np.ndarray, seed: int, component: int = 0) -> np.ndarray:
    """h = seed; for t in (dim, ids.., reduced weights.., reduced res, component): h = splitmix64(h ^ t)."""
    rk = reduce_keys(keys)
    n = rk.shape[0]
    h = np.full(n, np.uint64(seed & 0xFFFFFFFFFFFFFFFF), dtype=np.uint64)
    dim = rk[:, 0]
    cols = [rk[:, 0]]
    for c in range(4):
        cols.append(np.where(c <= dim, rk[:, 1 + c], 0))
    for c in range(4):
        cols.append(np.where(c <= dim, rk[:, 5 + c], 0))
    cols.append(rk[:, 9])
    cols.append(np.full(n, component, dtype=np.int64))
    for t in cols:
        h = splitmix64(h ^ t.astype(np.int64).view(np.uint64))
    return h


def uniform_from_keys(keys: np.ndarray, seed: int, component: int = 0) -> np.ndarray:
    """U = 2 * ((h >> 11) * 2^-53) - 1 in [-1, 1)."""
    h = hash_keys(keys, seed, component)
    return 2.0 * ((h >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)) - 1.0


def uniform_vec(keys: np.ndarray, seed: int) -> np.ndarray:
    """Node-major, component-interleaved (x,y,z) vector of U[-1,1) values (components 1,2,3)."""
    n = keys.shape[0]
    out = np.empty((n, 3))
    for c in range(3):
        out[:, c] = uniform_from_keys(keys, seed, c + 1)
    return out.reshape(-1)
