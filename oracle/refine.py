"""ORACLE (test infrastructure only): uniform structured refinement and node numbering.

P:194 -- "an unstructured coarse grid consisting of ... tetrahedrons in 3D on
which a structured refinement is performed [Bey1995]".  Implemented literally
as ITERATED Bey red refinement: every tet is split into 4 corner children and
4 children of the inner octahedron, which is cut along the diagonal joining
the midpoints of edges (0,2) and (1,3) (Bey's child ordering below).  A
macro tet's vertex order is ascending global id (reading R5 in DESIGN.md).

Coordinates are exact integers: a micro vertex is stored as its 4 barycentric
weights w.r.t. the macro tet's vertices, at lattice resolution n = 2^L.

Canonical node identity (contract shared with the C-ABI by
specification, not by code): every node lies in the relative interior of one
macro primitive (vertex/edge/face/cell); key = [dim, ascending vertex ids
(-1 padded), their positive integer weights (0 padded), res].  Canonical order
= lexicographic order of keys.  P2 vectors: node-major, (x,y,z) interleaved.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

# Bey's red refinement of (x0,x1,x2,x3); xij = midpoint of edge ij.
_BEY_CHILDREN = [
    ("0", "01", "02", "03"),
    ("01", "1", "12", "13"),
    ("02", "12", "2", "23"),
    ("03", "13", "23", "3"),
    ("01", "02", "03", "13"),
    ("01", "02", "12", "13"),
    ("02", "03", "13", "23"),
    ("02", "12", "13", "23"),
]

# local P2 node order of a tet: vertices 0..3, then edge midpoints 01,02,03,12,13,23
P2_EDGES = [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)]


def bey_refine_once(W: np.ndarray) -> np.ndarray:
    """W: (T,4,4) integer barycentric weights (rows = tet vertices); all even. -> (8T,4,4)."""
    pts = {str(i): W[:, i, :] for i in range(4)}
    for a, b in P2_EDGES:
        s = W[:, a, :] + W[:, b, :]
        assert np.all(s % 2 == 0)
        pts[f"{a}{b}"] = s // 2
    kids = [np.stack([pts[v] for v in ch], axis=1) for ch in _BEY_CHILDREN]
    # interleave so that children of one parent are contiguous
    return np.stack(kids, axis=1).reshape(-1, 4, 4)


def refine_macro(level: int) -> np.ndarray:
    """Micro tets of ONE macro tet after `level` Bey refinements: (8^L, 4, 4) weights at res 2^L."""
    n = 2 ** level
    W = (np.eye(4, dtype=np.int64) * n)[None]
    for _ in range(level):
        W = bey_refine_once(W)
    return W


def keys_from_weights(w: np.ndarray, res: int, macro_ids: np.ndarray) -> np.ndarray:
    """w: (N,4) weights over the (ascending) macro vertex ids macro_ids (N,4). -> (N,10) keys."""
    N = w.shape[0]
    keys = np.full((N, 10), -1, dtype=np.int64)
    keys[:, 5:9] = 0
    nz = w > 0
    keys[:, 0] = nz.sum(axis=1) - 1
    pos = np.cumsum(nz, axis=1) - 1          # slot of each nonzero
    for c in range(4):
        rows = np.nonzero(nz[:, c])[0]
        keys[rows, 1 + pos[rows, c]] = macro_ids[rows, c]
        keys[rows, 5 + pos[rows, c]] = w[rows, c]
    keys[:, 9] = res
    return keys


@dataclass
class LevelMesh:
    """All micro tets of all macro tets at refinement level L, with canonical numbering."""
    level: int
    macro_verts: np.ndarray
    macro_tets: np.ndarray
    macro_vtag: np.ndarray
    tet_macro: np.ndarray            # (T,)
    tet_w: np.ndarray                # (T,4,4) int weights at res n=2^L
    p2_keys: np.ndarray              # (N2,10) canonical order
    p1_keys: np.ndarray              # (N1,10)
    tet_p2: np.ndarray               # (T,10) canonical P2 node ids (local order: v0..v3, e01..e23)
    tet_p1: np.ndarray               # (T,4)
    X: np.ndarray                    # (T,4,3) unblended vertex coordinates
    p2_xt: np.ndarray                # (N2,3) unblended node coordinates
    p1_xt: np.ndarray                # (N1,3)
    extra: dict = field(default_factory=dict)

    @property
    def n_tets(self):
        return self.tet_w.shape[0]

    @property
    def n_p2(self):
        return self.p2_keys.shape[0]

    @property
    def n_p1(self):
        return self.p1_keys.shape[0]


def _coords(w: np.ndarray, res: int, macro_X: np.ndarray) -> np.ndarray:
    """x~ = sum_m (w_m / res) X_m ; macro_X: (N,4,3)."""
    return np.einsum("nm,nmd->nd", w.astype(np.float64) / res, macro_X)


def build_level(macro_verts, macro_tets, macro_vtag, level: int, macro_subset=None) -> LevelMesh:
    macro_tets = np.sort(np.asarray(macro_tets, dtype=np.int64), axis=1)   # reading R5
    macro_verts = np.asarray(macro_verts, dtype=np.float64)
    sel = np.arange(macro_tets.shape[0]) if macro_subset is None else np.asarray(macro_subset)
    ref = refine_macro(level)                                  # (8^L,4,4)
    nm = len(sel)
    T = nm * ref.shape[0]
    tet_macro = np.repeat(sel, ref.shape[0])
    tet_w = np.tile(ref, (nm, 1, 1))
    n = 2 ** level
    mids = macro_tets[tet_macro]                               # (T,4) ascending ids
    mX = macro_verts[mids]                                     # (T,4,3)
    # P2 nodes of every tet at res 2n: vertices 2w, edges w_a + w_b
    w2 = np.empty((T, 10, 4), dtype=np.int64)
    w2[:, :4] = 2 * tet_w
    for e, (a, b) in enumerate(P2_EDGES):
        w2[:, 4 + e] = tet_w[:, a] + tet_w[:, b]
    k2 = keys_from_weights(w2.reshape(-1, 4), 2 * n, np.repeat(mids, 10, axis=0))
    p2_keys, first2, inv2 = np.unique(k2, axis=0, return_index=True, return_inverse=True)
    tet_p2 = inv2.reshape(T, 10)
    k1 = keys_from_weights(tet_w.reshape(-1, 4), n, np.repeat(mids, 4, axis=0))
    p1_keys, first1, inv1 = np.unique(k1, axis=0, return_index=True, return_inverse=True)
    tet_p1 = inv1.reshape(T, 4)
    X = np.einsum("tvm,tmd->tvd", tet_w.astype(np.float64) / n, mX)
    p2_xt = _coords(w2.reshape(-1, 4)[first2], 2 * n, np.repeat(mX, 10, axis=0)[first2])
    p1_xt = _coords(tet_w.reshape(-1, 4)[first1], n, np.repeat(mX, 4, axis=0)[first1])
    return LevelMesh(level, macro_verts, macro_tets, np.asarray(macro_vtag), tet_macro, tet_w,
                     p2_keys, p1_keys, tet_p2, tet_p1, X, p2_xt, p1_xt)


def boundary_faces(macro_tets: np.ndarray, macro_vtag: np.ndarray):
    """Macro faces belonging to exactly one macro tet, with their tag (common vertex tag, else 0)."""
    faces = {}
    for t in np.sort(macro_tets, axis=1):
        for skip in range(4):
            f = tuple(int(v) for i, v in enumerate(t) if i != skip)
            faces[f] = faces.get(f, 0) + 1
    out = []
    for f, cnt in faces.items():
        if cnt == 1:
            tags = {int(macro_vtag[v]) for v in f}
            out.append((f, tags.pop() if len(tags) == 1 else 0))
    return out


BC_NONE, BC_DIRICHLET, BC_FREESLIP = 0, 1, 2


def node_bc(keys: np.ndarray, macro_tets, macro_vtag, bc_by_tag: dict) -> np.ndarray:
    """Per-node BC kind: a node is constrained iff its primitive is a sub-simplex of a
    boundary face whose tag carries that BC (Dirichlet dominates).  bc_by_tag: {tag: kind},
    key 'all' applies to every boundary face."""
    sub = {}
    for f, tag in boundary_faces(macro_tets, macro_vtag):
        kind = bc_by_tag.get(tag, bc_by_tag.get("all", BC_NONE))
        if kind == BC_NONE:
            continue
        for r in (1, 2, 3):
            for s in _subsets(f, r):
                if kind == BC_DIRICHLET or sub.get(s) != BC_DIRICHLET:
                    sub[s] = kind
    out = np.zeros(keys.shape[0], dtype=np.int32)
    for i in np.nonzero(keys[:, 0] <= 2)[0]:
        k = keys[i]
        d = int(k[0])
        out[i] = sub.get(tuple(int(x) for x in k[1:2 + d]), BC_NONE)
    return out


def _subsets(f, r):
    from itertools import combinations
    return [tuple(c) for c in combinations(f, r)]
