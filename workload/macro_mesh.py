"""Seeded synthetic workload: macro (coarse, unstructured) meshes.

This module produces INPUT DATA only: vertex coordinates, macro tetrahedra and
vertex tags. It contains none of the method's arithmetic (no refinement, no
blending, no finite-element work). Both the CUDA path (through the C-ABI
``hhg_mesh_create``) and the CPU oracle consume its output as plain arrays.

Paper: P:194-196 (``subsec:Mesh``) -- "an unstructured coarse grid consisting of
... tetrahedrons in 3D", the thick spherical shell built from "a triangular
truncated pyramid mesh, based on the hollow icosahedron", divided "into layers
of equal height" and "subdivided into tetrahedrons in each layer".
The concrete recipe (planar face subdivision into (ntan-1)^2 triangles, vertices
normalised to the sphere, nrad radial shells, sorted-id staircase prism split)
is the reading recorded in DESIGN.md (SURVEY.md section 8 "Common definitions").

Vertex tags: 0 = interior, 1 = inner sphere (CMB, r = r_min), 2 = outer sphere
(surface, r = r_max).  Macro tets are stored with ascending vertex ids.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

TAG_INTERIOR = 0
TAG_INNER = 1   # CMB
TAG_OUTER = 2   # surface


@dataclass
class MacroMesh:
    verts: np.ndarray   # (V, 3) float64
    tets: np.ndarray    # (T, 4) int32, each row ascending
    vtag: np.ndarray    # (V,) int32
    name: str = ""
    r_min: float = 0.0
    r_max: float = 0.0

    @property
    def n_verts(self) -> int:
        return int(self.verts.shape[0])

    @property
    def n_tets(self) -> int:
        return int(self.tets.shape[0])


def reference_tet() -> MacroMesh:
    """BASELINE config 1: the reference tetrahedron (0,0,0),(1,0,0),(0,1,0),(0,0,1).

    All four vertices carry the OUTER tag so that every boundary face is a
    tagged boundary face (config 1 puts zero Dirichlet on all faces)."""
    verts = np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0], [0.0, 1.0, 0.0], [0.0, 0.0, 1.0]])
    tets = np.array([[0, 1, 2, 3]], dtype=np.int32)
    vtag = np.full(4, TAG_OUTER, dtype=np.int32)
    return MacroMesh(verts, tets, vtag, name="reftet")


def _icosahedron():
    phi = (1.0 + 5.0 ** 0.5) / 2.0
    v = []
    for s1 in (-1.0, 1.0):
        for s2 in (-1.0, 1.0):
            v.append((0.0, s1, s2 * phi))
            v.append((s1, s2 * phi, 0.0))
            v.append((s2 * phi, 0.0, s1))
    v = np.array(v)
    # faces: triples of mutually adjacent vertices (edge length 2)
    n = len(v)
    d = np.linalg.norm(v[:, None, :] - v[None, :, :], axis=2)
    adj = np.abs(d - 2.0) < 1e-9
    faces = []
    for a in range(n):
        for b in range(a + 1, n):
            if not adj[a, b]:
                continue
            for c in range(b + 1, n):
                if adj[a, c] and adj[b, c]:
                    faces.append((a, b, c))
    assert len(faces) == 20
    return v, np.array(faces, dtype=np.int64)


def icoshell(ntan: int, nrad: int, r_min: float = 0.55, r_max: float = 1.0) -> MacroMesh:
    """Thick spherical shell macro mesh shell(ntan, nrad).

    #macro tets = 60 (ntan-1)^2 (nrad-1); shell(3,2) -> 240 (the paper's 240
    macro elements)."""
    if ntan < 2 or nrad < 2 or not (0.0 < r_min < r_max):
        raise ValueError("icoshell: need ntan>=2, nrad>=2, 0<r_min<r_max")
    ico, faces = _icosahedron()
    m = ntan - 1
    # surface points keyed by (sorted icosahedron vertex ids, integer weights)
    key_to_id: dict = {}
    pts = []
    face_grid = []
    for (a, b, c) in faces:
        grid = {}
        for i in range(m + 1):
            for j in range(m + 1 - i):
                w = {a: m - i - j, b: i, c: j}
                key = tuple(sorted((vid, wt) for vid, wt in w.items() if wt > 0))
                if key not in key_to_id:
                    key_to_id[key] = len(pts)
                    p = (w[a] * ico[a] + w[b] * ico[b] + w[c] * ico[c]) / m
                    pts.append(p / np.linalg.norm(p))
                grid[(i, j)] = key_to_id[key]
        face_grid.append(grid)
    # deterministic surface numbering: sort by key
    keys_sorted = sorted(key_to_id.keys())
    remap = {key_to_id[k]: n for n, k in enumerate(keys_sorted)}
    ns = len(pts)
    surf = np.empty((ns, 3))
    for old, new in remap.items():
        surf[new] = pts[old]
    tris = []
    for grid in face_grid:
        for i in range(m):
            for j in range(m - i):
                tris.append((grid[(i, j)], grid[(i + 1, j)], grid[(i, j + 1)]))
                if i + j < m - 1:
                    tris.append((grid[(i + 1, j)], grid[(i, j + 1)], grid[(i + 1, j + 1)]))
    tris = np.array([[remap[t] for t in tri] for tri in tris], dtype=np.int64)
    assert len(tris) == 20 * m * m
    radii = [r_min + l * (r_max - r_min) / (nrad - 1) for l in range(nrad)]
    verts = np.concatenate([r * surf for r in radii], axis=0)
    vtag = np.zeros(ns * nrad, dtype=np.int32)
    vtag[:ns] = TAG_INNER
    vtag[(nrad - 1) * ns:] = TAG_OUTER
    tets = []
    for l in range(nrad - 1):
        for tri in tris:
            p, q, r = sorted(int(x) for x in tri)
            pi, qi, ri = l * ns + p, l * ns + q, l * ns + r
            po, qo, ro = pi + ns, qi + ns, ri + ns
            tets.append(sorted((pi, qi, ri, ro)))
            tets.append(sorted((pi, qi, qo, ro)))
            tets.append(sorted((pi, po, qo, ro)))
    tets = np.array(tets, dtype=np.int32)
    return MacroMesh(verts, tets, vtag, name=f"shell({ntan},{nrad})", r_min=r_min, r_max=r_max)
