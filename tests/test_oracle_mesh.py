"""Pins of oracle/refine.py: iterated Bey refinement vs the Freudenthal lattice (written out
here independently), counts, the paper's printed DoF numbers (tests/golden), key invariants."""
import json
import os
from itertools import combinations

import numpy as np
import pytest

from oracle.refine import refine_macro, build_level, boundary_faces, node_bc, BC_DIRICHLET, BC_FREESLIP
from workload import icoshell, reference_tet, reduce_keys

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "paper_dof_counts.json")


def lattice_tets(n):
    """Freudenthal lattice of the reference tet: per anchor (i,j,k), s=i+j+k:
    up {000,100,010,001} if s<=n-1; 4 octahedron tets around diagonal 010-101 if s<=n-2;
    down {011,101,110,111} if s<=n-3."""
    out = set()
    up = ["000", "100", "010", "001"]
    octs = [["010", "100", "101", "110"], ["001", "010", "100", "101"],
            ["010", "011", "101", "110"], ["001", "010", "011", "101"]]
    down = ["011", "101", "110", "111"]
    for k in range(n):
        for j in range(n - k):
            for i in range(n - j - k):
                s = i + j + k
                a = np.array([i, j, k])
                groups = ([up] if s <= n - 1 else []) + (octs if s <= n - 2 else []) + ([down] if s <= n - 3 else [])
                for g in groups:
                    out.add(tuple(sorted(tuple(a + np.array([int(ch) for ch in v])) for v in g)))
    return out


@pytest.mark.parametrize("L", [1, 2, 3])
def test_iterated_bey_refinement_is_the_freudenthal_lattice(L):
    W = refine_macro(L)
    assert W.shape[0] == 8 ** L
    got = {tuple(sorted(tuple(int(x) for x in v[1:]) for v in t)) for t in W}
    assert got == lattice_tets(2 ** L)
    # equal volumes
    V = W[:, 1:, 1:] - W[:, :1, 1:]
    assert len(set(np.abs(np.round(np.linalg.det(V.astype(float)), 9)))) == 1


def test_interior_vertex_valence_24():
    W = refine_macro(3)
    n = 8
    cnt = {}
    for t in W:
        for v in t:
            cnt[tuple(v)] = cnt.get(tuple(v), 0) + 1
    interior = [c for v, c in cnt.items() if min(v) > 0]
    assert interior and all(c == 24 for c in interior)


def test_icoshell_macro_counts():
    m = icoshell(3, 2)
    assert m.n_verts == 84 and m.n_tets == 240
    edges = {e for t in m.tets for e in combinations(sorted(t), 2)}
    faces = {}
    for t in m.tets:
        for f in combinations(sorted(t), 3):
            faces[f] = faces.get(f, 0) + 1
    assert len(edges) == 402 and len(faces) == 560
    assert sum(1 for c in faces.values() if c == 1) == 160
    for nt, nr in [(3, 3), (5, 2), (5, 3)]:
        assert icoshell(nt, nr).n_tets == 60 * (nt - 1) ** 2 * (nr - 1)
    # macro vertices lie on their layer spheres
    r = np.linalg.norm(m.verts, axis=1)
    assert np.allclose(np.sort(np.unique(np.round(r, 12))), [0.55, 1.0])


def shell_counts(ntan, nrad, L):
    """Closed form: P1 nodes at level L = (10 m^2 + 2)((nrad-1) 2^L + 1), m = (ntan-1) 2^L;
    P2 nodes at level L = P1 nodes at level L+1."""
    def v(l):
        m = (ntan - 1) * 2 ** l
        return (10 * m * m + 2) * ((nrad - 1) * 2 ** l + 1)
    return v(L + 1), v(L)


@pytest.mark.parametrize("ntan,nrad,L", [(3, 2, 1), (3, 2, 2), (3, 3, 1), (5, 2, 1), (2, 2, 2)])
def test_built_node_counts_match_closed_form(ntan, nrad, L):
    m = icoshell(ntan, nrad)
    lm = build_level(m.verts, m.tets, m.vtag, L)
    assert (lm.n_p2, lm.n_p1) == shell_counts(ntan, nrad, L)
    assert lm.n_tets == m.n_tets * 8 ** L


def test_paper_printed_dof_counts():
    g = json.load(open(GOLDEN))
    for name, e in g.items():
        if name.startswith("_"):
            continue
        p2, p1 = shell_counts(e["ntan"], e["nrad"], e["level"])
        up = 3 * p2 + p1
        for val, printed in ((up, e["up_dofs_printed"]), (p2, e["temperature_dofs_printed"])):
            mant, ex = printed.split("e")
            sig = len(mant.replace(".", ""))
            assert f"{val:.{sig - 1}e}".replace("e+0", "e") == printed, (name, val, printed)


def test_single_macro_counts_level3():
    m = reference_tet()
    lm = build_level(m.verts, m.tets, m.vtag, 3)
    assert (lm.n_p2, lm.n_p1, lm.n_tets) == (969, 165, 512)
    bc = node_bc(lm.p2_keys, lm.macro_tets, lm.macro_vtag, {"all": BC_DIRICHLET})
    assert int((bc == 0).sum()) == 455
    bc1 = node_bc(lm.p1_keys, lm.macro_tets, lm.macro_vtag, {"all": BC_DIRICHLET})
    assert int((bc1 == 0).sum()) == 35


def test_shell_boundary_classification_by_radius():
    m = icoshell(3, 2)
    lm = build_level(m.verts, m.tets, m.vtag, 2)
    bc = node_bc(lm.p2_keys, lm.macro_tets, lm.macro_vtag, {2: BC_DIRICHLET, 1: BC_FREESLIP})
    r = np.linalg.norm(lm.p2_xt, axis=1)
    # unblended flat faces: node radii of a layer lie between the inscribed plane distance and r
    assert np.all(bc[np.isclose(r, 1.0)] == BC_DIRICHLET)
    assert np.all(bc[np.isclose(r, 0.55)] == BC_FREESLIP)
    on_outer = bc == BC_DIRICHLET
    assert on_outer.sum() == 10 * 16 ** 2 + 2      # P2 nodes on one sphere at L2: m = 2 * 2^(L+1)
    assert (bc == BC_FREESLIP).sum() == on_outer.sum()
    assert len(boundary_faces(lm.macro_tets, lm.macro_vtag)) == 160


def test_keys_are_level_independent_for_nested_nodes():
    m = icoshell(3, 2)
    l1 = build_level(m.verts, m.tets, m.vtag, 1)
    l2 = build_level(m.verts, m.tets, m.vtag, 2)
    k1 = {tuple(r) for r in reduce_keys(l1.p2_keys)}
    k2 = {tuple(r) for r in reduce_keys(l2.p2_keys)}
    kp1 = {tuple(r) for r in reduce_keys(l2.p1_keys)}
    assert k1 <= k2          # coarse P2 nodes are fine P2 nodes
    assert k1 == kp1         # level-1 P2 nodes are exactly the level-2 P1 nodes
