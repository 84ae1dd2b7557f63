"""C-ABI checks that need no GPU: the library loads, exports every symbol include/hhg_stokes.h
declares, and its host-side logic (lengths, canonical keys, argument errors) is right."""
import os
import re

import numpy as np
import pytest

import paper_2506_04157_b200 as hhg
from workload import icoshell, reference_tet

HEADER = os.path.join(os.path.dirname(os.path.dirname(__file__)), "include", "hhg_stokes.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    src = re.sub(r"^\s*typedef[^;]*;", "", src, flags=re.M | re.S)   # function-pointer typedefs are not symbols
    names = re.findall(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\s*\**\s+\**([A-Za-z_][A-Za-z0-9_]*)\s*\(", src, re.M)
    return sorted(set(n for n in names if n not in ("if", "return")))


def test_every_declared_symbol_is_exported():
    names = declared_functions()
    assert len(names) >= 30
    lib = hhg.lib()
    for n in names:
        assert hasattr(lib, n), n
    assert sorted(hhg.EXPORTS) == names


def test_version_names_the_arch():
    assert "sm_100a" in hhg.version()


@pytest.mark.parametrize("ntan,nrad,L", [(3, 2, 1), (3, 2, 2), (2, 3, 1)])
def test_canonical_keys_match_oracle(ntan, nrad, L):
    from oracle.refine import build_level
    m = icoshell(ntan, nrad)
    M = hhg.Mesh.from_macro(m, L)
    lm = build_level(m.verts, m.tets, m.vtag, L)
    assert np.array_equal(M.canonical_keys(L, hhg.HHG_P2), lm.p2_keys)
    assert np.array_equal(M.canonical_keys(L, hhg.HHG_P1), lm.p1_keys)
    assert M.canonical_len(L, hhg.HHG_P2VEC) == 3 * lm.n_p2


def test_vector_lengths():
    m = icoshell(3, 2)
    M = hhg.Mesh.from_macro(m, 4)
    for L in range(5):
        n1, n2 = 2 ** L, 2 ** (L + 1)
        assert M.vec_len(L, hhg.HHG_P1) == 240 * (n1 + 1) * (n1 + 2) * (n1 + 3) // 6
        assert M.vec_len(L, hhg.HHG_P2VEC) == 3 * 240 * (n2 + 1) * (n2 + 2) * (n2 + 3) // 6
    assert M.local_macros() == 240


def test_argument_errors():
    r = reference_tet()
    with pytest.raises(hhg.HHGError, match="HHG_EINVAL"):
        hhg.Mesh(r.verts, r.tets, r.vtag, level_max=9)
    with pytest.raises(hhg.HHGError, match="HHG_EINVAL"):
        hhg.Mesh(r.verts, np.array([[0, 1, 2, 2]]), r.vtag, level_max=1)
    M = hhg.Mesh.from_macro(r, 2)
    with pytest.raises(hhg.HHGError, match="HHG_ELEVEL"):
        M.vec_len(3, hhg.HHG_P1)
    with pytest.raises(hhg.HHGError, match="HHG_EINVAL"):
        M.vec_len(1, 7)
    with pytest.raises(hhg.HHGError, match="HHG_EDOMAIN"):
        M.blend_map(hhg.HHG_BLEND_SHELL)      # reference tet has a vertex at the origin
    with pytest.raises(hhg.HHGError, match="HHG_EINVAL"):
        M.set_bc(5, hhg.HHG_BC_DIRICHLET0)


@pytest.mark.parametrize("ntan,nrad", [(2, 2), (3, 2), (5, 3)])
def test_library_icoshell_generator_matches_workload(ntan, nrad):
    """hhg_icoshell_macro (the library's shell generator) reproduces the workload's shell(ntan, nrad):
    identical numbering, tets and tags, coordinates to 1e-15; 60 (ntan-1)^2 (nrad-1) macros."""
    import numpy as np
    import paper_2506_04157_b200 as hhg
    from workload import icoshell
    v, t, g = hhg.icoshell_macro(ntan, nrad, 0.55, 1.0)
    w = icoshell(ntan, nrad, 0.55, 1.0)
    assert t.shape[0] == 60 * (ntan - 1) ** 2 * (nrad - 1)
    assert np.array_equal(t, w.tets) and np.array_equal(g, w.vtag)
    assert np.abs(v - w.verts).max() <= 1e-15
    with pytest.raises(hhg.HHGError):
        hhg.icoshell_macro(1, 2)
