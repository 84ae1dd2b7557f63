"""Shared set-up for parity tests: builds the SAME seeded synthetic case on both sides.

CUDA side: macro mesh -> hhg_mesh_create / blend_map / hhg_set_bc; node keys and coordinates come
from the library (hhg_canonical_keys, hhg_node_coords); inputs from workload/ keyed by those keys.
Oracle side: its own refinement, numbering, coordinates; inputs from workload/ keyed by ITS keys.
Nothing computed by one side is fed to the other.  Comparison happens in canonical order.
"""
from __future__ import annotations

import numpy as np

from workload import uniform_vec, uniform_from_keys, viscosity

BC_SHELL = "shell"      # no-slip outer (surface), free-slip inner (CMB)
BC_ALL = "all"          # zero Dirichlet on every boundary face (config 1)


def rel_l2(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


# ------------------------------------------------------------------ oracle side
def oracle_bc(bc):
    from oracle.refine import BC_DIRICHLET, BC_FREESLIP
    return {2: BC_DIRICHLET, 1: BC_FREESLIP} if bc == BC_SHELL else {"all": BC_DIRICHLET}


def oracle_case(macro, level, blended, bc, eta_cj=None, gamma=0.0, build=("A", "B", "C")):
    from oracle.refine import build_level
    from oracle.operators import Discretisation, node_coords
    lm = build_level(macro.verts, macro.tets, macro.vtag, level)
    eta = None
    if eta_cj is not None:
        eta = viscosity(node_coords(lm, "P1", blended), lm.p1_keys, *eta_cj)
    d = Discretisation(lm, blended, eta, gamma, oracle_bc(bc), build=build)
    return lm, d, eta


# ------------------------------------------------------------------ CUDA side
def lib_mesh(macro, level_max, blended, bc):
    import paper_2506_04157_b200 as hhg
    M = hhg.Mesh.from_macro(macro, level_max)
    if blended:
        M.blend_map(hhg.HHG_BLEND_SHELL)
    if bc == BC_SHELL:
        M.set_bc(hhg.HHG_BND_OUTER, hhg.HHG_BC_DIRICHLET0)
        M.set_bc(hhg.HHG_BND_INNER, hhg.HHG_BC_FREESLIP)
    elif bc == BC_ALL:
        M.set_bc(hhg.HHG_BND_ALL, hhg.HHG_BC_DIRICHLET0)
    return M


def lib_coords_canonical(M, level, space):
    """Library node coordinates in canonical order (n,3) as numpy."""
    import torch
    xyz = M.node_coords(level, space)
    cols = [M.to_canonical(level, space, xyz[:, c].contiguous()) for c in range(3)]
    return torch.stack(cols, 1).cpu().numpy()


def lib_eta(M, level, eta_cj):
    import paper_2506_04157_b200 as hhg
    if eta_cj is None:
        return None
    keys = M.canonical_keys(level, hhg.HHG_P1)
    eta_c = viscosity(lib_coords_canonical(M, level, hhg.HHG_P1), keys, *eta_cj)
    return M.from_canonical(level, hhg.HHG_P1, eta_c)


def lib_u(M, level, seed):
    """Seeded velocity (canonical -> library layout), then constrained on the GPU (hhg_apply_bc)."""
    import paper_2506_04157_b200 as hhg
    keys = M.canonical_keys(level, hhg.HHG_P2)
    u = M.from_canonical(level, hhg.HHG_P2VEC, uniform_vec(keys, seed))
    return M.apply_bc(level, u)


def lib_p(M, level, seed):
    import paper_2506_04157_b200 as hhg
    keys = M.canonical_keys(level, hhg.HHG_P1)
    return M.from_canonical(level, hhg.HHG_P1, uniform_from_keys(keys, seed, 0))


def canon(M, level, space, v):
    return M.to_canonical(level, space, v).cpu().numpy()
