"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle.

Holds no arithmetic of the method (no refinement, blending, quadrature or
operator work): only macro-mesh data, counter-based random values keyed by node
identity, and the synthetic temperature/viscosity recipe.
"""
from .macro_mesh import MacroMesh, icoshell, reference_tet, TAG_INNER, TAG_OUTER, TAG_INTERIOR  # noqa: F401
from .seeded import splitmix64, uniform_from_keys, uniform_vec, hash_keys, reduce_keys  # noqa: F401
from .fields import temperature, viscosity, CONFIGS, GAMMA_TALA  # noqa: F401
