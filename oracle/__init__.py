"""CPU ORACLE for the blended P2-P1 compressible-Stokes hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` leg may import anything under ``oracle/``.  The product
path (``paper_2506_04157_b200``) never does: it fails loudly without its CUDA
library.

What it is: a plain, slow, obviously-correct numpy/scipy implementation written
from the paper (arxiv 2506.04157, /root/reference/PAPER.md, cited "P:<line>"):
  * refine.py    -- iterated Bey red refinement of each macro tet and the
                    canonical node numbering contract
  * fe.py        -- P2/P1 Lagrange bases, Q4 quadrature, shell blending map and
                    its Jacobian
  * operators.py -- element matrices of A, B, C from the weak forms
                    assembled into scipy CSR matrices; boundary masks and the
                    free-slip projection P_v; diag(A) without P_v
  * multigrid.py -- P2 nodal-interpolation prolongation and its transpose,
                    Chebyshev smoother, power iteration, Jacobi-PCG coarse solve
                    and the V-cycle of fig:ASolverStructure; P1 linear
                    prolongation (w-BFBT K multigrid); the A-block CG
  * stokes.py    -- FGMRES + Uzawa block preconditioners with the mass,
                    V-cycle BFBT and weighted BFBT Schur approximations
  * temperature.py -- the eq:WeakTemp operator, its symmetric part and the
                    Dirichlet solve
  * mmoc.py      -- RK4 particle back-tracking with brute-force point location
                    

Every function cites the passage it follows.  Readings of silent/garbled
passages are listed in DESIGN.md ("Readings").  All floating point is fp64.
Parity status: every function is pinned by a ``-m "not gpu"`` test in
tests/test_oracle_*.py against closed forms, exact rationals, invariants or
brute force; none is "parity unpinned" (the blended C is pinned by closed-form
shell integrals, tests/test_oracle_operators.py).
"""
