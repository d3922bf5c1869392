"""CPU fp64 ORACLE for the fractional-SPDE GRF sampler of arxiv 2605.02670.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import or run
anything under ``oracle/``.  The product path (``paper_2605_02670_b200``)
never imports it and fails loudly when its CUDA library is missing.

The oracle shares no code with the CUDA path.  Its only common dependency is
``synth/`` (seeded graph generators, no method arithmetic).  It computes the
*definition* of what the GPU path computes:

    u_s = sum_{l=-K^-}^{K^+} (c_I^{(l)} M_L + c_L^{(l)} (kappa^2 M_L + G))^{-1} W_s,
    W_s = M_L^{1/2} z_s,

PAPER.md P60-67 [eq:coefficients], P75-77 [eq:spde_approx_fem], P106-109 (§2.5
lumping), P137-160 (stencils), P335 (K^-/K^+).  Each node's system is solved by
a sparse direct factorization -- the plain C LDL^T of ``ldlt.c`` with a fixed
interior-first / minimum-degree-vertex ordering, or scipy's
SuperLU, a library primitive, as the second route that pins it -- no domain
decomposition, no Thomas, no PCG.  The sum runs in ascending l (SPEC S323).

Modules:
    mesh        Phase 1 mesh / DOF order                 (P122-123)
    fem         lumped + consistent mass, stiffness       (P126-160)
    quadrature  K^-, K^+, c_I, c_L; scalar sinc rule      (P54-67, P335)
    noise       Philox4x32-10 + fixed-algorithm Box-Muller (P99-109, P150)
    solve       per-node direct solves + quadrature sum  (P67-78, P313-324)
    ldlt        sparse LDL^T direct solver (ldlt.c)
    spectral    dense generalized-eigen oracle (tiny)
    dd          Schur / NN-preconditioner DEFINITIONS     (P111-118, P204-213, P298)
    rates       OLS log-log rate fit                      (P335)

Parity pins for each are in tests/test_oracle_*.py (``-m "not gpu"``).
"""
