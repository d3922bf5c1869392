"""Nested-mesh transfer and the strong-error study of PAPER.md §4.1 (P332-335), as plain
definitions (TEST INFRASTRUCTURE ONLY, see oracle/__init__.py).

* prolongation P (fine nodes x coarse nodes): linear (hat-function) interpolation of coarse
  nodal values at the fine nodes of the same graph, meshes nested edge by edge (fine n_e an
  integer multiple of coarse n_e)  -- SPEC S119-127;
* noise projection W_coarse = P^T W_fine ("we project the noise generated on the overkill
  mesh down", P335; SPEC S256-264);
* strong error (P335): err = mean_i (u_ok - P u_c)^T M_ok (u_ok - P u_c) over realizations,
  with u_ok solved on the overkill mesh from W_fine and u_c on the coarse mesh from P^T W_fine
  (the quadrature sums of oracle.solve.apply);
* the refinement sweep of P332-335: per level h_max = 2^-j the paper's quadrature step
  k = -1/(beta ln h) (k=None), the OLS rate of ln(RMS err) on ln h (the
  printed errors fall at the RMS rate 2 beta - 1/2 of P334).
Pinned in tests/test_oracle_refine.py: the sweep reproduces 2 beta - 1/2 (P334, Table 1 P450).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from . import fem, noise, quadrature, rates, solve
from .mesh import build_mesh


def prolongation(coarse, fine) -> sp.csr_matrix:
    """P[j, i] = coarse hat function i evaluated at fine node j (SPEC S119-127)."""
    if coarse.n_vertices != fine.n_vertices or coarse.n_edges != fine.n_edges:
        raise ValueError("meshes of different graphs")
    rows, cols, vals = [], [], []
    for v in range(fine.n_vertices):  # vertices coincide
        rows.append(fine.vertex_dof(v))
        cols.append(coarse.vertex_dof(v))
        vals.append(1.0)
    for e in range(fine.n_edges):
        nc, nf = int(coarse.n_el[e]), int(fine.n_el[e])
        if nf % nc:
            raise ValueError(f"edge {e}: fine n_e = {nf} is not a multiple of coarse n_e = {nc}")
        r = nf // nc
        for j in range(1, nf):  # fine interior node j at x = j h_f = (j / r) h_c
            c, q = divmod(j, r)
            w = q / r
            rows.append(fine.node(e, j))
            cols.append(coarse.node(e, c))
            vals.append(1.0 - w)
            if q:
                rows.append(fine.node(e, j))
                cols.append(coarse.node(e, c + 1))
                vals.append(w)
    return sp.csr_matrix((vals, (rows, cols)), shape=(fine.n_dofs, coarse.n_dofs))


def strong_error(graph, h_coarse, h_ok, kappa, beta, k, W_ok, u_ok=None):
    """Per-realization squared M_ok-norm errors [S] of the coarse solution upsampled to the
    overkill mesh, for overkill noise W_ok [S, N_ok] (P335).  k = None: each mesh uses the
    paper's step k = -1/(beta ln h) of its own h (P335); u_ok: the overkill solution if known."""
    fine = build_mesh(graph, h_ok)
    coarse = build_mesh(graph, h_coarse)
    P = prolongation(coarse, fine)
    Wc = (P.T @ np.asarray(W_ok).T).T
    if u_ok is None:
        k_ok = quadrature.k_from_h(beta, h_ok) if k is None else k
        u_ok = solve.apply(solve.setup(graph, h_ok, kappa, beta, k_ok), W_ok)
    k_c = quadrature.k_from_h(beta, h_coarse) if k is None else k
    u_c = solve.apply(solve.setup(graph, h_coarse, kappa, beta, k_c), Wc)
    d = u_ok - (P @ u_c.T).T
    M = fem.lumped_mass(fine)
    return np.einsum("si,i,si->s", d, M, d)


def strong_error_sweep(graph, levels, ok_level, kappa, beta, seed, n_real, k=None):
    """The study of P332-335 on `graph`: overkill h = 2^-ok_level, coarse h = 2^-j (j in levels),
    n_real overkill noise realizations (seeds seed..seed+n_real-1 of the canonical stream).
    Returns (h, mean squared errors, RMS rate from the OLS fit of ln RMS on ln h)."""
    h_ok = 2.0 ** -ok_level
    k_ok = quadrature.k_from_h(beta, h_ok) if k is None else k
    prob_ok = solve.setup(graph, h_ok, kappa, beta, k_ok)
    W = noise.white_noise(prob_ok.ML, seed, n_real)
    u_ok = solve.apply(prob_ok, W)
    hs = [2.0 ** -j for j in levels]
    ms = [float(strong_error(graph, hc, h_ok, kappa, beta, k, W, u_ok=u_ok).mean()) for hc in hs]
    r, _ = rates.fit_rate(hs, np.sqrt(ms))
    return hs, ms, r
