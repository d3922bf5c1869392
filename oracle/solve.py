"""Oracle GRF sample: the definition the DD/PCG path must reproduce.

u_s = sum_{l=-K^-}^{K^+} x_{l,s},   A^{(l)} x_{l,s} = W_s,
A^{(l)} = c_I^{(l)} M_L + c_L^{(l)} (kappa^2 M_L + G)

PAPER.md P67 (L^{-beta} ~= sum_l (c_I I + c_L L)^{-1}), P75-78
[eq:spde_approx_fem] ("solving A^{(l)} u^{(l)} = W for all l, and aggregating"),
P313-324 (accumulation u = sum_l u^{(l)}), with the lumped mass in both the
operator and the noise and one static W per sample (Q5).

Each A^{(l)} is factored once and applied to all requested samples; the
per-node results are summed in ascending l (SPEC S323).  Two direct solvers:
``method="ldlt"`` (default) is the plain C sparse LDL^T of oracle/ldlt.c with
the fixed interior-first + minimum-degree-vertex ordering of SURVEY §8c-O7
(factors 1e7-DOF meshes; nodes in parallel threads); ``method="superlu"`` is
scipy's SuperLU (a library sparse LU, COLAMD ordering), kept as the second,
independent route that pins the first (tests/test_oracle_ldlt.py).
"""
from __future__ import annotations

import dataclasses
import numpy as np
from scipy.sparse.linalg import splu

from . import fem, noise, quadrature
from .mesh import build_mesh


@dataclasses.dataclass
class Problem:
    mesh: object
    ML: np.ndarray
    G: object
    kappa: float
    plan: quadrature.Plan
    _ldlt: object = None

    def ldlt(self):
        """The mesh's ordering + symbolic factorization (oracle/ldlt.py), built on first use."""
        if self._ldlt is None:
            from .ldlt import Solver
            self._ldlt = Solver(self.mesh, self.G, self.ML)
        return self._ldlt


def setup(graph, h, kappa, beta, k) -> Problem:
    if not (kappa > 0):
        raise ValueError("kappa must be positive")
    mesh = build_mesh(graph, h)
    ML = fem.lumped_mass(mesh)
    G = fem.stiffness(mesh)
    return Problem(mesh, ML, G, float(kappa), quadrature.plan(beta, k))


def node_solve(prob: Problem, li: int, rhs: np.ndarray, method: str = "ldlt") -> np.ndarray:
    """x = (A^{(l)})^{-1} rhs for quadrature index li (0-based into plan.l); rhs [S, N]."""
    rhs = np.atleast_2d(np.asarray(rhs, dtype=np.float64))
    if method == "ldlt":
        return prob.ldlt().node_solve(prob.plan.c_I[li], prob.plan.c_L[li], prob.kappa, rhs)
    A = fem.operator(prob.ML, prob.G, prob.kappa, prob.plan.c_I[li], prob.plan.c_L[li])
    lu = splu(A, permc_spec="COLAMD")
    return lu.solve(np.ascontiguousarray(rhs.T)).T


def apply(prob: Problem, rhs: np.ndarray, node_range=None, return_residuals=False, method: str = "ldlt",
          threads=None):
    """sum_l (A^{(l)})^{-1} rhs, ascending l.  rhs [S, N] -> [S, N]."""
    rhs = np.atleast_2d(np.asarray(rhs, dtype=np.float64))
    L = prob.plan.n_nodes
    lo, hi = (0, L) if node_range is None else node_range
    if method == "ldlt" and not return_residuals:
        return prob.ldlt().apply(prob.plan, prob.kappa, rhs, (lo, hi), threads=threads)
    u = np.zeros_like(rhs)
    res = []
    for li in range(lo, hi):
        A = fem.operator(prob.ML, prob.G, prob.kappa, prob.plan.c_I[li], prob.plan.c_L[li])
        lu = splu(A, permc_spec="COLAMD")
        x = lu.solve(np.ascontiguousarray(rhs.T)).T
        if return_residuals:
            r = (A @ x.T).T - rhs
            res.append(np.linalg.norm(r, axis=1) / np.maximum(np.linalg.norm(rhs, axis=1), 1e-300))
        u = u + x
    if return_residuals:
        return u, np.array(res)
    return u


def sample(graph, h, kappa, beta, k, seed, n_samples, samples=None, node_range=None, method="ldlt", threads=None):
    """GRF samples u [len(samples), N] and their noise W.  `samples` picks sample indices of the call."""
    prob = setup(graph, h, kappa, beta, k)
    if samples is None:
        samples = list(range(n_samples))
    W = noise.white_noise(prob.ML, seed, n_samples, samples=samples)
    u = apply(prob, W, node_range=node_range, method=method, threads=threads)
    return u, W, prob
