"""Consistent-mass variant (PAPER.md P126-150) as plain definitions
(TEST INFRASTRUCTURE ONLY, see oracle/__init__.py).

* operator A^{(l)} = c_I M + c_L (kappa^2 M + G) with the CONSISTENT mass M (P129-136),
  the paper's mass mode applied to the whole operator (SPEC S208);
* noise W = R xi with R the Cholesky factor of M in the natural DOF order, M = R R^T
  (P148-150 "we compute R ... as the Cholesky-decomposition of M"; SPEC S241 "natural mesh
  ordering"), xi the same standard normals as the lumped stream: numpy's dense
  Cholesky (LAPACK) is the library primitive -- small meshes only;
* u = sum_l A_l^{-1} W in ascending l, each node by SuperLU.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
from scipy.sparse.linalg import splu

from . import fem, noise, quadrature
from .mesh import build_mesh


def operator(Mc, G, kappa, c_I, c_L):
    return (c_I * Mc + c_L * (kappa * kappa * Mc + G)).tocsc()


def noise_factor(mesh) -> np.ndarray:
    """Dense lower-triangular R with R R^T = M (consistent), natural DOF order."""
    return np.linalg.cholesky(fem.consistent_mass(mesh).toarray())


def white_noise(mesh, seed, n_samples, samples=None):
    """W_s = R xi_s, xi_s the standard normals of sample s of the SURVEY §8c-N stream."""
    R = noise_factor(mesh)
    samples = range(n_samples) if samples is None else samples
    xi = np.stack([noise.standard_normal(seed, s, np.arange(mesh.n_dofs)) for s in samples])
    return (R @ xi.T).T


def sample(graph, h, kappa, beta, k, seed, n_samples, samples=None):
    mesh = build_mesh(graph, h)
    Mc = fem.consistent_mass(mesh)
    G = fem.stiffness(mesh)
    plan = quadrature.plan(beta, k)
    W = white_noise(mesh, seed, n_samples, samples)
    u = np.zeros_like(W)
    for li in range(plan.n_nodes):
        A = operator(Mc, G, kappa, plan.c_I[li], plan.c_L[li])
        u = u + splu(A).solve(np.ascontiguousarray(W.T)).T
    return u, W
