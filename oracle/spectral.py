"""Dense spectral oracle for tiny graphs.

With M = M_L diagonal, K = kappa^2 M + G and K~ = M^{-1/2} K M^{-1/2} = Q diag(lam) Q^T:

    sum_l (c_I M + c_L K)^{-1} W = M^{-1/2} Q diag(Q_k(lam)) Q^T M^{-1/2} W      (quadrature)
    L_h^{-beta} M^{-1} W        = M^{-1/2} Q diag(lam^{-beta}) Q^T M^{-1/2} W   (exact discrete)

Q_k(lam) = sum_l 1/(c_I + c_L lam) is the scalar sinc rule (PAPER.md P67).  The
eigendecomposition (numpy.linalg.eigh, LAPACK) is a different route from the
sparse LU of solve.py, so agreement pins solve.py; the gap to the exact
fractional power is the quadrature error delta(lam) = Q_k(lam) - lam^{-beta},
which the tests check against its predicted size.
"""
from __future__ import annotations

import numpy as np

from . import fem, quadrature
from .mesh import build_mesh


def decompose(graph, h, kappa):
    mesh = build_mesh(graph, h)
    ML = fem.lumped_mass(mesh)
    G = fem.stiffness(mesh).toarray()
    isq = 1.0 / np.sqrt(ML)
    Kt = (kappa * kappa) * np.eye(len(ML)) + isq[:, None] * G * isq[None, :]
    lam, Q = np.linalg.eigh(Kt)
    return mesh, ML, lam, Q


def apply_quadrature(ML, lam, Q, plan: quadrature.Plan, W):
    isq = 1.0 / np.sqrt(ML)
    f = quadrature.sinc_scalar(lam, plan)
    return ((isq[:, None] * Q) @ (f[:, None] * (Q.T @ (isq[:, None] * W.T)))).T


def apply_exact(ML, lam, Q, beta, W):
    isq = 1.0 / np.sqrt(ML)
    f = lam ** (-beta)
    return ((isq[:, None] * Q) @ (f[:, None] * (Q.T @ (isq[:, None] * W.T)))).T
