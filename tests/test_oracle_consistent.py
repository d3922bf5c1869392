"""Pins of oracle/consistent.py (consistent-mass variant, NEXT-3)."""
import numpy as np
import scipy.linalg as sla

from oracle import consistent, fem, quadrature
from oracle.mesh import build_mesh
from synth import single_edge, tadpole


def test_spec_noise_factor_examples():
    # S245: 1x1 consistent M = (0.04) -> R = (0.2)
    assert np.isclose(np.linalg.cholesky(np.array([[0.04]]))[0, 0], 0.2, rtol=0, atol=1e-16)
    # S246: single edge with 3 interior nodes, h_e = 0.25 -> R R^T = M to 1e-14
    m = build_mesh(single_edge(1.0), 0.25)
    R = consistent.noise_factor(m)
    M = fem.consistent_mass(m).toarray()
    assert np.abs(R @ R.T - M).max() <= 1e-14 and np.allclose(R, np.tril(R))
    # stencil (S181): interior diagonal 2h/3, neighbours h/6
    i = m.node(0, 2)
    assert np.isclose(M[i, i], 2 * 0.25 / 3) and np.isclose(M[i, m.node(0, 1)], 0.25 / 6)


def test_noise_covariance_is_consistent_mass():
    m = build_mesh(tadpole(), 0.25)
    W = consistent.white_noise(m, 3, 20000)
    C = np.cov(W.T)
    M = fem.consistent_mass(m).toarray()
    se = np.sqrt((M.diagonal()[:, None] * M.diagonal()[None, :] + M * M) / 20000)
    assert np.all(np.abs(C - M) <= 5 * se + 1e-15)


def test_field_equals_spectral_quadrature():
    """u = sum_l (c_I M + c_L K)^{-1} W equals the quadrature evaluated on the generalized
    eigenpairs K q = lambda M q (M^-1-orthonormal Q): u = Q Q_k(Lambda) Q^T W (the same rule
    applied spectrally; a dropped term, wrong sign or transposed operand breaks it)."""
    g = tadpole()
    h, kappa, beta, k = 0.1, 5.0, 0.75, 0.5
    m = build_mesh(g, h)
    M = fem.consistent_mass(m).toarray()
    K = kappa * kappa * M + fem.stiffness(m).toarray()
    lam, Q = sla.eigh(K, M)  # Q^T M Q = I
    plan = quadrature.plan(beta, k)
    u, W = consistent.sample(g, h, kappa, beta, k, 1, 2)
    qk = sum(1.0 / (plan.c_I[l] + plan.c_L[l] * lam) for l in range(plan.n_nodes))
    u_spec = (Q @ (qk[:, None] * (Q.T @ W.T))).T
    assert np.abs(u - u_spec).max() <= 1e-11 * np.abs(u_spec).max()
