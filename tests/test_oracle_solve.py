"""Pins for oracle/solve.py + oracle/spectral.py (PAPER.md P67-78, P313-324; SURVEY App. A.2, §8c pin table).

* single edge: closed-form DCT eigen-expansion of the lumped P1 Neumann pencil (no matrix assembled)
* tadpole: dense generalized-eigen oracle vs sparse LU path (different LAPACK/SuperLU routes)
* quadrature gap to the exact discrete L_h^{-beta} shrinks like e^{-pi^2/(2k)}
* Kirchhoff vertex rows of each node's solution, evaluated by walking the mesh (P155-158, P38)
* Matern variance of the exact discrete field vs the R closed form
"""
import math

import numpy as np
import pytest

from oracle import fem, noise, quadrature, solve, spectral
from oracle.mesh import build_mesh
from synth import lattice, single_edge, tadpole


def _single_edge_closed_form(ell, h, kappa, plan, W):
    """u = sum_j Q_k(lam_j) phi_j (phi_j^T W) / ||phi_j||_M^2, phi_j(x_i) = cos(j pi i / n)."""
    n = math.ceil(ell / h)
    he = ell / n
    i = np.arange(n + 1)
    # canonical DOF order: interior nodes i=1..n-1, then vertex u (i=0), vertex v (i=n)
    order = np.concatenate([np.arange(1, n), [0, n]])
    mass = np.full(n + 1, he)
    mass[0] = mass[n] = he / 2
    u = np.zeros_like(W)
    for j in range(n + 1):
        phi = np.cos(j * math.pi * i / n)
        lam = kappa ** 2 + (4.0 / he ** 2) * math.sin(j * math.pi / (2 * n)) ** 2
        q = quadrature.sinc_scalar(lam, plan)
        nrm = (mass * phi * phi).sum()
        ph = phi[order]
        u += q * np.outer(W @ ph, ph) / nrm
    return u


@pytest.mark.parametrize("ell,h,kappa,beta,k", [(1.0, 0.05, 3.0, 0.75, 0.4), (2.3, 0.1, 1.0, 0.35, 0.3),
                                                (0.7, 0.01, 10.0, 0.6, 0.25)])
def test_single_edge_closed_form(ell, h, kappa, beta, k):
    u, W, prob = solve.sample(single_edge(ell), h, kappa, beta, k, seed=3, n_samples=2)
    ref = _single_edge_closed_form(ell, h, kappa, prob.plan, W)
    assert np.linalg.norm(u - ref) / np.linalg.norm(ref) < 1e-11


def test_tadpole_spectral_oracle():
    g = tadpole()
    mesh, ML, lam, Q = spectral.decompose(g, 0.01, 5.0)
    p = quadrature.plan(0.75, 0.5)
    W = noise.white_noise(ML, 0, 1)
    u, _, _ = solve.sample(g, 0.01, 5.0, 0.75, 0.5, seed=0, n_samples=1)
    us = spectral.apply_quadrature(ML, lam, Q, p, W)
    assert np.linalg.norm(u - us) / np.linalg.norm(us) < 1e-11
    assert lam.min() > 25.0 - 1e-9 and abs(lam.min() - 25.0) < 1e-8   # constant mode: lambda = kappa^2


def test_quadrature_gap_to_exact_fractional_power():
    g = tadpole()
    mesh, ML, lam, Q = spectral.decompose(g, 0.01, 5.0)
    W = noise.white_noise(ML, 0, 1)
    ue = spectral.apply_exact(ML, lam, Q, 0.75, W)

    def gap(k):
        uq = spectral.apply_quadrature(ML, lam, Q, quadrature.plan(0.75, k), W)
        d = uq - ue
        return math.sqrt((d * d * ML).sum() / (ue * ue * ML).sum())

    g5, g2 = gap(0.5), gap(0.2)
    assert 1e-5 < g5 < 2e-3      # ~4.9e-4 expected at k = 0.5
    assert g2 < 1e-8             # ~3.5e-10 expected at k = 0.2
    # the gap is delta(lam) = Q_k(lam) - lam^{-beta} applied spectrally, bounded by its max ratio
    p = quadrature.plan(0.75, 0.5)
    ratio = np.abs(quadrature.sinc_scalar(lam, p) * lam ** 0.75 - 1).max()
    assert g5 <= ratio * (1 + 1e-9)


def test_matern_variance():
    """E||u||_M^2 / |Gamma| = sum lam^{-2 beta} / |Gamma| ~ R Matern variance (SURVEY §8c Statistics)."""
    kappa, beta = 5.0, 0.75
    mesh, ML, lam, Q = spectral.decompose(tadpole(), 0.01, kappa)
    v = (lam ** (-2 * beta)).sum() / 3.0
    sigma2 = math.gamma(2 * beta - 0.5) / (math.gamma(2 * beta) * math.sqrt(4 * math.pi) * kappa ** (4 * beta - 1))
    assert abs(v / sigma2 - 1) < 0.01
    assert abs(v - 0.012748) < 5e-6


@pytest.mark.parametrize("graph,h", [(tadpole(), 0.01), (lattice(4, seed=1), 0.05)])
def test_node_solution_kirchhoff_rows(graph, h):
    """Vertex rows: (c_I + kappa^2 c_L) M_vv x_v + c_L sum_{(e,end) at v} (x_v - x_adj)/h_e = W_v."""
    kappa = 4.0
    prob = solve.setup(graph, h, kappa, 0.6, 0.3)
    mesh = prob.mesh
    W = noise.white_noise(prob.ML, 1, 1)
    for li in (0, prob.plan.n_nodes // 2, prob.plan.n_nodes - 1):
        cI, cL = prob.plan.c_I[li], prob.plan.c_L[li]
        x = solve.node_solve(prob, li, W)[0]
        lhs = (cI + kappa ** 2 * cL) * prob.ML[mesh.n_interior:] * x[mesh.n_interior:]
        for e in range(mesh.n_edges):
            n = int(mesh.n_el[e])
            for end, v in ((0, int(mesh.edge_u[e])), (1, int(mesh.edge_v[e]))):
                adj = mesh.node(e, 1 if end == 0 else n - 1)
                lhs[v] += cL * (x[mesh.vertex_dof(v)] - x[adj]) / mesh.h_e[e]
        rhs = W[0, mesh.n_interior:]
        scale = np.abs(rhs).max()
        assert np.abs(lhs - rhs).max() < 1e-10 * scale


def test_node_residuals_small():
    prob = solve.setup(lattice(6, seed=2), 0.02, 10.0, 0.6, 0.2)
    W = noise.white_noise(prob.ML, 0, 2)
    _, res = solve.apply(prob, W, return_residuals=True)
    assert res.max() < 1e-12


def test_sample_subset_consistency():
    """Sample j computed alone (samples=[j]) equals row j of the full call (counter-based noise)."""
    g = lattice(3, seed=4)
    u, W, _ = solve.sample(g, 0.1, 2.0, 0.55, 0.3, seed=5, n_samples=4)
    u2, W2, _ = solve.sample(g, 0.1, 2.0, 0.55, 0.3, seed=5, n_samples=4, samples=[2])
    assert np.array_equal(W[2], W2[0])
    assert np.allclose(u[2], u2[0], rtol=0, atol=0)
