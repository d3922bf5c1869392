"""Pins for oracle/dd.py: the DD DEFINITIONS against closed forms and the direct solve.

* local Schur block == SURVEY §7.4 closed form (sinh ratios), and its h->0 limit
  is the continuum Dirichlet-to-Neumann map with O(h^2) error (ratio 4 per halving)
* sum_e R_e^T S_e R_e == global Schur complement (P242-244: grad J_1 == grad J)
* paper-literal Neumann step (local full-edge solve of eq:neumann_block, P266-292)
  == S_e^{-1} r~  (P298 identity)
* condense -> Schur solve -> recover == direct per-node solve (P111-118, P300-311)
* single edge: NN-PCG converges in exactly 1 iteration (SPEC S399, S534)
"""
import math

import numpy as np
import pytest

from oracle import dd, fem, noise, solve
from synth import MetricGraph, lattice, single_edge, star_of_lattices, tadpole


def _closed_form_schur(a, b, m):
    beta = -b
    rho = a / beta
    th = math.acosh(rho / 2.0)
    q = math.exp(-th)
    den = 1.0 - q ** (2 * (m + 1))
    r1 = q * (1.0 - q ** (2 * m)) / den                 # sinh(m th)/sinh((m+1) th)
    r2 = q ** m * (1.0 - q * q) / den                   # sinh(th)/sinh((m+1) th)
    return a / 2.0 - beta * r1, -beta * r2


@pytest.mark.parametrize("ell,h", [(1.0, 0.01), (0.73, 0.05), (0.02, 0.01), (0.005, 0.01), (1.3, 0.3)])
def test_local_schur_closed_form(ell, h):
    prob = solve.setup(single_edge(ell), h, 3.0, 0.7, 0.4)
    m = int(prob.mesh.m_int[0])
    for li in range(0, prob.plan.n_nodes, max(1, prob.plan.n_nodes // 9)):
        a, b, share = dd.edge_coefficients(prob, li, 0)
        S = dd.local_schur(prob, li, 0)
        sd, so = _closed_form_schur(a, b, m)
        assert abs(S[0, 0] - sd) <= 1e-12 * abs(sd) and abs(S[1, 1] - sd) <= 1e-12 * abs(sd)
        assert abs(S[0, 1] - so) <= 1e-12 * abs(sd) and abs(S[0, 1] - S[1, 0]) <= 1e-12 * abs(sd)
        assert share == a / 2.0


def test_schur_dtn_limit_second_order():
    """S_e / c_L -> k_t [[coth k_t l, -csch k_t l], ...], k_t^2 = kappa^2 + c_I/c_L; error O(h^2)."""
    kappa, ell = 2.0, 0.7
    errs = []
    for h in (0.05, 0.025, 0.0125):
        prob = solve.setup(single_edge(ell), h, kappa, 0.7, 0.4)
        li = prob.plan.n_nodes // 2
        cI, cL = prob.plan.c_I[li], prob.plan.c_L[li]
        kt = math.sqrt(kappa ** 2 + cI / cL)
        S = dd.local_schur(prob, li, 0) / cL
        errs.append(abs(S[0, 0] / (kt / math.tanh(kt * ell)) - 1))
    assert 3.9 < errs[0] / errs[1] < 4.1 and 3.9 < errs[1] / errs[2] < 4.1


@pytest.mark.parametrize("graph,h", [(tadpole(), 0.05), (lattice(4, seed=1), 0.1), (star_of_lattices(2, 3), 0.25)])
def test_assembled_schur_is_global_schur(graph, h):
    prob = solve.setup(graph, h, 3.0, 0.65, 0.35)
    for li in (0, prob.plan.n_nodes // 3, prob.plan.n_nodes - 1):
        Sg = dd.global_schur(prob, li)
        Sa = dd.assembled_schur(prob, li)
        assert np.abs(Sg - Sa).max() <= 1e-12 * np.abs(Sg).max()
        assert np.allclose(Sg, Sg.T, rtol=0, atol=1e-13 * np.abs(Sg).max())
        assert np.linalg.eigvalsh(Sg).min() > 0


def test_neumann_step_is_inverse_local_schur():
    """Solve [A_II A_IG; A_GI A_GG][d_I; d_G] = [0; r~] on the full edge (eq:neumann_block) -> d_G = S_e^{-1} r~."""
    prob = solve.setup(single_edge(0.9), 0.1, 2.0, 0.6, 0.3)
    rng = np.random.default_rng(0)
    for li in range(0, prob.plan.n_nodes, 7):
        a, b, share = dd.edge_coefficients(prob, li, 0)
        m = int(prob.mesh.m_int[0])
        n = m + 2   # local order [v_left, interior..., v_right] = P A P^T (P269-292), tridiagonal
        T = np.diag(np.full(n, a)) + np.diag(np.full(n - 1, b), 1) + np.diag(np.full(n - 1, b), -1)
        T[0, 0] = T[-1, -1] = share
        r = rng.standard_normal(2)
        rhs = np.zeros(n)
        rhs[0], rhs[-1] = r
        d = np.linalg.solve(T, rhs)
        ref = np.linalg.solve(dd.local_schur(prob, li, 0), r)
        assert np.allclose([d[0], d[-1]], ref, rtol=1e-11, atol=0)


@pytest.mark.parametrize("graph,h,kappa", [(tadpole(), 0.01, 5.0), (lattice(4, seed=1), 0.05, 2.0),
                                           (MetricGraph(3, np.array([0, 0, 1]), np.array([1, 1, 2]),
                                                        np.array([0.5, 0.8, 0.004])), 0.01, 1.0)])
def test_condense_pcg_recover_equals_direct(graph, h, kappa):
    prob = solve.setup(graph, h, kappa, 0.7, 0.4)
    W = noise.white_noise(prob.ML, 2, 1)
    NI = prob.mesh.n_interior
    for li in (0, prob.plan.n_nodes // 2, prob.plan.n_nodes - 1):
        x = solve.node_solve(prob, li, W)[0]
        S = dd.assembled_schur(prob, li)
        g = dd.condensed_rhs(prob, li, W)[0]
        uG, it = dd.pcg(S, g, dd.nn_preconditioner(prob, li), rtol=1e-13)
        uI = dd.recover_interior(prob, li, W, uG)[0]
        xdd = np.concatenate([uI, uG])
        assert np.linalg.norm(xdd - x) <= 1e-11 * np.linalg.norm(x)
        assert it <= prob.mesh.n_vertices + 1


def test_single_edge_pcg_one_iteration():
    for ell, h in ((1.0, 0.01), (0.3, 0.05), (0.01, 0.05)):
        prob = solve.setup(single_edge(ell), h, 2.0, 0.8, 0.3)
        W = noise.white_noise(prob.ML, 0, 1)
        for li in range(0, prob.plan.n_nodes, 5):
            S = dd.assembled_schur(prob, li)
            g = dd.condensed_rhs(prob, li, W)[0]
            x, it = dd.pcg(S, g, dd.nn_preconditioner(prob, li), max_iter=1)
            # exact after one step; in fp64 the residual is at the cond(S) * eps rounding level
            res = np.linalg.norm(S @ x - g) / np.linalg.norm(g)
            assert res <= 50 * np.finfo(float).eps * np.linalg.cond(S)
            if np.linalg.cond(S) < 100:
                assert dd.pcg(S, g, dd.nn_preconditioner(prob, li))[1] == 1


def test_tadpole_pcg_at_most_two():
    prob = solve.setup(tadpole(), 0.01, 5.0, 0.75, 0.5)
    W = noise.white_noise(prob.ML, 0, 1)
    for li in range(prob.plan.n_nodes):
        S = dd.assembled_schur(prob, li)
        _, it = dd.pcg(S, dd.condensed_rhs(prob, li, W)[0], dd.nn_preconditioner(prob, li))
        assert it <= 2
