"""Pins for oracle/quadrature.py (PAPER.md P50-67, P335; SPEC S304-306, S318, S530)."""
import math

import numpy as np
import pytest
from scipy import integrate

from oracle import quadrature


def test_spec_plan_example():
    k = quadrature.k_from_h(0.5, 2.0 ** -4)            # S304
    assert abs(k - 0.72135) < 1e-5
    p = quadrature.plan(0.5, k)
    assert p.K_minus == 10 and p.K_plus == 10
    p = quadrature.plan(0.5, 1.0)                       # S305
    i0 = int(np.where(p.l == 0)[0][0])
    assert math.isclose(p.c_const, math.pi / 2, rel_tol=1e-15)
    assert p.c_I[i0] == p.c_const and p.c_L[i0] == p.c_const
    p = quadrature.plan(0.875, quadrature.k_from_h(0.875, 2.0 ** -4))   # S306
    assert abs(p.K_plus / p.K_minus - 7.0) < 0.5


@pytest.mark.parametrize("beta,k,L", [(0.75, 0.5, 55), (0.6, 0.2, 259), (0.75, 0.25, 212), (0.55, 0.3, 112),
                                      (0.3, 0.2, 296), (0.5, 0.2, 249), (0.75, 0.2, 331), (0.9, 0.2, 687)])
def test_config_node_counts(beta, k, L):
    """L = K^- + K^+ + 1; cfg2's 259 is BASELINE.json's "~259 quadrature nodes"."""
    assert quadrature.plan(beta, k).n_nodes == L


def test_coefficient_identities():
    p = quadrature.plan(0.6, 0.2)
    assert np.allclose(p.y, p.l * 0.2)
    assert np.allclose(p.c_L / p.c_I, np.exp(2 * p.y), rtol=1e-14)
    assert np.allclose(p.c_I * np.exp(2 * 0.6 * p.y), p.c_const, rtol=1e-13)


@pytest.mark.parametrize("beta", [3 / 8, 4 / 8, 5 / 8, 6 / 8, 7 / 8])
def test_scalar_sinc_rule(beta):
    """sum_l (c_I + c_L lam)^{-1} -> lam^{-beta}; < 1e-4 at k=0.2 (SPEC S318/S530); error ~ e^{-pi^2/(2k)}."""
    lam = np.array([1.0, 10.0, 100.0])
    e2 = np.abs(quadrature.sinc_scalar(lam, quadrature.plan(beta, 0.2)) / lam ** (-beta) - 1)
    assert e2.max() < 1e-4
    e5 = np.abs(quadrature.sinc_scalar(lam, quadrature.plan(beta, 0.5)) / lam ** (-beta) - 1)
    # exponential convergence: ratio of errors tracks e^{-pi^2/(2k)} (orders of magnitude)
    assert e2.max() < 1e-3 * e5.max()


def test_balakrishnan_integral_closed_form():
    """P52: sin(pi b)/pi int_0^inf s^{-b} (lam + s)^{-1} ds = lam^{-b}; the sinc sum is its quadrature."""
    beta, lam = 0.6, 7.0
    f = lambda y: math.exp((1 - beta) * y) / (lam + math.exp(y))
    val = integrate.quad(f, -60, 60, limit=400)[0] * math.sin(math.pi * beta) / math.pi
    assert math.isclose(val, lam ** (-beta), rel_tol=1e-9)
    q = quadrature.sinc_scalar(lam, quadrature.plan(beta, 0.1))
    assert math.isclose(q, lam ** (-beta), rel_tol=1e-12)


def test_plan_validation():
    for b in (0.25, 1.0, 0.1):
        with pytest.raises(ValueError):
            quadrature.plan(b, 0.2)
    with pytest.raises(ValueError):
        quadrature.plan(0.5, 0.0)
