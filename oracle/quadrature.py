"""Oracle quadrature plan (PAPER.md P54-67 [eq:coefficients], P335).

K^- = ceil(pi^2 / (4 k^2 beta)),  K^+ = ceil(pi^2 / (4 k^2 (1 - beta)))   (P335)
l = -K^-, ..., K^+ ascending, y_l = l k                  (P58)
c_const = pi / (2 k sin(pi beta)),  c_I = c_const e^{-2 beta y_l},
c_L = c_I e^{2 y_l}                                                       (P61-65)
L^{-beta} ~= sum_l (c_I I + c_L L)^{-1}                                   (P67)

The survey (§8c Q1) reads eq. [balakrishnan_quadrature] (P56) as a typo; the
coefficient form above is the one used everywhere.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np


@dataclasses.dataclass
class Plan:
    beta: float
    k: float
    K_minus: int
    K_plus: int
    l: np.ndarray
    y: np.ndarray
    c_const: float
    c_I: np.ndarray
    c_L: np.ndarray

    @property
    def n_nodes(self):
        return len(self.l)


def limits(beta: float, k: float):
    Km = math.ceil((math.pi * math.pi) / (4.0 * k * k * beta))
    Kp = math.ceil((math.pi * math.pi) / (4.0 * k * k * (1.0 - beta)))
    return Km, Kp


def plan(beta: float, k: float) -> Plan:
    if not (0.25 < beta < 1.0):
        raise ValueError("beta must lie in (1/4, 1) (P47)")
    if not (k > 0):
        raise ValueError("k must be positive")
    Km, Kp = limits(beta, k)
    l = np.arange(-Km, Kp + 1, dtype=np.int64)
    y = l * k
    c_const = math.pi / (2.0 * k * math.sin(math.pi * beta))
    c_I = np.array([c_const * math.exp(-2.0 * beta * yy) for yy in y])
    c_L = np.array([ci * math.exp(2.0 * yy) for ci, yy in zip(c_I, y)])
    return Plan(beta, k, Km, Kp, l, y, c_const, c_I, c_L)


def k_from_h(beta: float, h: float) -> float:
    """k = -1 / (beta ln h) (P335)."""
    return -1.0 / (beta * math.log(h))


def sinc_scalar(lam, p: Plan):
    """Q_k(lambda) = sum_l 1 / (c_I + c_L lambda), the scalar form of P67."""
    lam = np.asarray(lam, dtype=np.float64)
    out = np.zeros_like(lam)
    for ci, cl in zip(p.c_I, p.c_L):
        out = out + 1.0 / (ci + cl * lam)
    return out
