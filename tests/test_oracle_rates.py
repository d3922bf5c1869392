"""Pins for oracle/rates.py (PAPER.md P335 "ln err = c + r ln h"; Table 1 P443-456)."""
import os

import numpy as np
import pytest

from oracle.rates import fit_rate


def test_exact_power_laws():
    r, c = fit_rate([0.5, 0.25], [0.5, 0.25])          # SPEC S503
    assert abs(r - 1.0) < 1e-12
    h = 2.0 ** -np.arange(2, 7)
    r, c = fit_rate(h, 3.0 * h ** 2)                     # SPEC S504
    assert abs(r - 2.0) < 1e-12 and abs(np.exp(c) - 3.0) < 1e-10


def test_paper_table1_strong_rates(repo_root):
    """The OLS fit of P343-349 reproduces the printed Table 1 strong rates (P450) to 2 decimals."""
    data = np.loadtxt(os.path.join(repo_root, "tests", "golden", "paper_strong_error.txt"), comments="#", skiprows=4)
    printed = [0.26, 0.51, 0.76, 1.00, 1.25]
    for j, p in enumerate(printed):
        r, _ = fit_rate(data[:, 0], data[:, j + 1])
        assert round(r, 2) == pytest.approx(p, abs=1e-9)


def test_invalid_inputs():
    with pytest.raises(ValueError):
        fit_rate([0.5], [0.1])
    with pytest.raises(ValueError):
        fit_rate([0.5, 0.25], [0.1, -1.0])
