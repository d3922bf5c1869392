"""OLS rate fit  ln err = c + r ln h  (PAPER.md P335; SPEC S497-505)."""
from __future__ import annotations

import numpy as np


def fit_rate(h, err):
    """Return (r, c) of the least-squares line ln err = c + r ln h."""
    h = np.asarray(h, dtype=np.float64)
    err = np.asarray(err, dtype=np.float64)
    if len(h) < 2 or len(h) != len(err) or np.any(h <= 0) or np.any(err <= 0):
        raise ValueError("fit_rate needs >= 2 positive (h, err) pairs")
    x = np.log(h)
    y = np.log(err)
    xm, ym = x.mean(), y.mean()
    r = ((x - xm) * (y - ym)).sum() / ((x - xm) ** 2).sum()
    return r, ym - r * xm
