"""Oracle white noise W = M_L^{1/2} z (PAPER.md P99-109 [eq:wh_def], P150).

With the lumped mass the Cholesky factor R of eq. [wh_def] is the elementwise
square root of the diagonal (P109, P150).  The paper leaves the RNG open (SPEC
S272); the canonical stream below is SURVEY.md §8c-N and DESIGN.md "Noise
stream" -- both sides implement it independently and must agree bit for bit.

Stream, per sample j of a call with base seed sigma and per DOF i (canonical
index, mesh.py):
    key  = (lo32(sigma+j), hi32(sigma+j));  ctr = (lo32(i), hi32(i), 0, 0)
    (x0,x1,x2,x3) = Philox4x32-10(ctr, key)      (Salmon et al. 2011 constants)
    A = (x0 << 21) | (x1 >> 11);  u1 = (A + 1) * 2^-53  in (0, 1]
    B = (x2 << 21) | (x3 >> 11);  u2 = B * 2^-53        in [0, 1)
    z = sqrt(-2 ln_fixed(u1)) * cos2pi_fixed(u2)
    W_i = sqrt(M_L,ii) * z
ln_fixed / cos2pi_fixed are the fixed operation sequences below, built only
from correctly rounded IEEE +, -, *, /, sqrt, floor and frexp, with NO fused
multiply-add -- numpy evaluates each ufunc separately, so nothing contracts.
Series constants are the correctly rounded doubles 1.0/n (n a small integer),
so the only data-dependent division is s = (m-1)/(m+1) in ln_fixed.
"""
from __future__ import annotations

import numpy as np

_M0 = np.uint64(0xD2511F53)
_M1 = np.uint64(0xCD9E8D57)
_W0 = np.uint64(0x9E3779B9)
_W1 = np.uint64(0xBB67AE85)
_MASK = np.uint64(0xFFFFFFFF)
_S32 = np.uint64(32)

LN2 = 0.6931471805599453        # nearest double to ln 2
HALF_PI = 1.5707963267948966    # nearest double to pi/2
SQRT_HALF = 0.7071067811865476  # nearest double to sqrt(1/2)
LN_TERMS = 12                   # atanh series up to s^25/25
TRIG_TERMS = 10                 # Taylor series up to theta^20 / theta^21


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Philox4x32 with 10 rounds.  All args uint64 arrays holding 32-bit words."""
    c0, c1, c2, c3 = (np.asarray(x, dtype=np.uint64) for x in (c0, c1, c2, c3))
    k0 = np.asarray(k0, dtype=np.uint64)
    k1 = np.asarray(k1, dtype=np.uint64)
    for r in range(10):
        p0 = _M0 * c0
        p1 = _M1 * c2
        hi0, lo0 = p0 >> _S32, p0 & _MASK
        hi1, lo1 = p1 >> _S32, p1 & _MASK
        c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
        if r < 9:
            k0 = (k0 + _W0) & _MASK
            k1 = (k1 + _W1) & _MASK
    return c0, c1, c2, c3


def uniforms(x0, x1, x2, x3):
    """53-bit uniforms u1 in (0,1], u2 in [0,1) from one Philox block."""
    A = (x0 << np.uint64(21)) | (x1 >> np.uint64(11))
    B = (x2 << np.uint64(21)) | (x3 >> np.uint64(11))
    u1 = (A + np.uint64(1)).astype(np.float64) * 2.0 ** -53
    u2 = B.astype(np.float64) * 2.0 ** -53
    return u1, u2


def ln_fixed(x):
    """Natural log for x > 0 (normal): exponent split + atanh series.

    x = m 2^e with m in [sqrt(1/2), sqrt(2));  s = (m-1)/(m+1);
    ln m = 2 s (1 + s^2/3 + s^4/5 + ... + s^24/25);  ln x = e ln2 + ln m.
    """
    x = np.asarray(x, dtype=np.float64)
    m, e = np.frexp(x)
    small = m < SQRT_HALF
    m = np.where(small, m * 2.0, m)
    e = np.where(small, e - 1, e).astype(np.float64)
    f = m - 1.0
    s = f / (m + 1.0)
    s2 = s * s
    p = np.full_like(s, 1.0 / (2 * LN_TERMS + 1))
    for j in range(LN_TERMS - 1, -1, -1):
        p = (1.0 / (2 * j + 1)) + s2 * p
    t = s * p
    return e * LN2 + (t + t)


def _cos_poly(t2):
    """cos = 1 - t2/(2*1) (1 - t2/(4*3) (1 - ...)): Horner with reciprocal constants 1/((2j)(2j-1))."""
    p = np.ones_like(t2)
    for j in range(TRIG_TERMS, 0, -1):
        p = 1.0 - (t2 * (1.0 / float((2 * j) * (2 * j - 1)))) * p
    return p


def _sin_poly(t, t2):
    """sin = t (1 - t2/(3*2) (1 - t2/(5*4) (1 - ...))), reciprocal constants 1/((2j+1)(2j))."""
    p = np.ones_like(t2)
    for j in range(TRIG_TERMS, 0, -1):
        p = 1.0 - (t2 * (1.0 / float((2 * j + 1) * (2 * j)))) * p
    return t * p


def cos2pi_fixed(u):
    """cos(2 pi u) for u in [0,1): quadrant split of t = 4u, Taylor on |theta| <= pi/4."""
    u = np.asarray(u, dtype=np.float64)
    t = 4.0 * u
    q = np.floor(t + 0.5)
    f = t - q
    th = f * HALF_PI
    th2 = th * th
    c = _cos_poly(th2)
    s = _sin_poly(th, th2)
    qi = q.astype(np.int64) & 3
    return np.select([qi == 0, qi == 1, qi == 2], [c, -s, -c], s)


def standard_normal(seed: int, sample: int, dofs) -> np.ndarray:
    """z for DOF indices `dofs` of sample `sample` of a call with base seed `seed`."""
    dofs = np.asarray(dofs, dtype=np.uint64)
    key = np.uint64((int(seed) + int(sample)) & 0xFFFFFFFFFFFFFFFF)
    k0 = key & _MASK
    k1 = key >> _S32
    zero = np.zeros_like(dofs)
    x0, x1, x2, x3 = philox4x32_10(dofs & _MASK, dofs >> _S32, zero, zero, k0, k1)
    u1, u2 = uniforms(x0, x1, x2, x3)
    r = np.sqrt(-2.0 * ln_fixed(u1))
    return r * cos2pi_fixed(u2)


def white_noise(ML: np.ndarray, seed: int, n_samples: int, dofs=None, samples=None) -> np.ndarray:
    """W[s, i] = sqrt(M_L,ii) z_{s,i}  ([eq:wh_def], P150).  Returns [n_samples, len(dofs)]."""
    if dofs is None:
        dofs = np.arange(len(ML), dtype=np.int64)
    dofs = np.asarray(dofs, dtype=np.int64)
    if samples is None:
        samples = range(n_samples)
    sq = np.sqrt(ML[dofs])
    return np.stack([sq * standard_normal(seed, j, dofs) for j in samples])
