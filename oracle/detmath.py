"""Deterministic float64 log / log1p / expm1 built from IEEE +,-,*,/ only.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

The reference evaluates ``np.log`` (inside numpy's exponential draw,
``cache.py:101``) and ``np.log1p``/``np.expm1`` (Eq. 9, ``cache.py:115``) with
the platform libm.  libm and CUDA's libdevice may disagree in the last ulp, so
the build defines these three functions as fixed sequences of correctly
rounded IEEE operations (no FMA).  ``paper_2106_06150_b200/csrc/gns_common.cuh``
evaluates the *same* sequence with ``__dadd_rn``/``__dmul_rn``/``__ddiv_rn``,
which makes GPU and oracle bit-identical by construction; the functions are
checked against numpy's libm to a few ulp in ``tests/test_oracle.py::test_detmath_close_to_libm``.
"""

from __future__ import annotations

from fractions import Fraction
from math import factorial

import numpy as np

LN2_HI = float.fromhex("0x1.62e42fee00000p-1")
LN2_LO = float.fromhex("0x1.a39ef35793c76p-33")
INV_LN2 = float.fromhex("0x1.71547652b82fep+0")
SQRT_HALF = float.fromhex("0x1.6a09e667f3bcdp-1")
ONE_MINUS_1EM15 = 1.0 - 1e-15  # cache.py:115 literal, = 0x1.ffffffffffff7p-1

# atanh-series coefficients 1/(2i+1), correctly rounded
LOG_TERMS = 12
LOG1P_TERMS = 20
ATANH_C = [float(Fraction(1, 2 * i + 1)) for i in range(LOG1P_TERMS)]
# Taylor coefficients 1/n!, n = 1..EXPM1_TERMS, correctly rounded
EXPM1_TERMS = 18
EXP_C = [float(Fraction(1, factorial(n))) for n in range(1, EXPM1_TERMS + 1)]


def _atanh_series(s, nterms):
    """2*s*(1 + z/3 + z^2/5 + ...) with z = s*s, Horner from the top."""
    z = s * s
    p = np.full_like(s, ATANH_C[nterms - 1])
    for i in range(nterms - 2, -1, -1):
        p = p * z + ATANH_C[i]
    return (s * p) * 2.0


def det_log(x):
    """log(x) for positive normal float64 x."""
    x = np.asarray(x, dtype=np.float64)
    f, e = np.frexp(x)                       # x = f * 2^e, f in [0.5, 1)
    small = f < SQRT_HALF
    f = np.where(small, f * 2.0, f)          # exact
    e = np.where(small, e - 1, e).astype(np.float64)
    s = (f - 1.0) / (f + 1.0)
    poly = _atanh_series(s, LOG_TERMS)
    return e * LN2_HI + (e * LN2_LO + poly)


def det_log1p(x):
    """log1p(x) for float64 x in (-1, 0]."""
    x = np.asarray(x, dtype=np.float64)
    near = x > -0.5
    xs = np.where(near, x, 0.0)
    s = xs / (xs + 2.0)
    direct = _atanh_series(s, LOG1P_TERMS)
    u = np.where(near, 1.0, x + 1.0)         # exact for x <= -0.5 (Sterbenz)
    far = det_log(u)
    return np.where(near, direct, far)


def _expm1_taylor(y):
    p = np.full_like(y, EXP_C[EXPM1_TERMS - 1])
    for i in range(EXPM1_TERMS - 2, -1, -1):
        p = p * y + EXP_C[i]
    return y * p


def det_expm1(y):
    """expm1(y) for float64 y <= 0."""
    y = np.asarray(y, dtype=np.float64)
    near = y > -0.5
    tiny = y < -40.0                          # 1 - e^y rounds to 1 exactly
    yn = np.where(near, y, 0.0)
    direct = _expm1_taylor(yn)
    yf = np.where(near | tiny, -1.0, y)
    k = np.rint(yf * INV_LN2)
    r = (yf - k * LN2_HI) - k * LN2_LO
    er = _expm1_taylor(r) + 1.0
    far = np.ldexp(er, k.astype(np.int64)) - 1.0
    return np.where(near, direct, np.where(tiny, -1.0, far))


def inclusion_prob(p, cache_size: int):
    """Eq. 9 ``-expm1(|C| * log1p(-min(p, 1-1e-15)))`` with the p>=1 pin —
    restates ``cache.py:106-117`` with the deterministic transcendental pair."""
    p = np.clip(np.asarray(p, dtype=np.float64), 0.0, 1.0)
    out = -det_expm1(float(cache_size) * det_log1p(-np.minimum(p, ONE_MINUS_1EM15)))
    out = np.where(p >= 1.0, 1.0 if cache_size >= 1 else 0.0, out)
    return float(out) if out.ndim == 0 else out


def det_exp(y):
    """exp(y) for |y| < 700: k = rint(y/ln2), r = y - k ln2 (two-part),
    (expm1_taylor(r) + 1) * 2^k — gns_common.cuh det_exp / oracle/gen.cc."""
    y = np.asarray(y, dtype=np.float64)
    k = np.rint(y * INV_LN2)
    r = (y - k * LN2_HI) - k * LN2_LO
    return np.ldexp(_expm1_taylor(r) + 1.0, k.astype(np.int64))


def det_pow(a, b):
    """a**b = det_exp(b * det_log(a)) for a > 0 (the generator's inverse CDF)."""
    return det_exp(b * det_log(a))
