"""Host scalar special functions needed for per-state constants.

Restates /root/reference/pkg/src/loghmm/special.py:70-73 (log_gamma via
math.lgamma) and :131-202 (two-branch A&S Bessel I0 and log I0) so the host
can compute the von Mises normaliser exactly as the reference does.  The
device ports used by the M-step kernels live in csrc/hmm_mstep.cuh.
"""

from __future__ import annotations

import math

__all__ = ["log_gamma", "log_bessel_i0"]

_BESSEL_BRANCH = 3.75
_I0_SMALL = (1.0, 3.5156229, 3.0899424, 1.2067492, 0.2659732, 0.0360768, 0.0045813)
_I0_LARGE = (
    0.39894228,
    0.01328592,
    0.00225319,
    -0.00157565,
    0.00916281,
    -0.02057706,
    0.02635537,
    -0.01647633,
    0.00392377,
)


def _horner(coeffs, u: float) -> float:
    acc = 0.0
    for c in reversed(coeffs):
        acc = acc * u + c
    return acc


def log_gamma(x: float) -> float:
    if math.isnan(x) or x <= 0.0:
        raise ValueError(f"log_gamma requires a positive argument, got {x}")
    return math.lgamma(x)


def log_bessel_i0(x: float) -> float:
    """log I0(x), x >= 0 (special.py:195-202)."""
    if math.isnan(x) or x < 0.0:
        raise ValueError(f"log_bessel_i0 requires a non-negative argument, got {x}")
    if x <= _BESSEL_BRANCH:
        t2 = (x / _BESSEL_BRANCH) ** 2
        return math.log(_horner(_I0_SMALL, t2))
    u = _BESSEL_BRANCH / x
    return x - 0.5 * math.log(x) + math.log(_horner(_I0_LARGE, u))
