"""Scalar contrast functions (oracle, TEST INFRASTRUCTURE ONLY; float64).

    alpha = sum_m y_m^4 / M - 3                 PAPER.md:96-99, eq. (2)
    Upsilon(alpha) = alpha - 2 log(alpha/2 + 1)  PAPER.md:90-94, eq. (1) (natural log, A14)
    threshold(N, i, M) = 2 (N-i+2)(N-i+1) / M    PAPER.md:117-120 (Gaussianity test)
"""
from __future__ import annotations

import numpy as np


class DomainError(ValueError):
    """Upsilon undefined: alpha <= -2 (+1e-12), SPEC.md:118 / reading A13."""


ALPHA_FLOOR = -2.0 + 1e-12


def kurtosis_alpha(y, axis=-1):
    y = np.asarray(y, dtype=np.float64)
    M = y.shape[axis]
    return np.sum(y ** 4, axis=axis) / M - 3.0


def upsilon(alpha):
    """Eq. (1).  Raises DomainError when any alpha <= -2 + 1e-12."""
    a = np.asarray(alpha, dtype=np.float64)
    if np.any(a <= ALPHA_FLOOR):
        raise DomainError(f"Upsilon undefined for alpha <= -2: {a.min()}")
    return a - 2.0 * np.log(a / 2.0 + 1.0)


def upsilon_masked(alpha):
    """Eq. (1) with out-of-domain entries mapped to -inf (excluded from argmax, A13)."""
    a = np.asarray(alpha, dtype=np.float64)
    ok = a > ALPHA_FLOOR
    out = np.full(a.shape, -np.inf)
    out[ok] = a[ok] - 2.0 * np.log(a[ok] / 2.0 + 1.0)
    return out, ok


def gaussianity_threshold(N: int, i: int, M: int) -> float:
    """Right-hand side of the Gaussianity test (Alg. 1 :143, Alg. 2 :260)."""
    return 2.0 * (N - i + 2) * (N - i + 1) / M
