"""Centering and PCA whitening, oracle side (TEST INFRASTRUCTURE ONLY; float64).

The paper whitens "in advance" without saying how.
Readings A11/A12:
  * centre each row (Theorem 1 constraint sum_m y_im = 0);
  * covariance C = Xc Xc^T / M (divisor M, as in eq. (2));
  * symmetric eigendecomposition C = E D E^T, eigenvalues DESCENDING,
    each eigenvector's largest-|entry| made positive (ties -> lowest index);
  * V = D^{-1/2} E^T,  Xw = V Xc;
  * RankDeficient if any eigenvalue < eig_floor * max eigenvalue.
"""
from __future__ import annotations

import numpy as np


class RankDeficient(ValueError):
    pass


def center(X):
    X = np.asarray(X, dtype=np.float64)
    mean = X.mean(axis=1)
    return X - mean[:, None], mean


def whiten(X, eig_floor: float = 1e-12):
    """Return (Xw, mean, V, eigenvalues) with Xw = V (X - mean)."""
    Xc, mean = center(X)
    M = Xc.shape[1]
    C = (Xc @ Xc.T) / M
    C = 0.5 * (C + C.T)
    d, E = np.linalg.eigh(C)
    order = np.argsort(-d, kind="stable")
    d, E = d[order], E[:, order]
    if d[-1] < eig_floor * d[0] or d[-1] <= 0:
        raise RankDeficient(f"covariance eigenvalue {d[-1]:.3e} below floor {eig_floor:.1e} * {d[0]:.3e}")
    for k in range(E.shape[1]):
        j = int(np.argmax(np.abs(E[:, k])))
        if E[j, k] < 0:
            E[:, k] = -E[:, k]
    V = (E / np.sqrt(d)).T
    return V @ Xc, mean, V, d
