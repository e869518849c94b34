"""Evaluation measures (oracle, TEST INFRASTRUCTURE ONLY; float64).

    cosine divergence  delta = 1 - |S_cos(u, v)|         PAPER.md:371-377 (§4.3)
    fluctuation = mean delta over the T(T-1) ordered run pairs
    ordering error  E = ||W A - I||_0 / N^2              PAPER.md:307-309 (§4.2), tau-thresholded
    row Amari index (reading A23, north_star "Amari index ~ 0 on easy cases")
"""
from __future__ import annotations

import itertools

import numpy as np


def cosine_divergence(u, v) -> float:
    u = np.asarray(u, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    nu, nv = np.linalg.norm(u), np.linalg.norm(v)
    if nu == 0 or nv == 0:
        raise ValueError("zero vector")
    return float(1.0 - abs(u @ v) / (nu * nv))


def fluctuation(runs):
    """Per-component mean of delta(i,t,u) over all ordered pairs t != u."""
    runs = [np.asarray(r, dtype=np.float64) for r in runs]
    T = len(runs)
    n = runs[0].shape[0]
    out = np.zeros(n)
    for t, u in itertools.permutations(range(T), 2):
        for i in range(n):
            out[i] += cosine_divergence(runs[t][i], runs[u][i])
    return out / (T * (T - 1))


def ordering_error(W, A, tau: float = 0.1) -> float:
    """||P - I||_0 / N^2 with P = W A after per-row sign disambiguation."""
    P = np.asarray(W, dtype=np.float64) @ np.asarray(A, dtype=np.float64)
    for r in range(P.shape[0]):
        j = int(np.argmax(np.abs(P[r])))
        if P[r, j] < 0:
            P[r] = -P[r]
    N = P.shape[1]
    return float(np.count_nonzero(np.abs(P - np.eye(P.shape[0], N)) > tau)) / (P.shape[0] * N)


def amari_rows(P) -> float:
    """Row Amari index of the k x N loading matrix P (0 iff each row has one nonzero)."""
    P = np.abs(np.asarray(P, dtype=np.float64))
    k, N = P.shape
    if N < 2:
        return 0.0
    return float(np.sum(P.sum(axis=1) / P.max(axis=1) - 1.0) / (k * (N - 1)))
