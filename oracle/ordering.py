"""O1 -- batched projection form of Fast Ordering ICA (oracle, TEST INFRASTRUCTURE ONLY).

This is the parity reference for the CUDA path.  Plain numpy float64, one step
per line of the paper's Algorithm 2, with the orthonormality
constraint applied by the projection of Algorithm 1 (E = W^T W, w <- w - E w;
PAPER.md:131-135, :150, :158) instead of the §3.3 reduction of X.  The two are
the same iteration (G^T G = I - W^T W; checked against oracle/reduced.py, O3).

Readings used: A1/A2 convergence test d = 1 - |w.w_prev| <= tol,
evaluated as 0.5 ||w - s w_prev||^2 with s = sign(w.w_prev); A3 eq. (5) shape;
A4 unconverged rows excluded by default; A6 cluster selection; A7/A8 fresh
N(0,1) draws per component from oracle/rng.py; A13 domain; A15 alpha at the
final w; A17 canonical sign; A18 degenerate candidates; A19 do-while with t<K.

The M axis is processed in blocks purely to bound memory: the sums are the
plain definitions of eq. (4)-(5) (library matmul per block, blocks summed in
order).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import rng
from .contrast import gaussianity_threshold
from .select import canonical_sign, select

DEGENERATE_NORM = 1e-12


class AllCandidatesDegenerate(RuntimeError):
    pass


@dataclass
class ComponentResult:
    i: int                       # 1-based component index
    w: np.ndarray                # accepted row (canonical sign), N
    alpha: float                 # alpha_q = sum y^4/M - 3 at the final w_q
    upsilon: float               # Upsilon(alpha_q)
    index: int                   # q, global candidate id accepted
    p: int                       # raw argmax id
    cluster_size: int
    iters: int                   # updates applied to candidate q
    n_converged: int
    n_unconverged: int
    n_degenerate: int
    n_domain: int
    gaussian_flag: bool
    near_tie: bool
    no_converged: bool
    sum_active: int              # sum_t L_act(t): rows updated over all iterations
    n_iter: int                  # iterations executed (max t)
    stopped: bool = False        # Gaussianity stop fired (STOP_ON_GAUSSIANITY)

    @property
    def objective(self) -> float:
        return self.alpha + 3.0


@dataclass
class CandidateState:
    """Per-candidate end state of one component (diagnostics / parity)."""
    ids: np.ndarray
    W: np.ndarray
    iters: np.ndarray
    converged: np.ndarray
    degenerate: np.ndarray
    alpha: np.ndarray            # at final w, for eligible rows (nan otherwise)


def project(V: np.ndarray, W_acc: np.ndarray) -> np.ndarray:
    """w <- w - E w with E = W_acc^T W_acc, row-wise."""
    if W_acc.shape[0] == 0:
        return V.copy()
    return V - (V @ W_acc.T) @ W_acc


def batch_step(B: np.ndarray, X: np.ndarray, block: int = 8192):
    """One batched update before normalisation (eq. (4)-(5)).

    Z = B X;  returns (Z o Z o Z) X^T / M - 3 B  and  s4 = sum_m z^4 per row.
    """
    L, M = B.shape[0], X.shape[1]
    G = np.zeros((L, X.shape[0]))
    s4 = np.zeros(L)
    for m0 in range(0, M, block):
        Xb = X[:, m0:m0 + block]
        Z = B @ Xb                      # eq. (4)
        Z2 = Z * Z
        s4 += np.sum(Z2 * Z2, axis=1)
        G += (Xb @ (Z2 * Z).T).T        # eq. (5), accumulated over M ((X Z^3^T)^T: same product)
    return G / M - 3.0 * B, s4


def alpha_rows(B: np.ndarray, X: np.ndarray, block: int = 8192) -> np.ndarray:
    """alpha_l = sum_m z_lm^4 / M - 3 with Z = B X (eq. (2))."""
    M = X.shape[1]
    s4 = np.zeros(B.shape[0])
    for m0 in range(0, M, block):
        Z = B @ X[:, m0:m0 + block]
        Z2 = Z * Z
        s4 += np.sum(Z2 * Z2, axis=1)
    return s4 / M - 3.0


def convergence_distance(Wn: np.ndarray, Wp: np.ndarray) -> np.ndarray:
    """d = 1 - |w . w_prev| for unit rows, as 0.5 ||w - s w_prev||^2 (reading A1/A2)."""
    dot = np.sum(Wn * Wp, axis=1)
    s = np.where(dot < 0, -1.0, 1.0)
    return 0.5 * np.sum((Wn - s[:, None] * Wp) ** 2, axis=1)


def run_component(X, W_acc, i, seed, ids, K, tol, include_unconverged=False, block=8192):
    """Candidate phase of one component: init + do-while."""
    N = X.shape[0]
    R = rng.candidates(seed, i, ids, N)                      # P:237 random matrix
    W0 = project(R, W_acc)                                   # P:150 (A9)
    nrm = np.linalg.norm(W0, axis=1)
    degenerate = nrm < DEGENERATE_NORM                       # A18
    W = W0 / np.where(degenerate, 1.0, nrm)[:, None]         # P:239 normalise
    nL = len(ids)
    iters = np.zeros(nL, dtype=np.int64)
    converged = np.zeros(nL, dtype=bool)
    active = np.nonzero(~degenerate)[0]
    t = 0
    sum_active = 0
    while active.size:                                       # do ...
        Wp = W[active]                                       # P:242 B_prev
        sum_active += active.size
        G, _ = batch_step(Wp, X, block)
        G = project(G, W_acc)                                # P:158 (projection form)
        n = np.linalg.norm(G, axis=1)
        dg = n < DEGENERATE_NORM
        Wn = G / np.where(dg, 1.0, n)[:, None]               # P:247 normalise
        t += 1
        d = convergence_distance(Wn, Wp)                     # P:249-250 (A1/A2)
        c = (d <= tol) & ~dg
        W[active[~dg]] = Wn[~dg]
        iters[active] = t
        converged[active[c]] = True                          # P:251-252 -> B_conv
        degenerate[active[dg]] = True
        active = active[~c & ~dg]
        if not t < K:                                        # ... while t<K and B≠∅
            break
    return W, iters, converged, degenerate, sum_active, t


def select_component(X, W, ids, iters, converged, degenerate, i, include_unconverged=False,
                     raw_argmax=False, block=8192):
    """Alpha of the eligible rows, argmax + cluster rule (A6)."""
    N, M = X.shape
    if degenerate.all():
        raise AllCandidatesDegenerate(f"component {i}: all {len(ids)} candidates degenerate")
    elig = converged.copy()
    if include_unconverged:
        elig |= ~degenerate
    no_conv = not elig.any()
    if no_conv:
        elig = ~degenerate
    e = np.nonzero(elig)[0]
    alpha = np.full(len(ids), np.nan)
    alpha[e] = alpha_rows(W[e], X, block)
    s = select(np.asarray(ids)[e], W[e], alpha[e], raw_argmax=raw_argmax)
    q = e[s["q"]]
    n_conv = int(converged.sum())
    n_deg = int(degenerate.sum())
    res = ComponentResult(
        i=i, w=canonical_sign(W[q]), alpha=s["alpha_q"], upsilon=s["upsilon_q"],
        index=s["id_q"], p=s["id_p"], cluster_size=s["cluster_size"], iters=int(iters[q]),
        n_converged=n_conv, n_unconverged=len(ids) - n_conv - n_deg, n_degenerate=n_deg,
        n_domain=s["n_domain"],
        gaussian_flag=bool(s["upsilon_q"] < gaussianity_threshold(N, i, M)),
        near_tie=s["near_tie"], no_converged=no_conv, sum_active=0, n_iter=0)
    return res, alpha


def extract(X, L, K, tol, N_out, seed, include_unconverged=False, stop_on_gaussianity=False,
            W_prefix=None, raw_argmax=False, ids=None, block=8192, keep_candidates=False):
    """Fast Ordering ICA, projection form (Alg. 2 PAPER.md:220-268 + Alg. 1 E-projection).

    X: N x M whitened data (float64; pass the exact fp32 data upcast).
    Returns (W_acc, [ComponentResult], [CandidateState] if keep_candidates).
    """
    X = np.asarray(X, dtype=np.float64)
    N, M = X.shape
    ids = np.arange(L, dtype=np.int64) if ids is None else np.asarray(ids, dtype=np.int64)
    W_acc = np.zeros((0, N)) if W_prefix is None else np.array(W_prefix, dtype=np.float64).reshape(-1, N)
    results: List[ComponentResult] = []
    states: List[CandidateState] = []
    i = W_acc.shape[0] + 1
    while i <= N_out:
        W, iters, conv, deg, sum_active, t = run_component(X, W_acc, i, seed, ids, K, tol, include_unconverged, block)
        res, alpha = select_component(X, W, ids, iters, conv, deg, i, include_unconverged, raw_argmax, block)
        res.sum_active, res.n_iter = sum_active, t
        if keep_candidates:
            states.append(CandidateState(ids=ids.copy(), W=W, iters=iters, converged=conv, degenerate=deg, alpha=alpha))
        if stop_on_gaussianity and res.gaussian_flag:
            res.stopped = True
            results.append(res)
            break
        results.append(res)
        W_acc = np.vstack([W_acc, res.w[None, :]])
        i += 1
    return (W_acc, results, states) if keep_candidates else (W_acc, results)


def algorithmic_flops(results, N: int, M: int) -> float:
    """F_alg = sum_i sum_t L_act(i,t) (4 N M + 3 M)."""
    return float(sum(r.sum_active for r in results)) * (4.0 * N * M + 3.0 * M)
