"""O2 -- Algorithm 1, Original Ordering ICA, one candidate at a time (oracle, TEST INFRASTRUCTURE ONLY).

Literal transcription of PAPER.md:123-167 (float64, plain loops over l):
the FastICA function with the convergence test read as A1
(sign-invariant, d = 1 - |w.w_prev| <= tol) and the driver loop.
Used on tiny sizes only, to cross-check the batched form O1 row by row.
"""
from __future__ import annotations

import numpy as np

from . import rng
from .contrast import gaussianity_threshold, kurtosis_alpha
from .ordering import DEGENERATE_NORM, AllCandidatesDegenerate, ComponentResult
from .select import canonical_sign, select


class DegenerateCandidate(ValueError):
    pass


def fastica_one_unit(w0, X, E, K, tol, trajectory=None):
    """PAPER.md:149-165.  Returns (w, y, t, converged)."""
    X = np.asarray(X, dtype=np.float64)
    M = X.shape[1]
    w = w0 - E @ w0                                  # :150
    n = np.sqrt(w @ w)
    if n < DEGENERATE_NORM:
        raise DegenerateCandidate("projected initial vector vanishes")
    w = w / n                                        # :151
    t = 0                                            # :152
    converged = False
    while True:                                      # :153 do
        w_prev = w                                   # :154
        y = w @ X                                    # :155
        w = X @ (y * y * y) / M - 3.0 * w            # :156-157
        w = w - E @ w                                # :158
        n = np.sqrt(w @ w)
        if n < DEGENERATE_NORM:
            raise DegenerateCandidate("update vanished")
        w = w / n                                    # :159
        t += 1                                       # :160
        if trajectory is not None:
            trajectory.append(w.copy())
        d = 1.0 - abs(w @ w_prev)
        converged = d <= tol
        if not (t < K and not converged):            # :161-162 (A1)
            break
    y = w @ X                                        # :163
    return w, y, t, converged                        # :164


def ordering_ica_reference(X, L, K, tol, N_out, seed, include_unconverged=False,
                           stop_on_gaussianity=False, raw_argmax=False):
    """Algorithm 1 driver, same eligibility/selection readings as O1."""
    X = np.asarray(X, dtype=np.float64)
    N, M = X.shape
    W_acc = np.zeros((0, N))
    results = []
    for i in range(1, N_out + 1):                    # :130
        E = W_acc.T @ W_acc if i > 1 else np.zeros((N, N))   # :131-135
        R = rng.candidates(seed, i, np.arange(L), N)  # :136-137
        ws, alphas, its, conv, deg = [], [], [], [], []
        for l in range(L):                           # :138
            try:
                w, y, t, c = fastica_one_unit(R[l], X, E, K, tol)   # :139
                ws.append(w); alphas.append(kurtosis_alpha(y)); its.append(t); conv.append(c); deg.append(False)  # :140
            except DegenerateCandidate:
                ws.append(np.zeros(N)); alphas.append(np.nan); its.append(0); conv.append(False); deg.append(True)
        conv, deg = np.array(conv), np.array(deg)
        if deg.all():
            raise AllCandidatesDegenerate(f"component {i}")
        elig = conv | (~deg if include_unconverged else False)
        no_conv = not elig.any()
        if no_conv:
            elig = ~deg
        e = np.nonzero(elig)[0]
        s = select(e, np.array(ws)[e], np.array(alphas)[e], raw_argmax=raw_argmax)   # :142 (+A6)
        q = s["id_q"]
        res = ComponentResult(
            i=i, w=canonical_sign(ws[q]), alpha=s["alpha_q"], upsilon=s["upsilon_q"], index=q,
            p=s["id_p"], cluster_size=s["cluster_size"], iters=its[q], n_converged=int(conv.sum()),
            n_unconverged=int(L - conv.sum() - deg.sum()), n_degenerate=int(deg.sum()), n_domain=s["n_domain"],
            gaussian_flag=bool(s["upsilon_q"] < gaussianity_threshold(N, i, M)), near_tie=s["near_tie"],
            no_converged=no_conv, sum_active=int(np.sum(its)), n_iter=int(np.max(its)))
        results.append(res)
        if stop_on_gaussianity and res.gaussian_flag:   # :143-145
            res.stopped = True
            break
        W_acc = np.vstack([W_acc, res.w[None, :]])   # :146
    return W_acc, results
