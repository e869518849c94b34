"""O3 -- Algorithm 2 literally, with the §3.3 reduction of X (oracle, TEST INFRASTRUCTURE ONLY).

PAPER.md:195-215 and :220-268, float64:
    F = I_N - W^T W                         (:199, :229)
    F~ = first N-i+1 rows of F              (:203, :230)
    G = (F~ F~^T)^{-1/2} F~                 (:206, :231)
    X~ = G X                                (:210, :232)
    B random L x (N-i+1), rows normalised   (:237-239)
    do: B_prev = B; Z = B X~; B = (Z o Z o Z) X~^T / M - 3 B; per-row normalise,
        converged rows move to B_conv       (:241-256; A1/A2 reading)
    Z = B_conv X~; alpha; p = argmax Upsilon (:257-259)
    W <- [W; b_p G]                         (:264)
Reading A9: the initial rows are b0 = G r / ||G r|| for the same N-dim draw r
used by O1 (then G^T b0 = P r / ||P r||: identical trajectories).
Reading A20: if F~ F~^T is singular (SPEC.md:245 worked example), the rows of F
are chosen by greedy pivoting on residual norm instead of taking the first ones.
"""
from __future__ import annotations

import numpy as np

from . import rng
from .contrast import gaussianity_threshold
from .ordering import DEGENERATE_NORM, AllCandidatesDegenerate, ComponentResult, alpha_rows, convergence_distance
from .select import canonical_sign, select


class IllConditionedComplement(ValueError):
    pass


def sym_inv_sqrt(S, floor: float = 1e-10):
    """R = S^{-1/2} for symmetric positive definite S."""
    S = 0.5 * (np.asarray(S, dtype=np.float64) + np.asarray(S, dtype=np.float64).T)
    d, U = np.linalg.eigh(S)
    if d.min() < floor:
        raise IllConditionedComplement(f"min eigenvalue {d.min():.3e} < {floor:.1e}")
    return (U / np.sqrt(d)) @ U.T


def _pivot_rows(F, k):
    """Greedy pivoted choice of k rows of F spanning its row space (A20 fallback)."""
    R = F.copy()
    chosen = []
    for _ in range(k):
        norms = np.linalg.norm(R, axis=1)
        norms[chosen] = -1.0
        j = int(np.argmax(norms))
        chosen.append(j)
        v = R[j] / norms[j]
        R = R - np.outer(R @ v, v)
    return sorted(chosen)


def complement_basis(W, N: int, floor: float = 1e-10):
    """G ((N-i+1) x N) with G G^T = I, G W^T = 0, G^T G = I - W^T W."""
    W = np.asarray(W, dtype=np.float64).reshape(-1, N)
    if W.shape[0] == 0:
        return np.eye(N)                                   # :234-235
    F = np.eye(N) - W.T @ W                                # :229
    d = N - W.shape[0]
    Ft = F[:d]                                             # :230 delete bottom i-1 rows
    try:
        return sym_inv_sqrt(Ft @ Ft.T, floor) @ Ft         # :231
    except IllConditionedComplement:
        Ft = F[_pivot_rows(F, d)]
        return sym_inv_sqrt(Ft @ Ft.T, floor) @ Ft


def ordering_ica_fast_reduced(X, L, K, tol, N_out, seed, include_unconverged=False,
                              stop_on_gaussianity=False, raw_argmax=False, block=8192, trajectories=None):
    X = np.asarray(X, dtype=np.float64)
    N, M = X.shape
    W = np.zeros((0, N))
    results = []
    ids = np.arange(L)
    for i in range(1, N_out + 1):                           # :227
        G = complement_basis(W, N)                          # :228-236
        Xr = G @ X                                          # :232
        R = rng.candidates(seed, i, ids, N)
        B = R @ G.T                                         # :237 (A9: b0 = G r)
        nrm = np.linalg.norm(B, axis=1)
        deg = nrm < DEGENERATE_NORM
        B = B / np.where(deg, 1.0, nrm)[:, None]            # :239
        conv = np.zeros(L, dtype=bool)
        its = np.zeros(L, dtype=np.int64)
        active = np.nonzero(~deg)[0]
        t = 0
        sum_active = 0
        traj = [] if trajectories is not None else None
        while active.size:                                  # :241 do
            Bp = B[active]                                  # :242
            sum_active += active.size
            Z = np.zeros((active.size, Xr.shape[0]))
            for m0 in range(0, M, block):
                Xb = Xr[:, m0:m0 + block]
                Zb = Bp @ Xb                                # :243
                Z += (Xb @ (Zb * Zb * Zb).T).T              # :244
            Bn = Z / M - 3.0 * Bp                           # :245
            n = np.linalg.norm(Bn, axis=1)
            dg = n < DEGENERATE_NORM
            Bn = Bn / np.where(dg, 1.0, n)[:, None]         # :247
            t += 1                                          # :255
            d = convergence_distance(Bn, Bp)               # :249-250 (A2)
            c = (d <= tol) & ~dg
            B[active[~dg]] = Bn[~dg]
            its[active] = t
            conv[active[c]] = True                          # :251-252
            deg[active[dg]] = True
            if traj is not None:
                traj.append((active.copy(), Bn @ G))
            active = active[~c & ~dg]
            if not t < K:                                   # :256
                break
        if trajectories is not None:
            trajectories.append(traj)
        if deg.all():
            raise AllCandidatesDegenerate(f"component {i}")
        elig = conv | (~deg if include_unconverged else False)
        no_conv = not elig.any()
        if no_conv:
            elig = ~deg
        e = np.nonzero(elig)[0]
        alpha = alpha_rows(B[e], Xr, block)                 # :257-258
        Wfull = B[e] @ G                                    # rows b G (full coordinates)
        s = select(ids[e], Wfull, alpha, raw_argmax=raw_argmax)   # :259 (+A6)
        q = e[s["q"]]
        res = ComponentResult(
            i=i, w=canonical_sign(B[q] @ G), alpha=s["alpha_q"], upsilon=s["upsilon_q"], index=int(ids[q]),
            p=s["id_p"], cluster_size=s["cluster_size"], iters=int(its[q]), n_converged=int(conv.sum()),
            n_unconverged=int(L - conv.sum() - deg.sum()), n_degenerate=int(deg.sum()), n_domain=s["n_domain"],
            gaussian_flag=bool(s["upsilon_q"] < gaussianity_threshold(N, i, M)), near_tie=s["near_tie"],
            no_converged=no_conv, sum_active=sum_active, n_iter=t)
        results.append(res)
        if stop_on_gaussianity and res.gaussian_flag:       # :260-262
            res.stopped = True
            break
        W = np.vstack([W, res.w[None, :]])                  # :264
    return W, results
