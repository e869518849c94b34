"""Selection of the accepted candidate (oracle, TEST INFRASTRUCTURE ONLY; float64).

PAPER.md:142 (Alg. 1) and :259 (Alg. 2): p = argmax_l Upsilon(alpha_l).
Reading A6: many candidates converge onto the same optimum and
their Upsilon differ only by arithmetic noise, so the raw argmax index is not
well defined.  We take
    p = argmax Upsilon (ties -> lowest id),
    C = {l eligible : 1 - |w_l . w_p| <= DELTA_CLUSTER},
    q = min C   (the accepted candidate; its w, alpha, Upsilon are reported),
    near_tie  iff  Upsilon_p - max_{l not in C} Upsilon_l <= NEAR_TIE_REL * Upsilon_p.
Reading A17: the accepted row is sign-canonicalised (largest-|entry| positive,
ties -> lowest index); +-w are the same solution.
Reading A13: alpha <= -2 + 1e-12 is outside eq. (1)'s domain; such candidates
are excluded and counted.
"""
from __future__ import annotations

import numpy as np

from .contrast import DomainError, upsilon_masked

DELTA_CLUSTER = 1e-6
NEAR_TIE_REL = 1e-6


def canonical_sign(w):
    w = np.asarray(w, dtype=np.float64)
    j = int(np.argmax(np.abs(w)))
    return w if w[j] >= 0 else -w


def select(ids, W, alpha, raw_argmax: bool = False):
    ids = np.asarray(ids, dtype=np.int64)
    W = np.asarray(W, dtype=np.float64)
    alpha = np.asarray(alpha, dtype=np.float64)
    ups, ok = upsilon_masked(alpha)
    if not ok.any():
        raise DomainError("no eligible candidate has alpha > -2")
    order = np.lexsort((ids, -ups))
    p = int(order[0])
    cos = np.abs(W @ W[p])
    in_c = ((1.0 - cos) <= DELTA_CLUSTER) & ok
    if raw_argmax:
        q = p
    else:
        cand = np.nonzero(in_c)[0]
        q = int(cand[np.argmin(ids[cand])])
    rest = ups[~in_c & ok]
    second = float(rest.max()) if rest.size else -np.inf
    near_tie = bool(ups[p] - second <= NEAR_TIE_REL * ups[p])
    return dict(q=q, p=p, id_q=int(ids[q]), id_p=int(ids[p]), upsilon_q=float(ups[q]),
                alpha_q=float(alpha[q]), upsilon_p=float(ups[p]), second=second,
                cluster_size=int(in_c.sum()), near_tie=near_tie, n_domain=int((~ok).sum()))
