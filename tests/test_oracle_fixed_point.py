"""Pins for the one-step update and the convergence test (oracle/ordering.py, oracle/fastica.py).

Pins (not restatements of the formula):
  * brute-force central differences of f(w) = sum_m (w.x_m)^4 / M  -> G + 3w = grad f / 4;
  * algebraic identity w.g = alpha(w) tying G to s4 (a dropped -3w or a wrong 1/M breaks it);
  * fixed-point invariants of converged candidates (g parallel to w, ||g|| = |alpha|);
  * the source-recovery special case;
  * chord / cosine geometry of the convergence test.
"""
import math

import numpy as np
import pytest

import datagen
from datagen import sources as S
from oracle import fastica, ordering, rng, whiten


def _white(cfg_name="p_ragged", M=None):
    cfg = datagen.PARITY[cfg_name]
    ds = datagen.make_dataset(cfg, M=M)
    Xw, _, V, _ = whiten.whiten(ds.X.numpy())
    return cfg, Xw, V, ds


def test_gradient_by_central_differences():
    rng_ = np.random.default_rng(3)
    X = rng_.standard_normal((4, 400)) * np.array([[1.0], [0.5], [2.0], [1.3]])
    M = X.shape[1]

    def f(w):                                   # brute force, sample by sample
        tot = 0.0
        for m in range(M):
            y = sum(w[n] * X[n, m] for n in range(4))
            tot += y ** 4
        return tot / M

    w = rng_.standard_normal(4)
    w /= np.linalg.norm(w)
    G, s4 = ordering.batch_step(w[None, :], X)
    h = 1e-5
    num = np.array([(f(w + h * e) - f(w - h * e)) / (2 * h) for e in np.eye(4)])
    assert np.allclose(4.0 * (G[0] + 3.0 * w), num, rtol=1e-7, atol=1e-9)
    assert s4[0] / M == pytest.approx(f(w), rel=1e-12)


def test_update_identity_w_dot_g_equals_alpha():
    cfg, Xw, _, _ = _white()
    W = rng.candidates(5, 1, np.arange(40), Xw.shape[0])
    W /= np.linalg.norm(W, axis=1, keepdims=True)
    G, s4 = ordering.batch_step(W, Xw, block=777)          # ragged blocks
    alpha = s4 / Xw.shape[1] - 3.0
    assert np.abs(np.sum(W * G, axis=1) - alpha).max() < 1e-12
    # with an accepted prefix the projection keeps the identity (P w = w)
    W_acc = np.linalg.qr(np.random.default_rng(0).standard_normal((Xw.shape[0], 2)))[0].T
    Wp = ordering.project(W, W_acc)
    Wp /= np.linalg.norm(Wp, axis=1, keepdims=True)
    G, s4 = ordering.batch_step(Wp, Xw)
    Gp = ordering.project(G, W_acc)
    assert np.abs(np.sum(Wp * Gp, axis=1) - (s4 / Xw.shape[1] - 3.0)).max() < 1e-12
    assert np.abs(Gp @ W_acc.T).max() < 1e-12


def test_blocking_does_not_change_the_sum():
    cfg, Xw, _, _ = _white()
    W = rng.candidates(9, 1, np.arange(7), Xw.shape[0])
    G1, s1 = ordering.batch_step(W, Xw, block=10 ** 9)
    G2, s2 = ordering.batch_step(W, Xw, block=1000)
    assert np.allclose(G1, G2, rtol=1e-12, atol=1e-12) and np.allclose(s1, s2, rtol=1e-12)


def test_fixed_point_invariants_of_converged_candidates():
    cfg, Xw, _, _ = _white()
    ids = np.arange(64)
    W, iters, conv, deg, _, _ = ordering.run_component(Xw, np.zeros((0, Xw.shape[0])), 1, cfg.cand_seed, ids, 200, 1e-10)
    assert conv.sum() >= 60
    Wc = W[conv]
    G, s4 = ordering.batch_step(Wc, Xw)
    alpha = s4 / Xw.shape[1] - 3.0
    ng = np.linalg.norm(G, axis=1)
    cos = np.sum(G * Wc, axis=1) / ng
    assert np.all(1.0 - np.abs(cos) < 1e-8)                      # g parallel to w
    assert np.allclose(ng, np.abs(alpha), rtol=1e-6)             # ||g|| = |alpha|
    assert np.all(np.sign(cos) == np.sign(alpha))                # w_new = sign(alpha) w


def test_source_recovery_special_case():
    """A = I, unit-variance independent sources: one update from e_j gives +-e_j."""
    g = S._gen(21, "cpu")
    M = 100_000
    X = np.vstack([S.laplace(M, g, "cpu").numpy()] + [S.gaussian(M, g, "cpu").numpy() for _ in range(4)])
    G, _ = ordering.batch_step(np.eye(5)[:1], X)
    w = G[0] / np.linalg.norm(G[0])
    assert np.abs(np.abs(w) - np.eye(5)[0]).max() < 5e-2


def test_convergence_distance_geometry():
    rng_ = np.random.default_rng(4)
    B = rng_.standard_normal((6, 5))
    B /= np.linalg.norm(B, axis=1, keepdims=True)
    assert np.all(ordering.convergence_distance(B, B) == 0)
    assert np.all(ordering.convergence_distance(-B, B) == 0)
    th = 1e-3
    e1, e2 = np.eye(5)[:1], np.eye(5)[1:2]
    Bt = math.cos(th) * e1 + math.sin(th) * e2
    d = ordering.convergence_distance(Bt, e1)[0]
    assert d == pytest.approx(1 - math.cos(th), rel=1e-9)            # 1 - |cos| (BASELINE tol rule)
    chord = 2 * math.sin(th / 2)                                     # SPEC.md:273 chord length
    assert d == pytest.approx(chord ** 2 / 2, rel=1e-9)


def test_degenerate_candidate():
    cfg, Xw, _, _ = _white()
    N = Xw.shape[0]
    W_acc = np.eye(N)[:3]
    with pytest.raises(fastica.DegenerateCandidate):
        fastica.fastica_one_unit(W_acc[1] * 2.0, Xw, W_acc.T @ W_acc, 10, 1e-10)
    assert np.abs(ordering.project(W_acc[1:2], W_acc)).max() == 0.0


def test_sign_flip_start_converges_to_same_axis():
    """w0 = -w* converges to +-w* (SPEC.md:182)."""
    cfg, Xw, _, _ = _white()
    N = Xw.shape[0]
    w, _, t, c = fastica.fastica_one_unit(rng.candidates(1, 1, [0], N)[0], Xw, np.zeros((N, N)), 200, 1e-10)
    w2, _, t2, c2 = fastica.fastica_one_unit(-w, Xw, np.zeros((N, N)), 200, 1e-10)
    assert c and c2 and 1 - abs(w @ w2) < 1e-12
