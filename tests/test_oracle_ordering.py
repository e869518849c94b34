"""Pins for the extraction driver and selection (oracle O1 / O2 / O3).

Pins against what the paper and mathematics fix:
  * brute-force global maximum of Upsilon(alpha(w)) on the sphere (N = 2, 3): Theorem 1
    says the accepted component is the GLOBAL maximiser;
  * Upsilon, not sum y^4, is the selection key (uniform vs Student-t case, A5);
  * the last component is the closed-form null vector of the accepted rows;
  * W W^T = I and non-increasing Upsilon (Theorem 1);
  * L = 1, component 1 equals textbook deflation FastICA (scikit-learn, fun='cube');
  * Alg. 1 (O2) == Alg. 2 batched (O1) == Alg. 2 reduced (O3);
  * complement basis properties + SPEC.md:245 singular example, sym_inv_sqrt diag(4,9);
  * Amari index gates (A23), Gaussian-data stop, Laplace+Gaussian;
  * selection rule A6 on constructed clusters; metric worked examples.
"""
import math

import numpy as np
import pytest
from scipy.optimize import minimize

import datagen
from datagen import Config
from oracle import contrast, fastica, metrics, ordering, reduced, rng, select, whiten


def _prep(cfg, M=None, seed=None):
    ds = datagen.make_dataset(cfg, M=M, seed=seed)
    Xw, _, V, _ = whiten.whiten(ds.X.numpy())
    return Xw.astype(np.float32).astype(np.float64), V, ds


def _ups_of(w, X):
    y = w @ X
    return float(contrast.upsilon(np.mean(y ** 4) - 3.0))


def _refine(obj, x0):
    r = minimize(lambda x: -obj(x), x0, method="Nelder-Mead", options=dict(xatol=1e-12, fatol=1e-15, maxiter=4000))
    return r.x


MIX3 = Config("mix3", 3, 5000, 64, 200, 1e-10, 3,
              (("laplace", 1), ("uniform", 1), ("student_t", 1, 7.0)), data_seed=77, cand_seed=78)


def test_brute_force_global_max_N2():
    cfg = MIX3.with_(N=2, recipe=(("laplace", 1), ("uniform", 1)), N_out=1)
    X, _, _ = _prep(cfg)
    W, res = ordering.extract(X, cfg.L, cfg.K, cfg.tol, 1, cfg.cand_seed)
    th = np.linspace(0, np.pi, 20_000, endpoint=False)
    U = np.stack([np.cos(th), np.sin(th)], 1)
    a = np.concatenate([np.mean((U[k:k + 2000] @ X) ** 4, axis=1) - 3.0 for k in range(0, len(U), 2000)])
    best = th[np.argmax(contrast.upsilon(a))]
    tb = _refine(lambda t: _ups_of(np.array([math.cos(t[0]), math.sin(t[0])]), X), [best])[0]
    wb = np.array([math.cos(tb), math.sin(tb)])
    assert 1 - abs(wb @ W[0]) <= 1e-8
    assert res[0].upsilon == pytest.approx(_ups_of(wb, X), rel=1e-9)


def _fib_sphere(n):
    k = np.arange(n) + 0.5
    phi = np.arccos(1 - 2 * k / n)
    th = np.pi * (1 + 5 ** 0.5) * k
    return np.stack([np.cos(th) * np.sin(phi), np.sin(th) * np.sin(phi), np.cos(phi)], 1)


def test_brute_force_global_max_N3_two_steps():
    X, _, _ = _prep(MIX3)
    W, res = ordering.extract(X, MIX3.L, MIX3.K, MIX3.tol, 2, MIX3.cand_seed)
    # step 1: Fibonacci sphere (upper hemisphere suffices by symmetry) then local refinement
    P = _fib_sphere(20_000)
    ups = np.concatenate([contrast.upsilon(np.mean((P[k:k + 2000] @ X) ** 4, 1) - 3) for k in range(0, len(P), 2000)])
    p0 = P[np.argmax(ups)]

    def sph(x):
        v = np.array([math.sin(x[0]) * math.cos(x[1]), math.sin(x[0]) * math.sin(x[1]), math.cos(x[0])])
        return v

    x0 = [math.acos(np.clip(p0[2], -1, 1)), math.atan2(p0[1], p0[0])]
    w1 = sph(_refine(lambda x: _ups_of(sph(x), X), x0))
    assert 1 - abs(w1 @ W[0]) <= 1e-8
    assert res[0].upsilon == pytest.approx(_ups_of(w1, X), rel=1e-9)
    # step 2: the circle orthogonal to the accepted w1
    Q = np.linalg.svd(W[:1])[2][1:]                     # orthonormal basis of w1-perp
    th = np.linspace(0, np.pi, 20_000, endpoint=False)
    C = np.cos(th)[:, None] * Q[0] + np.sin(th)[:, None] * Q[1]
    ups2 = np.concatenate([contrast.upsilon(np.mean((C[k:k + 2000] @ X) ** 4, 1) - 3) for k in range(0, len(C), 2000)])
    t0 = th[np.argmax(ups2)]
    t2 = _refine(lambda t: _ups_of(math.cos(t[0]) * Q[0] + math.sin(t[0]) * Q[1], X), [t0])[0]
    w2 = math.cos(t2) * Q[0] + math.sin(t2) * Q[1]
    assert 1 - abs(w2 @ W[1]) <= 1e-8
    assert res[1].upsilon >= _ups_of(w2, X) * (1 - 1e-9)


def test_upsilon_not_fourth_moment_is_the_key():
    """Uniform (alpha~-1.2, Upsilon~0.6) vs t(9) (alpha~1.2, Upsilon~0.3): accept the uniform (A5)."""
    cfg = Config("ut", 2, 20000, 64, 200, 1e-10, 1, (("uniform", 1), ("student_t", 1, 9.0)), data_seed=5, cand_seed=6)
    X, V, ds = _prep(cfg)
    W, res = ordering.extract(X, cfg.L, cfg.K, cfg.tol, 1, cfg.cand_seed)
    P = W @ V @ ds.A.numpy()
    assert abs(P[0, 0]) / np.linalg.norm(P[0]) > 0.99          # uniform source is row 0
    assert res[0].alpha < 0
    # and argmax of sum y^4 alone would have picked the other cluster
    Wc, _, st = ordering.extract(X, cfg.L, cfg.K, cfg.tol, 1, cfg.cand_seed, keep_candidates=True)
    s = st[0]
    ok = s.converged
    assert s.alpha[ok].max() > 0 and np.argmax(s.alpha[ok]) != np.argmin(s.alpha[ok])


def test_last_component_closed_form():
    cfg = datagen.get(0)
    X, _, _ = _prep(cfg)
    W, res = ordering.extract(X, cfg.L, cfg.K, cfg.tol, cfg.N, cfg.cand_seed)
    null = np.linalg.svd(W[:-1])[2][-1]
    assert 1 - abs(null @ W[-1]) < 1e-12
    last = res[-1]
    assert last.n_converged == cfg.L and last.cluster_size == cfg.L and last.iters == 1
    assert last.index == 0                                       # cluster min id


@pytest.mark.parametrize("seed", range(5))
def test_orthonormal_and_nonincreasing_upsilon(seed):
    cfg = datagen.get(0)
    X, V, ds = _prep(cfg, seed=1000 + 17 * seed)
    W, res = ordering.extract(X, cfg.L, cfg.K, cfg.tol, cfg.N_out, cfg.cand_seed + seed)
    assert np.abs(W @ W.T - np.eye(cfg.N_out)).max() < 1e-12
    ups = [r.upsilon for r in res]
    assert all(a >= b for a, b in zip(ups, ups[1:])), ups
    assert metrics.amari_rows(W @ V @ ds.A.numpy()) <= 0.1      # A23 gate, cfg 0


def test_amari_easy_case():
    cfg = Config("easy", 4, 100_000, 32, 200, 1e-10, 4, (("laplace", 4),), data_seed=9, cand_seed=10)
    X, V, ds = _prep(cfg)
    W, res = ordering.extract(X, cfg.L, cfg.K, cfg.tol, cfg.N_out, cfg.cand_seed)
    assert metrics.amari_rows(W @ V @ ds.A.numpy()) <= 0.02


def test_matches_sklearn_deflation_fastica_L1():
    from sklearn.decomposition import FastICA

    cfg = datagen.PARITY["p_ragged"]
    ds = datagen.make_dataset(cfg)
    Xw, _, _, _ = whiten.whiten(ds.X.numpy())                    # exact fp64 whitening: mean(y^2) = 1
    from oracle import rng
    w0 = rng.candidates(cfg.cand_seed, 1, [0], cfg.N)[0]
    Wst = ordering.run_component(Xw, np.zeros((0, cfg.N)), 1, cfg.cand_seed, np.array([0]), 500, 1e-14)
    w_or = Wst[0][0]
    init = np.eye(cfg.N)
    init[0] = w0
    ica = FastICA(n_components=cfg.N, algorithm="deflation", fun="cube", whiten=False, w_init=init, max_iter=500, tol=1e-14)
    ica.fit(Xw.T)
    w_sk = ica.components_[0]
    assert 1 - abs(w_sk @ w_or) / np.linalg.norm(w_sk) <= 1e-10


def test_alg1_alg2_reduced_equivalence():
    cfg = Config("eq6", 6, 8000, 24, 200, 1e-10, 6,
                 (("laplace", 2), ("gg_uniform", 2, 0.6, 1.6), ("uniform", 1), ("student_t", 1, 8.0)),
                 data_seed=31, cand_seed=32)
    X, _, _ = _prep(cfg)
    W1, r1 = ordering.extract(X, cfg.L, cfg.K, cfg.tol, cfg.N_out, cfg.cand_seed)
    W2, r2 = fastica.ordering_ica_reference(X, cfg.L, cfg.K, cfg.tol, cfg.N_out, cfg.cand_seed)
    W3, r3 = reduced.ordering_ica_fast_reduced(X, cfg.L, cfg.K, cfg.tol, cfg.N_out, cfg.cand_seed)
    assert [r.index for r in r1] == [r.index for r in r2] == [r.index for r in r3]
    assert np.abs(W1 - W2).max() < 1e-9 and np.abs(W1 - W3).max() < 1e-9
    for a, b, c in zip(r1, r2, r3):
        assert a.iters == b.iters == c.iters and a.n_converged == b.n_converged == c.n_converged
        assert a.alpha == pytest.approx(b.alpha, abs=1e-10) and a.alpha == pytest.approx(c.alpha, abs=1e-10)
        assert a.sum_active == c.sum_active


def test_reduced_trajectory_equivalence():
    """O3 iterates mapped through G^T equal O1's projected iterates step by step."""
    cfg = Config("tr5", 5, 6000, 10, 200, 1e-10, 3, (("laplace", 3), ("uniform", 2)), data_seed=41, cand_seed=42)
    X, _, _ = _prep(cfg)
    W1, r1 = ordering.extract(X, cfg.L, cfg.K, cfg.tol, cfg.N_out, cfg.cand_seed)
    trajs = []
    reduced.ordering_ica_fast_reduced(X, cfg.L, cfg.K, cfg.tol, cfg.N_out, cfg.cand_seed, trajectories=trajs)
    from oracle import rng
    for i, traj in enumerate(trajs, start=1):
        W_acc = W1[: i - 1]
        E = W_acc.T @ W_acc
        for l in range(cfg.L):
            tr = []
            fastica.fastica_one_unit(rng.candidates(cfg.cand_seed, i, [l], cfg.N)[0], X, E, cfg.K, cfg.tol, trajectory=tr)
            steps = [W[list(a).index(l)] for a, W in traj if l in a]
            assert len(steps) == len(tr)
            assert max(np.abs(s - t).max() for s, t in zip(steps, tr)) < 1e-9


def test_complement_basis_properties():
    rng_ = np.random.default_rng(5)
    Wq = np.linalg.qr(rng_.standard_normal((5, 2)))[0].T
    G = reduced.complement_basis(Wq, 5)
    assert G.shape == (3, 5)
    assert np.abs(G @ G.T - np.eye(3)).max() < 1e-9
    assert np.abs(G @ Wq.T).max() < 1e-9
    assert np.abs(G.T @ G - (np.eye(5) - Wq.T @ Wq)).max() < 1e-9
    # SPEC.md:245 singular example: W = e1^T, N = 3 -> fallback still a valid basis
    G1 = reduced.complement_basis(np.eye(3)[:1], 3)
    assert np.abs(G1 @ G1.T - np.eye(2)).max() < 1e-12 and np.abs(G1[:, 0]).max() < 1e-12
    assert np.allclose(reduced.complement_basis(np.zeros((0, 4)), 4), np.eye(4))
    R = reduced.sym_inv_sqrt(np.diag([4.0, 9.0]))
    assert np.allclose(R, np.diag([0.5, 1 / 3]), atol=1e-14)
    Qr = np.array([[math.cos(0.3), -math.sin(0.3)], [math.sin(0.3), math.cos(0.3)]])
    S2 = Qr @ np.diag([4.0, 9.0]) @ Qr.T
    R2 = reduced.sym_inv_sqrt(S2)
    assert np.abs(R2 @ S2 @ R2 - np.eye(2)).max() < 1e-10


def test_determinism_bitwise():
    cfg = datagen.PARITY["p_ragged"]
    X, _, _ = _prep(cfg)
    W1, r1 = ordering.extract(X, cfg.L, cfg.K, cfg.tol, 3, cfg.cand_seed)
    W2, r2 = ordering.extract(X, cfg.L, cfg.K, cfg.tol, 3, cfg.cand_seed)
    assert np.array_equal(W1, W2) and [r.alpha for r in r1] == [r.alpha for r in r2]


def test_gaussianity_stop_mechanics():
    """PAPER.md:143-145 / :260-262: the flagged component is not appended and the loop stops.

    3 Laplace (Upsilon ~ 1.2) + 2 Gaussian sources: the Laplace components are far above
    2(N-i+2)(N-i+1)/M and never flagged; the first flagged component comes after them.
    (SPEC.md:189's ">= 9/10 pure-Gaussian seeds stop at i = 1" is NOT a property the paper
    fixes and was not reproduced: 3/10 seeds at N=5, M=1e5, L=20 -- see DESIGN.md §2.)
    """
    cfg = Config("lg5", 5, 100_000, 20, 200, 1e-10, 5, (("laplace", 3), ("gaussian", 2)), data_seed=500, cand_seed=600)
    X, V, ds = _prep(cfg)
    W_all, r_all = ordering.extract(X, cfg.L, cfg.K, cfg.tol, 5, cfg.cand_seed)
    assert not any(r.gaussian_flag for r in r_all[:3])
    assert all(r.upsilon > 100 * contrast.gaussianity_threshold(5, r.i, cfg.M) for r in r_all[:3])
    W, res = ordering.extract(X, cfg.L, cfg.K, cfg.tol, 5, cfg.cand_seed, stop_on_gaussianity=True)
    flagged = [r.i for r in r_all if r.gaussian_flag]
    if flagged:
        k = flagged[0]
        assert k >= 4 and res[-1].stopped and res[-1].i == k and W.shape[0] == k - 1
        assert np.array_equal(W, W_all[: k - 1])
    else:
        assert W.shape[0] == 5
    P = W[:3] @ V @ ds.A.numpy()
    assert np.all(np.abs(P[:, :3]).max(1) / np.linalg.norm(P, axis=1) > 0.99)


def test_laplace_plus_gaussian_first_component():
    cfg = Config("lg", 2, 10_000, 20, 200, 1e-10, 1, (("laplace", 1), ("gaussian", 1)), data_seed=71, cand_seed=72)
    X, V, ds = _prep(cfg)
    W, res = ordering.extract(X, cfg.L, cfg.K, cfg.tol, 1, cfg.cand_seed)
    P = (W @ V @ ds.A.numpy())[0]
    assert abs(P[0]) / np.linalg.norm(P) > 0.99


def test_selection_rule_clusters_and_ties():
    rng_ = np.random.default_rng(8)
    a = np.linalg.qr(rng_.standard_normal((4, 2)))[0].T
    W = np.array([a[1], a[0], a[0] * -1, a[0] + 1e-5 * a[1], a[1]])
    W /= np.linalg.norm(W, axis=1, keepdims=True)
    ids = np.array([10, 4, 7, 2, 1])
    alpha = np.array([1.0, 2.0, 2.0 + 1e-9, 2.0 - 1e-9, 1.0])
    s = select.select(ids, W, alpha)
    assert s["id_p"] == 7 and s["cluster_size"] == 3 and s["id_q"] == 2 and not s["near_tie"]
    assert select.select(ids, W, alpha, raw_argmax=True)["id_q"] == 7
    # exact tie between clusters: p = lowest id among the tied maxima, flagged near_tie
    alpha2 = np.array([2.0, 2.0, 1.0, 1.0, 1.0])
    s2 = select.select(ids, W, alpha2)
    assert s2["id_p"] == 4 and s2["near_tie"]
    # out-of-domain alpha excluded (A13)
    s3 = select.select(ids, W, np.array([-2.5, 0.5, 0.4, 0.3, 0.2]))
    assert s3["n_domain"] == 1 and s3["id_p"] == 4
    assert np.array_equal(select.canonical_sign(np.array([0.1, -0.9, 0.9])), [-0.1, 0.9, -0.9])


def test_metric_worked_examples():
    A = np.random.default_rng(3).standard_normal((3, 3))
    Wi = np.linalg.inv(A)
    assert metrics.ordering_error(Wi, A) == 0 and metrics.ordering_error(-Wi, A) == 0
    assert metrics.ordering_error(Wi[[1, 0, 2]], A) == pytest.approx(4 / 9)
    u = np.array([1.0, 0.0])
    assert metrics.cosine_divergence(u, -u) == 0 and metrics.cosine_divergence(u, [0, 1.0]) == 1
    runs = [np.array([[math.cos(t), math.sin(t)]]) for t in (0, math.pi / 3, 2 * math.pi / 3)]
    assert metrics.fluctuation(runs)[0] == pytest.approx(0.5)
    assert metrics.amari_rows(np.eye(3)[:2] * [[2.0], [-1.0]]) == 0


# ---- reading A4 pinned against the literal algorithms (Alg. 1: every FastICA
# run returns after at most K updates and the argmax runs over ALL L runs
# Alg. 2: the argmax runs over B_conv only).  The reference below is the per-candidate FastICA
# function of PAPER.md:149-165 (oracle.fastica.fastica_one_unit) followed by the paper's plain
# argmax p = argmax_l Upsilon(alpha_l) written out here (ties -> lowest l): no eligibility code,
# no cluster rule (O1 is run with raw_argmax, the paper's p itself).
def _literal_component(X, W_acc, i, seed, L, K, tol, over):
    N, M = X.shape
    E = W_acc.T @ W_acc if W_acc.shape[0] else np.zeros((N, N))
    R = rng.candidates(seed, i, np.arange(L), N)
    ws, alphas, its, conv = [], [], [], []
    for l in range(L):
        w, y, t, c = fastica.fastica_one_unit(R[l], X, E, K, tol)
        ws.append(w)
        alphas.append(np.sum(y ** 4) / M - 3.0)
        its.append(t)
        conv.append(c)
    alphas, conv = np.array(alphas), np.array(conv)
    ups = alphas - 2.0 * np.log(alphas / 2.0 + 1.0)                   # eq. (1)
    pool = np.arange(L) if over == "all" else np.nonzero(conv)[0]      # Alg. 1: all runs; Alg. 2: B_conv
    p = int(pool[np.argmax(ups[pool])])                               # PAPER.md:142 / :259
    return p, ws[p], alphas[p], np.array(its), conv


@pytest.mark.parametrize("K", [1, 3, 5, 9])   # K = 9: some runs converged, some not
def test_include_unconverged_is_literal_alg1(K):
    """OICA_INCLUDE_UNCONVERGED (O1 include_unconverged=True) is Algorithm 1's selection: argmax
    over every run after <= K updates, converged or not."""
    cfg = datagen.PARITY["p_ragged"].with_(L=60)
    X, _, _ = _prep(cfg)
    W1, r1 = ordering.extract(X, cfg.L, K, cfg.tol, 2, cfg.cand_seed, include_unconverged=True, raw_argmax=True)
    W_acc = np.zeros((0, cfg.N))
    for k in range(2):
        p, w, a, its, conv = _literal_component(X, W_acc, k + 1, cfg.cand_seed, cfg.L, K, cfg.tol, "all")
        assert r1[k].index == p
        assert 1.0 - abs(float(r1[k].w @ w)) <= 1e-9 and abs(r1[k].alpha - a) <= 1e-9 * abs(a + 3.0)
        assert r1[k].n_converged == int(conv.sum())
        W_acc = np.vstack([W_acc, select.canonical_sign(w)[None, :]])
    assert np.abs(W1 - W_acc).max() < 1e-9


@pytest.mark.parametrize("K", [7, 9, 12])
def test_default_excludes_unconverged_as_alg2(K):
    """The default (reading A4) is Algorithm 2's selection: argmax over B_conv only,
    at a cap where some runs converge and some do not."""
    cfg = datagen.PARITY["p_ragged"].with_(L=60)
    X, _, _ = _prep(cfg)
    W1, r1 = ordering.extract(X, cfg.L, K, cfg.tol, 2, cfg.cand_seed, raw_argmax=True)
    W_acc = np.zeros((0, cfg.N))
    for k in range(2):
        p, w, a, its, conv = _literal_component(X, W_acc, k + 1, cfg.cand_seed, cfg.L, K, cfg.tol, "conv")
        assert 0 < conv.sum() < cfg.L, "the cap must leave some runs unconverged for this pin"
        assert not r1[k].no_converged and r1[k].index == p
        assert 1.0 - abs(float(r1[k].w @ w)) <= 1e-9 and abs(r1[k].alpha - a) <= 1e-9 * abs(a + 3.0)
        W_acc = np.vstack([W_acc, select.canonical_sign(w)[None, :]])


def test_no_converged_fallback_is_literal_alg1():
    """K = 1: no run can converge in one update, B_conv is empty; reading A4's fallback (all runs
    compete, flagged no_converged) is then Algorithm 1's argmax over all runs."""
    cfg = datagen.PARITY["p_ragged"].with_(L=60)
    X, _, _ = _prep(cfg)
    W1, r1 = ordering.extract(X, cfg.L, 1, cfg.tol, 2, cfg.cand_seed, raw_argmax=True)
    W_acc = np.zeros((0, cfg.N))
    for k in range(2):
        p, w, a, its, conv = _literal_component(X, W_acc, k + 1, cfg.cand_seed, cfg.L, 1, cfg.tol, "all")
        assert not conv.any() and r1[k].no_converged and r1[k].n_converged == 0
        assert r1[k].index == p and 1.0 - abs(float(r1[k].w @ w)) <= 1e-9
        W_acc = np.vstack([W_acc, select.canonical_sign(w)[None, :]])


def test_algorithmic_flops_counts_every_row_update():
    """F_alg = sum_t L_act(t) (4NM + 3M): every run is active in exactly the
    iterations that update it, so sum_t L_act(t) = sum_l t_l with t_l the per-run update counts of
    the literal per-candidate loop; 4NM + 3M is the flop count of one update
    (y = w X: 2NM, y^3: 2M, X y^3: 2NM, and y^4 for alpha: M)."""
    cfg = datagen.PARITY["p_ragged"].with_(L=40)
    X, _, _ = _prep(cfg)
    N, M = X.shape
    for K in (2, 200):
        W1, r1 = ordering.extract(X, cfg.L, K, cfg.tol, 2, cfg.cand_seed, raw_argmax=True)
        W_acc = np.zeros((0, N))
        total = 0
        for k in range(2):
            p, w, a, its, conv = _literal_component(X, W_acc, k + 1, cfg.cand_seed, cfg.L, K, cfg.tol, "all")
            assert r1[k].sum_active == int(its.sum()) and r1[k].n_iter == int(its.max())
            total += int(its.sum())
            W_acc = np.vstack([W_acc, r1[k].w[None, :]])
        assert ordering.algorithmic_flops(r1, N, M) == float(total) * (4.0 * N * M + 3.0 * M)
        assert ordering.algorithmic_flops(r1, N, M) == float(total) * (2 * N * M + 2 * M + 2 * N * M + M)
