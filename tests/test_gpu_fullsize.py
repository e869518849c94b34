"""GPU parity at BASELINE.json's full sizes, in the launch configuration bench.py times.

The full-L oracle is out of reach at these sizes (cfg 3 alone is hours of fp64 numpy), so the
checks follow SURVEY.md §8(c) "tier C": outputs the oracle can compute one by one, plus
properties that hold at any size.  This module uses a DEVICE draw of each recipe (a second data
set besides the goldens' host draw); tests/test_gpu_certificate.py certifies every component of
cfgs 3 and 4 at full L on the goldens' data.

Component 1 (no prefix, so every oracle input is the seeded data and the candidate generator):
  * sampled candidates: a seeded sample of global ids (chosen without looking at the GPU) is run
    through the oracle's candidate phase (oracle.ordering.run_component with ids=sample); the GPU's
    end state of the same ids (full-L run, AUTO precision = the bench's tensor-core kernel at
    M >= 16384) must agree: converged flag, direction |cos| >= 0.9999;
  * the accepted candidate q: the oracle replays candidate q from its seed; the GPU's accepted row
    and objective must match it (|cos| >= 0.9999, rel. error of sum y^4/M <= 1e-4, north_star);
  * certificate of the selection rule (reading A6): no sampled converged candidate
    outside q's cluster has a larger Upsilon (beyond the near-tie margin), and no sampled id < q
    lies in q's cluster (q = min C).
Components 2-3 (the prefix is the GPU's own, so only properties are checked): orthonormal rows
(S:194), the accepted row is a fixed point of the projected update, the oracle-computed
alpha at the GPU's row equals the reported one, Upsilon non-increasing (Theorem 1).

Inputs: datagen raw signals, whitened by the ORACLE in fp64 and cast to fp32 (both sides consume
the same fp32 values).  Also checked here: oica_whiten against the oracle's whitening at full size.
"""
import functools
import time

import numpy as np
import pytest
import torch

import datagen
from oracle import contrast, ordering, whiten
from paper_2408_17118_b200 import oica

pytestmark = pytest.mark.gpu

FULL = ["cfg1_artificial", "cfg2_eeg_shaped", "cfg3_large", "cfg4_scaling"]
N_SAMPLE = 24


@functools.lru_cache(maxsize=1)
def prepared(name):
    cfg = datagen.get(name)
    ds = datagen.make_dataset(cfg, device="cuda", dtype=torch.float64, keep_sources=False)
    Xraw = ds.X.float().cpu().numpy()           # fp32 raw signals: the same values on both sides
    del ds
    torch.cuda.empty_cache()
    Xw, mean, V, d = whiten.whiten(Xraw.astype(np.float64))
    X32 = np.ascontiguousarray(Xw.astype(np.float32))
    del Xw
    return cfg, Xraw, X32, (mean, V, d)


def sample_ids(cfg):
    rs = np.random.default_rng(12345 + cfg.N)
    ids = set(range(8)) | set(rs.choice(cfg.L, N_SAMPLE - 8, replace=False).tolist())
    return np.array(sorted(ids), dtype=np.int64)


@pytest.mark.parametrize("name", FULL)
def test_fullsize_component_parity(name):
    t0 = time.time()
    cfg, _, X32, _ = prepared(name)
    X64 = X32.astype(np.float64)
    stream = torch.cuda.Stream()
    with oica.Context(0, oica.PREC_AUTO, stream=stream) as ctx:
        Xd = torch.from_numpy(X32).cuda()
        ctx.set_data(Xd)
        ctx.init_candidates(cfg.cand_seed, cfg.L)
        r1 = ctx.extract(1, cfg.K, cfg.tol)
        cand = ctx.candidates()
        prec = ctx.stats()["precision"]
        r3 = ctx.extract(3, cfg.K, cfg.tol, W_prefix=r1.W[:1])
    assert prec == (oica.PREC_TC if cfg.M >= 16384 else oica.PREC_FP32)
    assert r1.n_extracted == 1 and r3.n_extracted == 3
    q = int(r1.index[0])
    w_g = r1.W[0]

    # -- sampled candidates (oracle one by one, ids chosen without the GPU) and the accepted
    #    candidate q replayed from its seed (rows are independent: one batched oracle call)
    ids = sample_ids(cfg)
    run = np.union1d(ids, [q])
    W_r, _, conv_r, _, _, _ = ordering.run_component(X64, np.zeros((0, cfg.N)), 1, cfg.cand_seed, run,
                                                     cfg.K, cfg.tol)
    sel = np.searchsorted(run, ids)
    W_o, conv_o = W_r[sel], conv_r[sel]
    conv_g = cand["state"][ids] == 1
    assert np.sum(conv_g != conv_o) <= 1, (ids, conv_g, conv_o)
    both = conv_g & conv_o
    cos = np.abs(np.sum(cand["W"][ids][both] * W_o[both], axis=1))
    assert cos.min() >= 0.9999, cos
    a_r = np.full(len(run), np.nan)
    a_r[conv_r] = ordering.alpha_rows(W_r[conv_r], X64)
    ups_o = np.where(conv_o, contrast.upsilon(np.where(conv_o, a_r[sel], 0.0)), -np.inf)
    iq = int(np.searchsorted(run, q))
    assert conv_r[iq], "oracle: the accepted candidate does not converge"
    Wq = W_r[iq:iq + 1]
    a_q = float(a_r[iq])
    u_q = float(contrast.upsilon(a_q))
    cos_q = abs(float(Wq[0] @ w_g))
    rel_q = abs((r1.alpha[0] + 3.0) - (a_q + 3.0)) / (a_q + 3.0)
    assert cos_q >= 0.9999 and rel_q <= 1e-4, (cos_q, rel_q)

    # -- selection certificate over the sample (A6)
    cos_to_q = np.abs(W_o @ Wq[0])
    in_c = conv_o & ((1.0 - cos_to_q) <= 1e-6)
    out_c = conv_o & ~in_c
    if out_c.any():
        assert ups_o[out_c].max() <= u_q * (1 + 1e-6), (ups_o[out_c].max(), u_q)
    assert not np.any(in_c & (ids < q)), (ids[in_c], q)
    # GPU-side consistency of q = min C over ALL candidates
    cl = (cand["state"] == 1) & (1.0 - np.abs(cand["W"] @ w_g) <= 1e-6)
    assert cl[q] and np.nonzero(cl)[0].min() == q

    # -- components 2..3: properties at any size
    W3 = r3.W
    assert np.abs(W3 @ W3.T - np.eye(3)).max() < 1e-10
    for k in range(1, 3):
        P_acc = W3[:k]
        w = W3[k]
        g, s4 = ordering.batch_step(w[None, :], X64)
        g = ordering.project(g, P_acc)[0]
        wn = g / np.linalg.norm(g)
        assert 1.0 - abs(float(wn @ w)) <= 1e-7, k      # converged fixed point (tol 1e-10 on the GPU path)
        a_k = float(s4[0] / cfg.M - 3.0)
        assert abs((r3.alpha[k] + 3.0) - (a_k + 3.0)) <= 1e-9 * (a_k + 3.0), (k, r3.alpha[k], a_k)
    ups = np.array([r1.upsilon[0], r3.upsilon[1], r3.upsilon[2]])
    assert np.all(np.diff(ups) <= 1e-6 * ups[0]), ups
    print(name, "q", q, "cos_q", 1 - cos_q, "rel", rel_q, "sample conv", int(conv_o.sum()), "/", len(ids),
          "max 1-cos", float(1 - cos.min()), "secs", round(time.time() - t0, 1))


@pytest.mark.parametrize("name", ["cfg4_scaling"])
def test_fullsize_whitening(name):
    cfg, Xraw, X32_o, (mean_o, V_o, d_o) = prepared(name)
    with oica.Context(0) as ctx:
        Xd = torch.from_numpy(Xraw).cuda()
        Xw = torch.empty_like(Xd)
        mean, V, eig = ctx.whiten(Xd, Xw)
    scale = np.abs(Xraw[:, :4096]).max()
    assert np.abs(mean - mean_o).max() <= 1e-12 * scale
    assert np.allclose(eig, d_o, rtol=1e-8)
    assert np.abs(V - V_o).max() < 1e-6 * np.abs(V_o).max()
    cols = np.random.default_rng(7).choice(cfg.M, 4096, replace=False)
    Xs = Xw[:, torch.from_numpy(cols).cuda()].cpu().numpy()
    assert np.abs(Xs - X32_o[:, cols]).max() < 1e-5 * np.abs(X32_o[:, cols]).max()
