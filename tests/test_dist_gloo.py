"""L-shard selection across ranks, world_size 2 on CPU (gloo).

Each rank owns a contiguous block of global candidate ids (as oica_init_candidates splits
them), forms its local cluster records exactly as the device kernels do (eligible converged
candidates, clusters by 1-|cos| <= 1e-6, q = minimum id, alpha at q's final w), exchanges
them with an all-gather, and decides with liboica's host merge (the same source as the
device merge kernel).  Both ranks must reach the single-process oracle decision.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import datagen
from oracle import contrast, ordering, whiten
from paper_2408_17118_b200 import oica

MAXC = oica.MAX_CLUSTERS


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def local_records(X, W, ids, conv, N):
    """Per-rank stage of K5 (census/argmax/assign/alpha_exact/finish) in numpy."""
    recs = np.zeros((MAXC, 6))
    rows = np.zeros((MAXC, N))
    e = np.nonzero(conv)[0]
    alpha = ordering.alpha_rows(W[e], X) if e.size else np.zeros(0)
    ups, ok = contrast.upsilon_masked(alpha)
    assigned = np.zeros(e.size, dtype=bool)
    umax = None
    for c in range(MAXC):
        cand = np.nonzero(~assigned & ok)[0]
        if umax is not None:
            cand = cand[ups[cand] >= umax - max(1e-2 * abs(umax), 1e-7)]
        if cand.size == 0:
            break
        p = cand[np.lexsort((ids[e][cand], -ups[cand]))[0]]
        if umax is None:
            umax = ups[p]
        mem = np.nonzero(~assigned & ok & ((1 - np.abs(W[e] @ W[e][p])) <= 1e-6))[0]
        assigned[mem] = True
        q = mem[np.argmin(ids[e][mem])]
        a = float(ordering.alpha_rows(W[e][q:q + 1], X)[0])
        recs[c] = [contrast.upsilon(a), a, ids[e][q], mem.size, 0, 1]
        rows[c] = W[e][q]
    return recs, rows


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = datagen.PARITY["p_ragged"]
    ds = datagen.make_dataset(cfg)
    Xw, _, _, _ = whiten.whiten(ds.X.numpy())
    X = Xw.astype(np.float32).astype(np.float64)
    N, L = cfg.N, cfg.L
    lo, hi = L * rank // world, L * (rank + 1) // world          # oica_init_candidates split
    ids = np.arange(lo, hi)
    W, iters, conv, deg, _, _ = ordering.run_component(X, np.zeros((0, N)), 1, cfg.cand_seed, ids, cfg.K, cfg.tol)
    recs, rows = local_records(X, W, ids, conv, N)
    R = [torch.zeros(MAXC, 6, dtype=torch.float64) for _ in range(world)]
    Wl = [torch.zeros(MAXC, N, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(R, torch.from_numpy(recs))
    dist.all_gather(Wl, torch.from_numpy(rows))
    allr = torch.cat(R).numpy()
    allw = torch.cat(Wl).numpy()
    recl = [dict(upsilon=r[0], alpha=r[1], q=int(r[2]), size=int(r[3]), iters=0, valid=int(r[5])) for r in allr]
    m = oica.merge_records(recl, allw)
    q.put((rank, int(allr[m["winner"]][2]), m["size"], float(allr[m["winner"]][1])))
    dist.destroy_process_group()


def test_lshard_selection_two_ranks_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # every rank reaches the same decision ...
    assert out[0][1:] == out[1][1:]
    # ... and it is the single-process oracle's decision (A6)
    cfg = datagen.PARITY["p_ragged"]
    ds = datagen.make_dataset(cfg)
    Xw, _, _, _ = whiten.whiten(ds.X.numpy())
    X = Xw.astype(np.float32).astype(np.float64)
    _, res = ordering.extract(X, cfg.L, cfg.K, cfg.tol, 1, cfg.cand_seed)
    assert out[0][1] == res[0].index and out[0][2] == res[0].cluster_size
    assert out[0][3] == pytest.approx(res[0].alpha, rel=1e-12)
