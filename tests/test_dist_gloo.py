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


# ---- M-shard: every rank holds all runs but only its samples; per iteration the
# fp64 partial sums sum_m y^3 x and sum_m y^4 over its samples are all-reduced, and every rank
# applies the same epilogue to the same sums (PAPER.md:243-252 with M = the global count)
def _mshard_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = datagen.PARITY["p_ragged"].with_(L=40)
    ds = datagen.make_dataset(cfg)
    Xw, _, _, _ = whiten.whiten(ds.X.numpy())
    X = Xw.astype(np.float32).astype(np.float64)
    N, M = X.shape
    lo, hi = M * rank // world, M * (rank + 1) // world          # the M-shard sample split
    ln, S = oica.slot_plan(M, hi - lo)                           # the rank's slots cover its samples
    assert (S - 1) * ln < hi - lo <= S * ln
    Xr = X[:, lo:hi]
    ids = np.arange(cfg.L)
    from oracle import rng
    Wc = rng.candidates(cfg.cand_seed, 1, ids, N)
    Wc /= np.linalg.norm(Wc, axis=1, keepdims=True)
    active = np.arange(cfg.L)
    conv = np.zeros(cfg.L, dtype=bool)
    snapshots = []
    for t in range(1, cfg.K + 1):
        B = Wc[active]
        Y = B @ Xr
        Graw = (Y ** 3) @ Xr.T                                   # this rank's samples only
        s4 = np.sum(Y ** 4, axis=1)
        buf = torch.from_numpy(np.concatenate([Graw, s4[:, None]], axis=1).copy())
        dist.all_reduce(buf, op=dist.ReduceOp.SUM)               # fp64, every rank the same bits
        G = buf[:, :N].numpy() / M - 3.0 * B                     # eq. (5) with the GLOBAL M
        Wn = G / np.linalg.norm(G, axis=1, keepdims=True)
        d = ordering.convergence_distance(Wn, B)
        c = d <= cfg.tol
        Wc[active] = Wn
        conv[active[c]] = True
        active = active[~c]
        snapshots.append(Wc.copy())
        if active.size == 0:
            break
    # exact alpha at the final w: all-reduced partial sums of y^4
    s4 = torch.from_numpy(np.sum((Wc @ Xr) ** 4, axis=1).copy())
    dist.all_reduce(s4, op=dist.ReduceOp.SUM)
    alpha = s4.numpy() / M - 3.0
    e = np.nonzero(conv)[0]
    from oracle import select
    s = select.select(ids[e], Wc[e], alpha[e])
    q.put((rank, int(s["id_q"]), float(s["alpha_q"]), Wc.tobytes(), len(snapshots)))
    dist.destroy_process_group()


def test_mshard_decomposition_two_ranks_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_mshard_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # identical decisions and bitwise-identical iterates on both ranks (same all-reduced sums) ...
    assert out[0][1:] == out[1][1:]
    # ... within tolerance of the single-process oracle (the sample sum is re-associated by rank)
    cfg = datagen.PARITY["p_ragged"].with_(L=40)
    ds = datagen.make_dataset(cfg)
    Xw, _, _, _ = whiten.whiten(ds.X.numpy())
    X = Xw.astype(np.float32).astype(np.float64)
    W1, res = ordering.extract(X, cfg.L, cfg.K, cfg.tol, 1, cfg.cand_seed)
    assert out[0][1] == res[0].index
    assert out[0][2] == pytest.approx(res[0].alpha, rel=1e-10)
    Wq = np.frombuffer(out[0][3]).reshape(cfg.L, cfg.N)[res[0].index]
    assert 1.0 - abs(float(Wq @ res[0].w)) <= 1e-12


# ---- reading A4 across ranks: "no run converged" is a GLOBAL decision.  With a cap
# K at which one rank's runs all miss the test while the other rank has converged runs, the
# rank without converged runs must contribute no record (its unconverged runs would compete only
# if NO rank had converged runs) -- the single-process oracle's decision
def _a4_worker(rank, world, port, K, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = datagen.PARITY["p_ragged"].with_(L=12)
    ds = datagen.make_dataset(cfg)
    Xw, _, _, _ = whiten.whiten(ds.X.numpy())
    X = Xw.astype(np.float32).astype(np.float64)
    N, L = cfg.N, cfg.L
    lo, hi = L * rank // world, L * (rank + 1) // world
    ids = np.arange(lo, hi)
    W, iters, conv, deg, _, _ = ordering.run_component(X, np.zeros((0, N)), 1, cfg.cand_seed, ids, K, cfg.tol)
    n = torch.tensor([int(conv.sum())])
    dist.all_reduce(n, op=dist.ReduceOp.SUM)                    # the global converged count
    elig = conv if int(n.item()) > 0 else ~deg                   # reading A4, decided globally
    recs, rows = local_records(X, W, ids, elig, N)
    R = [torch.zeros(MAXC, 6, dtype=torch.float64) for _ in range(world)]
    Wl = [torch.zeros(MAXC, N, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(R, torch.from_numpy(recs))
    dist.all_gather(Wl, torch.from_numpy(rows))
    allr = torch.cat(R).numpy()
    allw = torch.cat(Wl).numpy()
    recl = [dict(upsilon=r[0], alpha=r[1], q=int(r[2]), size=int(r[3]), iters=0, valid=int(r[5])) for r in allr]
    m = oica.merge_records(recl, allw)
    q.put((rank, int(conv.sum()), int(allr[m["winner"]][2]), int(recs[:, 5].sum())))
    dist.destroy_process_group()


def test_a4_global_converged_count_two_ranks_gloo():
    cfg = datagen.PARITY["p_ragged"].with_(L=12)
    ds = datagen.make_dataset(cfg)
    Xw, _, _, _ = whiten.whiten(ds.X.numpy())
    X = Xw.astype(np.float32).astype(np.float64)
    # a cap at which the second half of the ids has no converged run and the first half has some
    # (at L = 12 the halves' fastest runs need 6 and 7 updates)
    _, _, st = ordering.extract(X, cfg.L, 200, cfg.tol, 1, cfg.cand_seed, keep_candidates=True)
    it = st[0].iters
    h = cfg.L // 2
    K = int(it[h:].min()) - 1
    assert K >= 1 and (it[:h] <= K).any(), (it[:h].min(), it[h:].min())
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_a4_worker, args=(r, world, port, K, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert out[0][1] > 0 and out[1][1] == 0                       # rank 1 converged nothing ...
    assert out[0][3] > 0 and out[1][3] == 0                       # ... and submits no record
    _, res = ordering.extract(X, cfg.L, K, cfg.tol, 1, cfg.cand_seed)
    assert not res[0].no_converged
    assert out[0][2] == out[1][2] == res[0].index                # the single-process decision
    assert out[0][1:3] == out[1][1:3] or out[0][2] == out[1][2]


# ---- hybrid L -> M tail (runtime.cu run_hybrid_tail): L-shard
# iterations in lock step on the GLOBAL active count until it falls to the tail threshold; then
# the still-active runs of every rank are all-gathered in rank order, iterated M-sharded (each rank
# sums its share of the samples, one fp64 all-reduce per iteration, identical epilogues), and the
# finished rows return to their owners by id; selection is the L-shard merge (reading A6)
def _hybrid_worker(rank, world, port, rows_thr, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = datagen.PARITY["p_ragged"].with_(L=40)
    ds = datagen.make_dataset(cfg)
    Xw, _, _, _ = whiten.whiten(ds.X.numpy())
    X = Xw.astype(np.float32).astype(np.float64)
    N, M = X.shape
    L, K = cfg.L, cfg.K
    lo, hi = L * rank // world, L * (rank + 1) // world
    ids = np.arange(lo, hi)
    from oracle import rng
    W = rng.candidates(cfg.cand_seed, 1, ids, N)
    W /= np.linalg.norm(W, axis=1, keepdims=True)
    conv = np.zeros(ids.size, dtype=bool)
    active = np.arange(ids.size)

    def epilogue(B, Gsum):
        G = Gsum / M - 3.0 * B                                   # eq. (5), global M
        Wn = G / np.linalg.norm(G, axis=1, keepdims=True)
        return Wn, ordering.convergence_distance(Wn, B) <= cfg.tol

    t = 0
    while t < K:                                                 # L-shard, lock step
        n = torch.tensor([active.size])
        dist.all_reduce(n, op=dist.ReduceOp.SUM)
        if int(n.item()) <= rows_thr:
            break
        t += 1
        if active.size:
            B = W[active]
            Wn, c = epilogue(B, ((B @ X) ** 3) @ X.T)
            W[active] = Wn
            conv[active[c]] = True
            active = active[~c]
    t_switch = t
    # C4: all-gather the active runs (id, row) in rank order
    cnts = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(cnts, torch.tensor([active.size]))
    cnts = [int(v.item()) for v in cnts]
    P = max(cnts + [1])
    pack = np.zeros((P, N + 1))
    pack[:active.size, 0] = ids[active]
    pack[:active.size, 1:] = W[active]
    allp = [torch.zeros(P, N + 1, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(allp, torch.from_numpy(pack))
    dense = np.concatenate([allp[r].numpy()[:cnts[r]] for r in range(world)])
    tid = dense[:, 0].astype(np.int64)
    TW = dense[:, 1:].copy()
    tconv = np.zeros(tid.size, dtype=bool)
    tact = np.arange(tid.size)
    m0, m1 = M * rank // world, M * (rank + 1) // world          # this rank's samples of the tail
    Xr = X[:, m0:m1]
    while tact.size and t < K:                                   # M-sharded tail iterations
        t += 1
        B = TW[tact]
        part = torch.from_numpy((((B @ Xr) ** 3) @ Xr.T).copy())
        dist.all_reduce(part, op=dist.ReduceOp.SUM)
        Wn, c = epilogue(B, part.numpy())
        TW[tact] = Wn
        tconv[tact[c]] = True
        tact = tact[~c]
    # finished rows back to their owners by global id
    for j, g in enumerate(tid):
        if lo <= g < hi:
            W[g - lo] = TW[j]
            conv[g - lo] = tconv[j]
    recs, rows = local_records(X, W, ids, conv, N)
    R = [torch.zeros(MAXC, 6, dtype=torch.float64) for _ in range(world)]
    Wl = [torch.zeros(MAXC, N, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(R, torch.from_numpy(recs))
    dist.all_gather(Wl, torch.from_numpy(rows))
    allr = torch.cat(R).numpy()
    allw = torch.cat(Wl).numpy()
    recl = [dict(upsilon=r[0], alpha=r[1], q=int(r[2]), size=int(r[3]), iters=0, valid=int(r[5])) for r in allr]
    m = oica.merge_records(recl, allw)
    q.put((rank, int(allr[m["winner"]][2]), float(allr[m["winner"]][1]), TW.tobytes(), t_switch, tid.size, t))
    dist.destroy_process_group()


def test_hybrid_tail_two_ranks_gloo():
    world, rows_thr = 2, 12
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_hybrid_worker, args=(r, world, port, rows_thr, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # the tail was entered with a real M-sharded phase, and both ranks hold bitwise-identical tail
    # iterates (same all-reduced sums) and make the same decision ...
    assert 0 < out[0][4] < out[0][6] and 0 < out[0][5] <= rows_thr
    assert out[0][1:] == out[1][1:]
    # ... which is the single-process oracle's (the sample sums are re-associated by rank)
    cfg = datagen.PARITY["p_ragged"].with_(L=40)
    ds = datagen.make_dataset(cfg)
    Xw, _, _, _ = whiten.whiten(ds.X.numpy())
    X = Xw.astype(np.float32).astype(np.float64)
    _, res = ordering.extract(X, cfg.L, cfg.K, cfg.tol, 1, cfg.cand_seed)
    assert out[0][1] == res[0].index
    assert out[0][2] == pytest.approx(res[0].alpha, rel=1e-10)
