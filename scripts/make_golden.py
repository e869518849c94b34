#!/usr/bin/env python
"""Write the float64 ORACLE's results for full-size configs to tests/golden/ (SURVEY §8(c) tiers A/B).

    python scripts/make_golden.py cfg0 cfg1 cfg2 cfg3_L256 [--threads 8]

Calls only oracle/ and datagen/ (no CUDA path): the stored expected values are the oracle's.
Inputs: datagen's seeded raw signals on the CPU, whitened by the oracle in fp64 and cast to
fp32 (the GPU tests rebuild exactly these fp32 values and check the stored SHA-256).
  tier A: cfgs 0 and 1 (3 data/candidate seeds each), cfg 2 at full L, all N_out components
  tier B: cfgs 3 and 4 at full N, M with L' = 256 (candidate ids 0..255: an exact sub-problem),
          all 64 (cfg 3) / all 32 (cfg 4) components; `--resume` continues a stored golden from
          its last component (the prefix is the stored ORACLE rows)
  tier C: `cfg3_tierC` / `cfg4_tierC`: for every component i, a seeded sample of 256 candidate
          ids from [256, L) (chosen without any GPU output) replayed by the oracle's candidate
          phase on the tier-B golden's own prefix (oracle rows 1..i-1): final w (fp32), alpha at
          the final w, iterations, converged/degenerate flags -> tests/golden/tierc_<cfg>.npz.
          With the tier-B result it certifies the full-L selection (SURVEY §8(c) tier C).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import datagen  # noqa: E402  (input recipe only)

JOBS = {
    "cfg0_s0": ("cfg0_tiny", 0, None, None),
    "cfg0_s1": ("cfg0_tiny", 1, None, None),
    "cfg0_s2": ("cfg0_tiny", 2, None, None),
    "cfg1": ("cfg1_artificial", 0, None, None),
    "cfg1_s1": ("cfg1_artificial", 1, None, None),
    "cfg1_s2": ("cfg1_artificial", 2, None, None),
    "cfg2": ("cfg2_eeg_shaped", 0, None, None),
    "cfg3_L256": ("cfg3_large", 0, 256, None),   # all 64 components (105 s per 8 on 8 cores)
    "cfg4_L256": ("cfg4_scaling", 0, 256, None),  # all 32 components (~70 s each on 8 cores)
}
# tier C: (tier-B golden it extends, sample size per component, sample seed base)
TIER_C = {"cfg3_tierC": ("cfg3_L256", 256, 9003), "cfg4_tierC": ("cfg4_L256", 256, 9004)}


def tierc_ids(L_sub, L, n, seed_base, i):
    """Seeded sample of n global ids from [L_sub, L) for component i (no GPU input)."""
    rs = np.random.default_rng(seed_base * 1000 + i)
    return np.sort(rs.choice(np.arange(L_sub, L, dtype=np.int64), n, replace=False))


def job_config(name):
    import datagen
    cfg_name, seed_shift, L, N_out = JOBS[name]
    cfg = datagen.get(cfg_name)
    cfg = cfg.with_(data_seed=cfg.data_seed + 100 * seed_shift, cand_seed=cfg.cand_seed + 100 * seed_shift)
    if L is not None:
        cfg = cfg.with_(L=L)
    if N_out is not None:
        cfg = cfg.with_(N_out=N_out)
    return cfg


def prepared_input(cfg):
    """Seeded raw signals (CPU generator) -> oracle whitening (fp64) -> fp32 (the parity input)."""
    import datagen
    from oracle import whiten
    ds = datagen.make_dataset(cfg, keep_sources=False)
    Xw, _, _, _ = whiten.whiten(ds.X.numpy())
    return np.ascontiguousarray(Xw.astype(np.float32))


def digest(X32):
    return hashlib.sha256(X32.tobytes()).hexdigest()


def fingerprint(X32):
    """Tolerant identity of the input: BLAS-dependent summation order in the data generation and
    whitening can change the last bits of X32 between CPUs, which leaves every stored result
    within its gates; the test checks the input against these values (row sums, fixed samples)."""
    rs = np.random.default_rng(0)
    idx = rs.integers(0, X32.size, 256)
    return {"row_sums": [float(v) for v in X32.astype(np.float64).sum(axis=1)],
            "sample_index": [int(v) for v in idx], "sample_value": [float(v) for v in X32.reshape(-1)[idx]]}


def _components(res):
    return [{"i": r.i, "index": int(r.index), "alpha": r.alpha, "upsilon": r.upsilon,
             "near_tie": bool(r.near_tie), "cluster_size": int(r.cluster_size),
             "n_converged": int(r.n_converged), "sum_active": int(r.sum_active),
             "n_iter": int(r.n_iter), "w": [float(v) for v in r.w]} for r in res]


def resume(name, out_dir):
    """Continue a stored golden to cfg.N_out components: prefix = the stored oracle rows."""
    from oracle import ordering
    path = os.path.join(out_dir, f"oracle_{name}.json")
    rec = json.load(open(path))
    cfg = job_config(name)
    have = len(rec["components"])
    if have >= cfg.N_out:
        print(name, "already has", have, "components", flush=True)
        return
    t0 = time.time()
    X32 = prepared_input(cfg)
    assert digest(X32) == rec["x32_sha256"], "input differs from the one the golden was computed on"
    X64 = X32.astype(np.float64)
    del X32
    for k in range(have, cfg.N_out):          # one component per call: checkpoint after each
        Wp = np.array([c["w"] for c in rec["components"]])
        t1 = time.time()
        _, res = ordering.extract(X64, cfg.L, cfg.K, cfg.tol, k + 1, cfg.cand_seed, W_prefix=Wp)
        rec["components"] += _components(res)
        rec["N_out"] = len(rec["components"])
        rec["oracle_seconds"] = rec["oracle_seconds"] + (time.time() - t1)
        json.dump(rec, open(path, "w"))
        print(name, "component", k + 1, "index", res[0].index, round(time.time() - t1, 1), "s", flush=True)
    print(name, "resumed in", round(time.time() - t0, 1), "s", flush=True)


def tier_c(name, out_dir):
    """Oracle replays of sampled candidates on the tier-B golden's prefix (see module doc)."""
    from oracle import ordering
    base, n, seed_base = TIER_C[name]
    g = json.load(open(os.path.join(out_dir, f"oracle_{base}.json")))
    cfg = datagen.get(g["config"])
    assert cfg.data_seed == g["data_seed"] and cfg.cand_seed == g["cand_seed"]
    X32 = prepared_input(cfg)
    assert digest(X32) == g["x32_sha256"], "input differs from the tier-B golden's"
    X64 = X32.astype(np.float64)
    del X32
    Wg = np.array([c["w"] for c in g["components"]])
    C = len(g["components"])
    out = {"ids": np.zeros((C, n), np.int64), "W": np.zeros((C, n, cfg.N), np.float32),
           "alpha": np.full((C, n), np.nan), "iters": np.zeros((C, n), np.int32),
           "converged": np.zeros((C, n), bool), "degenerate": np.zeros((C, n), bool),
           "seconds": np.zeros(C)}
    part = os.path.join(out_dir, f"tierc_{g['config']}.partial.npz")
    start = 0
    if os.path.exists(part):
        z = np.load(part)
        start = int(z["done"])
        for k in out:
            out[k] = z[k]
    for k in range(start, C):
        t1 = time.time()
        i = k + 1
        ids = tierc_ids(g["L"], cfg.L, n, seed_base, i)
        W, iters, conv, deg, _, _ = ordering.run_component(X64, Wg[:k], i, cfg.cand_seed, ids, cfg.K, cfg.tol)
        a = np.full(n, np.nan)
        e = ~deg
        a[e] = ordering.alpha_rows(W[e], X64)
        out["ids"][k], out["W"][k], out["alpha"][k] = ids, W.astype(np.float32), a
        out["iters"][k], out["converged"][k], out["degenerate"][k] = iters, conv, deg
        out["seconds"][k] = time.time() - t1
        np.savez(part, done=k + 1, **out)
        print(name, "component", i, "converged", int(conv.sum()), "/", n, round(out["seconds"][k], 1), "s", flush=True)
    meta = {"job": name, "golden": f"oracle_{base}.json", "config": g["config"], "L_sub": g["L"], "L": cfg.L,
            "K": cfg.K, "tol": cfg.tol, "n_sample": n, "sample_seed_base": seed_base, "x32_sha256": g["x32_sha256"]}
    np.savez_compressed(os.path.join(out_dir, f"tierc_{g['config']}.npz"), meta=json.dumps(meta), **out)
    os.remove(part)
    print(name, "done in", round(float(out["seconds"].sum()), 1), "s", flush=True)


def run(name, out_dir):
    from oracle import ordering
    cfg = job_config(name)
    t0 = time.time()
    X32 = prepared_input(cfg)
    W, res = ordering.extract(X32.astype(np.float64), cfg.L, cfg.K, cfg.tol, cfg.N_out, cfg.cand_seed)
    rec = {"job": name, "config": cfg.name, "N": cfg.N, "M": cfg.M, "L": cfg.L, "K": cfg.K, "tol": cfg.tol,
           "N_out": cfg.N_out, "data_seed": cfg.data_seed, "cand_seed": cfg.cand_seed, "x32_sha256": digest(X32), "x32_fingerprint": fingerprint(X32),
           "oracle_seconds": time.time() - t0, "components": _components(res)}
    path = os.path.join(out_dir, f"oracle_{name}.json")
    json.dump(rec, open(path, "w"))
    print(name, "done in", round(rec["oracle_seconds"], 1), "s ->", path, flush=True)


def add_fingerprint(name, out_dir):
    """Add the input fingerprint to an existing golden (the oracle results are not recomputed)."""
    path = os.path.join(out_dir, f"oracle_{name}.json")
    rec = json.load(open(path))
    X32 = prepared_input(job_config(name))
    assert digest(X32) == rec["x32_sha256"], "input differs from the one the golden was computed on"
    rec["x32_fingerprint"] = fingerprint(X32)
    json.dump(rec, open(path, "w"))
    print(name, "fingerprint added", flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("jobs", nargs="+", choices=sorted(JOBS) + sorted(TIER_C))
    ap.add_argument("--fingerprint-only", action="store_true")
    ap.add_argument("--resume", action="store_true", help="continue stored goldens to N_out components")
    ap.add_argument("--threads", type=int, default=max(1, len(os.sched_getaffinity(0))))
    ap.add_argument("--out", default=os.path.join(ROOT, "tests", "golden"))
    a = ap.parse_args()
    from threadpoolctl import threadpool_limits
    with threadpool_limits(a.threads, user_api="blas"):
        for j in a.jobs:
            if j in TIER_C:
                tier_c(j, a.out)
            elif a.resume:
                resume(j, a.out)
            elif a.fingerprint_only:
                add_fingerprint(j, a.out)
            else:
                run(j, a.out)


if __name__ == "__main__":
    main()
