#!/usr/bin/env python
"""Write the float64 ORACLE's results for full-size configs to tests/golden/ (SURVEY §8(c) tiers A/B).

    python scripts/make_golden.py cfg0 cfg1 cfg2 cfg3_L256 [--threads 8]

Calls only oracle/ and datagen/ (no CUDA path): the stored expected values are the oracle's.
Inputs: datagen's seeded raw signals on the CPU, whitened by the oracle in fp64 and cast to
fp32 (the GPU tests rebuild exactly these fp32 values and check the stored SHA-256).
  tier A: cfgs 0 and 1 (3 data/candidate seeds each), cfg 2 at full L, all N_out components
  tier B: cfgs 3 and 4 at full N, M with L' = 256 (candidate ids 0..255: an exact sub-problem),
          all 64 components (cfg 3) / the first 16 (cfg 4)
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

JOBS = {
    "cfg0_s0": ("cfg0_tiny", 0, None, None),
    "cfg0_s1": ("cfg0_tiny", 1, None, None),
    "cfg0_s2": ("cfg0_tiny", 2, None, None),
    "cfg1": ("cfg1_artificial", 0, None, None),
    "cfg1_s1": ("cfg1_artificial", 1, None, None),
    "cfg1_s2": ("cfg1_artificial", 2, None, None),
    "cfg2": ("cfg2_eeg_shaped", 0, None, None),
    "cfg3_L256": ("cfg3_large", 0, 256, None),   # all 64 components (105 s per 8 on 8 cores)
    "cfg4_L256": ("cfg4_scaling", 0, 256, 16),   # 16 of 32 components (~90 s each)
}


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


def run(name, out_dir):
    from oracle import ordering
    cfg = job_config(name)
    t0 = time.time()
    X32 = prepared_input(cfg)
    W, res = ordering.extract(X32.astype(np.float64), cfg.L, cfg.K, cfg.tol, cfg.N_out, cfg.cand_seed)
    rec = {"job": name, "config": cfg.name, "N": cfg.N, "M": cfg.M, "L": cfg.L, "K": cfg.K, "tol": cfg.tol,
           "N_out": cfg.N_out, "data_seed": cfg.data_seed, "cand_seed": cfg.cand_seed, "x32_sha256": digest(X32), "x32_fingerprint": fingerprint(X32),
           "oracle_seconds": time.time() - t0,
           "components": [{"i": r.i, "index": int(r.index), "alpha": r.alpha, "upsilon": r.upsilon,
                           "near_tie": bool(r.near_tie), "cluster_size": int(r.cluster_size),
                           "n_converged": int(r.n_converged), "sum_active": int(r.sum_active),
                           "n_iter": int(r.n_iter), "w": [float(v) for v in r.w]} for r in res]}
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
    ap.add_argument("jobs", nargs="+", choices=sorted(JOBS))
    ap.add_argument("--fingerprint-only", action="store_true")
    ap.add_argument("--threads", type=int, default=max(1, len(os.sched_getaffinity(0))))
    ap.add_argument("--out", default=os.path.join(ROOT, "tests", "golden"))
    a = ap.parse_args()
    from threadpoolctl import threadpool_limits
    with threadpool_limits(a.threads, user_api="blas"):
        for j in a.jobs:
            if a.fingerprint_only:
                add_fingerprint(j, a.out)
            else:
                run(j, a.out)


if __name__ == "__main__":
    main()
