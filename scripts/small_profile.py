#!/usr/bin/env python
"""Small-problem timing: wall/device time of a whole extraction where the host
round trips, not the contraction, set the pace -- cfg 1 (all 32 components) and the paper's Exp. 1
(N = 20, M = 1e4, K = 30, tol 5e-13) at L = 20 / 100.  Prints one JSON line per case.

    python scripts/small_profile.py [--reps 5] [--cases cfg1,exp1_L20,exp1_L100]
"""
import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import datagen  # noqa: E402
from paper_2408_17118_b200 import oica  # noqa: E402


def case(name, eager):
    fl = oica.EAGER if eager else 0
    if name == "cfg1":
        return datagen.get("cfg1_artificial"), fl
    if name == "cfg2":
        return datagen.get("cfg2_eeg_shaped"), fl
    L = int(name.split("_L")[1])
    return datagen.EXPERIMENTS["exp1_ordering"].with_(L=L), fl


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--cases", default="cfg1,exp1_L20,exp1_L100")  # also: cfg2 (EEG-shaped, 32 components)
    ap.add_argument("--eager", action="store_true")
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    for name in a.cases.split(","):
        cfg, flags = case(name, a.eager)
        ds = datagen.make_dataset(cfg, device=dev, dtype=torch.float32, keep_sources=False)
        X = ds.X.contiguous()
        del ds
        st = torch.cuda.Stream()
        with oica.Context(0, oica.PREC_AUTO, stream=st) as ctx:
            Xw = torch.empty_like(X)
            ctx.whiten(X, Xw)
            ctx.set_data(Xw)
            ctx.init_candidates(cfg.cand_seed, cfg.L)
            ctx.extract(cfg.N_out, cfg.K, cfg.tol, flags=flags)   # warm-up (allocations, graphs)
            ctx.reset_stats()
            walls, devs = [], []
            for _ in range(a.reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                e0.record(st)
                r = ctx.extract(cfg.N_out, cfg.K, cfg.tol, flags=flags)
                e1.record(st)
                torch.cuda.synchronize()
                walls.append(time.perf_counter() - t0)
                devs.append(e0.elapsed_time(e1) / 1e3)
            s = ctx.stats()
        flops = sum(int(r.sum_active[k]) * (4.0 * cfg.N * cfg.M + 3.0 * cfg.M) for k in range(r.n_extracted))
        print(json.dumps({"case": name, "N": cfg.N, "M": cfg.M, "L": cfg.L, "K": cfg.K, "components": int(r.n_extracted),
                          "wall_ms_median": 1e3 * float(np.median(walls)), "device_ms_median": 1e3 * float(np.median(devs)),
                          "tflops": flops / float(np.median(devs)) / 1e12,
                          "launches_per_extract": s["kernel_launches"] / a.reps, "iterations_per_extract": s["iterations"] / a.reps,
                          "step_ms_per_extract": s["step_ms"] / a.reps, "graph_ms_per_extract": s["graph_ms"] / a.reps,
                          "graph_iterations_per_extract": s["graph_iterations"] / a.reps,
                          "precision": s["precision"],
                          # result digest (W, alpha, index, row-iterations): bitwise comparisons across builds
                          "result_sha": hashlib.sha256(np.ascontiguousarray(r.W).tobytes() + r.alpha.tobytes() +
                                                       r.index.tobytes() + np.asarray(r.sum_active).tobytes()
                                                       ).hexdigest()[:16]}), flush=True)


if __name__ == "__main__":
    main()
