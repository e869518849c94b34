#!/usr/bin/env python
"""Per-iteration log of an extraction: where an iteration stops being tensor-bound.

    python scripts/iteration_log.py cfg4_scaling [--components 2] [--out gpurun_out/iterlog_cfg4.json]

Synthetic data of the config's recipe (datagen, on the device) whitened by liboica, then
oica_extract_components for the first components; prints and stores one record per iteration:
active runs L_act, step-kernel ms (CUDA events), algorithmic TFLOP/s, and the floor an iteration
cannot beat however few rows are active: streaming the fp16 X plane once from HBM (2 N M bytes at
the measured copy bandwidth).
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import datagen  # noqa: E402
from paper_2408_17118_b200 import oica  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--components", type=int, default=2)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    cfg = datagen.get(a.config)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    bw = float(peaks["hbm_gbs"])   # measured copy bandwidth (read + write bytes), GB/s
    dev = torch.device("cuda:0")
    with oica.Context(0, oica.PREC_AUTO) as ctx:
        ds = datagen.make_dataset(cfg, device=dev, dtype=torch.float32, keep_sources=False)
        X = ds.X.contiguous()
        del ds
        Xw = torch.empty_like(X)
        ctx.whiten(X, Xw)
        del X
        ctx.set_data(Xw)
        ctx.init_candidates(cfg.cand_seed, cfg.L)
        # EAGER: host-launched iterations, each step timed by its own events (the device-side loop
        # of short iterations runs the same arithmetic but is not timed iteration by iteration)
        ctx.extract(1, cfg.K, cfg.tol, flags=oica.EAGER)   # warm-up
        res = ctx.extract(a.components, cfg.K, cfg.tol, flags=oica.EAGER)
        log = ctx.iteration_log()
        prec = ctx.stats()["precision"]
    floor_ms = 2.0 * cfg.N * cfg.M / (bw * 1e9) * 1e3
    for r in log:
        r["tflops"] = r["flops"] / (r["step_ms"] * 1e-3) / 1e12
        r["x_stream_floor_ms"] = floor_ms
        print(f"comp {r['component']:3d} it {r['iteration']:3d} L_act {r['L_act']:7d} fine {r['fine_rows']:6d} "
              f"{r['step_ms']:9.3f} ms {r['tflops']:8.1f} TFLOP/s  (X-stream floor {floor_ms:.3f} ms)", flush=True)
    out = {"config": cfg.name, "N": cfg.N, "M": cfg.M, "L": cfg.L, "precision": prec, "hbm_gbps": bw,
           "x_stream_floor_ms": floor_ms, "components": [int(v) for v in res.index[:res.n_extracted]],
           "records": log}
    if a.out:
        os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
        json.dump(out, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
