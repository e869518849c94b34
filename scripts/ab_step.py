#!/usr/bin/env python
"""A/B of the step kernel between two builds of the library (dev aid): extracts components 1..k of
a config with host-launched iterations (per-step CUDA-event timing) and prints the step kernel's
algorithmic TFLOP/s.  Run once per library: OICA_LIB=<lib.so> python scripts/ab_step.py cfg2_eeg_shaped 6"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import datagen  # noqa: E402
from paper_2408_17118_b200 import oica  # noqa: E402

cfg = datagen.get(sys.argv[1])
k = int(sys.argv[2]) if len(sys.argv) > 2 else 6
ds = datagen.make_dataset(cfg, device="cuda", dtype=torch.float32, keep_sources=False)
X = ds.X.contiguous()
with oica.Context(0, oica.PREC_AUTO) as ctx:
    Xw = torch.empty_like(X)
    ctx.whiten(X, Xw)
    ctx.set_data(Xw)
    ctx.init_candidates(cfg.cand_seed, cfg.L)
    ctx.extract(2, cfg.K, cfg.tol, flags=oica.EAGER)
    ctx.reset_stats()
    r = ctx.extract(k, cfg.K, cfg.tol, flags=oica.EAGER)
    st = ctx.stats()
print(json.dumps({"lib": os.path.basename(oica.LIB_PATH), "config": cfg.name, "components": k,
                  "step_tflops": st["step_flops"] / (st["step_ms"] / 1e3) / 1e12, "step_ms": st["step_ms"],
                  "launches": st["step_launches"], "index": [int(v) for v in r.index]}))
