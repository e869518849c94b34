#!/usr/bin/env python
"""Small extractions for compute-sanitizer (memcheck / racecheck / synccheck): the FP32 step (K2b)
and the tensor-core step (K2a), the fused update (few-row and many-row variants, the 1024-thread
compaction), the device-side loop (CUDA graph) and host-launched iterations, the selection (K5).

    compute-sanitizer --tool memcheck python scripts/sanitize_run.py
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import datagen  # noqa: E402
from datagen import Config  # noqa: E402
from paper_2408_17118_b200 import oica  # noqa: E402

cases = [
    (Config("san_fp32", 8, 2000, 64, 200, 1e-10, 3, (("laplace", 4), ("gg_uniform", 4, 0.5, 1.5)),
            data_seed=11, cand_seed=12), oica.PREC_FP32),
    (Config("san_tc", 32, 20000, 160, 200, 1e-10, 2, (("laplace", 16), ("gg_uniform", 16, 0.5, 1.5)),
            data_seed=13, cand_seed=14), oica.PREC_TC),
    (Config("san_wide", 144, 20000, 2100, 200, 1e-10, 1, (("gg_uniform", 144, 0.5, 1.9),),
            data_seed=15, cand_seed=16), oica.PREC_TC),   # > 2048 rows: the many-row update + compaction
]
only = sys.argv[1:] or None
for cfg, prec in cases:
    if only and cfg.name not in only:
        continue
    ds = datagen.make_dataset(cfg, device="cuda", dtype=torch.float32, keep_sources=False)
    X = ds.X.contiguous()
    with oica.Context(0, prec) as ctx:
        Xw = torch.empty_like(X)
        ctx.whiten(X, Xw)
        ctx.set_data(Xw)
        ctx.init_candidates(cfg.cand_seed, cfg.L)
        a = ctx.extract(cfg.N_out, cfg.K, cfg.tol)
        b = ctx.extract(cfg.N_out, cfg.K, cfg.tol, flags=oica.EAGER)
        c = ctx.extract(cfg.N_out, 4, cfg.tol, flags=oica.INCLUDE_UNCONVERGED)
        assert np.array_equal(a.W, b.W)
        print(cfg.name, "ok", list(a.index), list(c.index), flush=True)
