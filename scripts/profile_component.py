#!/usr/bin/env python
"""Profile one component of an extraction (dev aid): extracts components 1..k-1, then component k
inside an NVTX range "comp" (for `ncu --nvtx --nvtx-include comp/`).

    python scripts/profile_component.py cfg2_eeg_shaped 30
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import datagen  # noqa: E402
from paper_2408_17118_b200 import oica  # noqa: E402

cfg = datagen.get(sys.argv[1])
k = int(sys.argv[2])
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
    r = ctx.extract(k - 1, cfg.K, cfg.tol)
    W = np.array(r.W[: k - 1])
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push("comp")
    r = ctx.extract(k, cfg.K, cfg.tol, W_prefix=W)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
    print("component", k, "n_iter", int(r.n_iter[k - 1]), "sum_active", int(r.sum_active[k - 1]))
