#!/usr/bin/env python
"""Dev aid: one cfg-2 extraction of the first components with host-launched iterations (EAGER), so
ncu sees every step launch (the tail iterations' grids and durations)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import datagen  # noqa: E402
from paper_2408_17118_b200 import oica  # noqa: E402

cfg = datagen.get(sys.argv[1] if len(sys.argv) > 1 else "cfg2_eeg_shaped")
k = int(sys.argv[2]) if len(sys.argv) > 2 else 2
ds = datagen.make_dataset(cfg, device="cuda", dtype=torch.float32, keep_sources=False)
X = ds.X.contiguous()
with oica.Context(0, oica.PREC_AUTO) as ctx:
    Xw = torch.empty_like(X)
    ctx.whiten(X, Xw)
    ctx.set_data(Xw)
    ctx.init_candidates(cfg.cand_seed, cfg.L)
    r = ctx.extract(k, cfg.K, cfg.tol, flags=oica.EAGER)
print(list(r.index[:k]), list(r.n_iter[:k]))
