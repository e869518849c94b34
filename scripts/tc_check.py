#!/usr/bin/env python
"""Quick check of the fused step (TC and FP32) against the float64 oracle across padded-N variants."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import datagen  # noqa: E402
from datagen import Config  # noqa: E402
from oracle import ordering, rng, whiten  # noqa: E402
from paper_2408_17118_b200 import oica  # noqa: E402

cases = [(12, 5003, 300), (32, 20000, 257), (40, 12000, 130), (128, 40000, 300), (256, 40000, 300)]
if len(sys.argv) > 1:
    cases = [c for c in cases if str(c[0]) in sys.argv[1:]]
for N, M, L in cases:
    cfg = Config(f"c{N}", N, M, L, 200, 1e-10, 1, (("laplace", N // 2), ("gg_uniform", N - N // 2, 0.5, 1.5)),
                 data_seed=11 + N, cand_seed=12)
    ds = datagen.make_dataset(cfg)
    Xw, _, _, _ = whiten.whiten(ds.X.numpy())
    X32 = np.ascontiguousarray(Xw.astype(np.float32))
    X64 = X32.astype(np.float64)
    W = rng.candidates(7, 1, np.arange(L), N)
    W /= np.linalg.norm(W, axis=1, keepdims=True)
    Gref, s4ref = ordering.batch_step(W, X64)
    Graw = (Gref + 3.0 * W) * M
    bound = (np.abs(W @ X64) ** 3) @ np.abs(X64).T
    for prec in (oica.PREC_FP32, oica.PREC_TC):
        with oica.Context(0, prec) as ctx:
            ctx.set_data(torch.from_numpy(X32).cuda())
            ctx.init_candidates(1, L)
            G = torch.zeros(L, N, dtype=torch.float64, device="cuda")
            s4 = torch.zeros(L, dtype=torch.float64, device="cuda")
            t0 = time.time()
            ctx.fixed_point_step(torch.from_numpy(W).cuda(), G, s4)
            torch.cuda.synchronize()
            dt = time.time() - t0
            g = G.cpu().numpy()
            err = np.abs(g - Graw) / bound
            rel = np.linalg.norm(g - Graw, axis=1) / np.linalg.norm(Graw, axis=1)
            s4e = np.abs(s4.cpu().numpy() - s4ref) / s4ref
            print(f"N={N} M={M} L={L} prec={prec} slots={ctx.stats()['slots']} max|dG|/bound={err.max():.3e} "
                  f"max row rel={rel.max():.3e} s4 rel={s4e.max():.3e} t={dt:.3f}s", flush=True)
