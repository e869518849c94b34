#!/usr/bin/env python
"""Dev aid (experiment build): hash of the tensor-core step's G for one set of inputs, so two step
layouts (OICA_TC_RING) can be checked bitwise equal.  Prints one JSON line per (N, L, fine rows).

    OICA_LIB=.../liboica_exp.so OICA_TC_RING=24 python scripts/layout_bitwise.py
"""
import hashlib
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_17118_b200 import oica  # noqa: E402

for N, L, M in ((16, 300, 40_000), (32, 1024, 20_000), (48, 700, 50_000), (64, 4096, 250_000), (64, 130, 250_000)):
    for nfine in (0, 37):
        g = torch.Generator(device="cuda").manual_seed(N + L)
        X = torch.randn(N, M, device="cuda", generator=g)
        W = torch.randn(L, N, device="cuda", dtype=torch.float64, generator=g)
        W /= W.norm(dim=1, keepdim=True)
        G = torch.zeros(L, N, device="cuda", dtype=torch.float64)
        s4 = torch.zeros(L, device="cuda", dtype=torch.float64)
        fine = None
        if nfine:
            fine = np.zeros(L, np.uint8)
            fine[L - nfine:] = 1
        with oica.Context(0, oica.PREC_TC) as ctx:
            ctx.set_data(X)
            ctx.init_candidates(1, L)
            ctx.fixed_point_step(W, G, s4, fine)
            torch.cuda.synchronize()
        h = hashlib.sha1(G.cpu().numpy().tobytes()).hexdigest()[:16]
        print(json.dumps({"ring": os.environ.get("OICA_TC_RING", "0"), "N": N, "L": L, "M": M, "fine": nfine,
                          "G_sha1": h}), flush=True)
