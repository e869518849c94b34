#!/usr/bin/env python
"""Time k_step_tc variants (dev experiment): python scripts/tc_variants.py <mode> [N]
Runs oica_fixed_point_step on random data at the cfg4/cfg3 shapes; prints algorithmic TFLOP/s.
The variants (OICA_TC_EPI, OICA_TC_CL, OICA_TC_RING, ...) exist only in the experiment build:
python -m paper_2408_17118_b200.build --experiments, then OICA_LIB=.../liboica_exp.so."""
import json
import os
import sys
import threading
import time

import numpy as np
import torch

sys.path.insert(0, os.environ.get("OICA_PKG_ROOT") or os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_17118_b200 import oica  # noqa: E402

shapes = {256: (4_000_000, 65536), 128: (1_000_000, 16384), 64: (250_000, 4096), 32: (250_000, 4096)}
Ns = [int(a) for a in sys.argv[2:]] or [256, 128]
for N in Ns:
    M, L = shapes[N]
    g = torch.Generator(device="cuda").manual_seed(1)
    X = torch.randn(N, M, device="cuda", generator=g)
    W = torch.randn(L, N, device="cuda", dtype=torch.float64, generator=g)
    W /= W.norm(dim=1, keepdim=True)
    G = torch.empty(L, N, device="cuda", dtype=torch.float64)
    s4 = torch.empty(L, device="cuda", dtype=torch.float64)
    with oica.Context(0, oica.PREC_TC) as ctx:
        ctx.set_data(X)
        ctx.init_candidates(1, L)
        ctx.fixed_point_step(W, G, s4)
        ctx.reset_stats()
        ctx.fixed_point_step(W, G, s4)
        reps = max(3, int(1500.0 / max(ctx.stats()["step_ms"], 1e-3)))   # >= ~1.5 s timed (steady clocks)
        ctx.reset_stats()
        clk, stop = [], [False]

        def poll():
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(0)
            while not stop[0]:
                clk.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                time.sleep(0.02)
        th = threading.Thread(target=poll, daemon=True)
        th.start()
        for _ in range(reps):
            ctx.fixed_point_step(W, G, s4)
        stop[0] = True
        th.join()
        st = ctx.stats()
    ms = st["step_ms"] / reps
    tf = L * 4.0 * N * M / (ms / 1e3) / 1e12
    print(json.dumps({"mode": os.environ.get("OICA_TC_EPI", "0"), "N": N, "M": M, "L": L, "ms": ms, "tflops": tf, "sm_mhz": float(np.median(clk)) if clk else None,
                      "tflops_per_ghz": tf / (float(np.median(clk)) / 1e3) if clk else None,
                      "g_norm": float(G.norm())}), flush=True)
    del X, W, G, s4
    torch.cuda.empty_cache()
