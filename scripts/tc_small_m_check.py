import json, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
sys.path.insert(0, "/root/repo/tests")
from test_gpu_golden import _input
from paper_2408_17118_b200 import oica
for name in ["cfg1", "cfg0_s0", "cfg0_s1", "cfg0_s2"]:
    g = json.load(open(f"/root/repo/tests/golden/oracle_{name}.json"))
    cfg, X32 = _input(g)
    for prec in (oica.PREC_FP32, oica.PREC_TC):
        with oica.Context(0, prec) as ctx:
            ctx.set_data(torch.from_numpy(X32).cuda()); ctx.init_candidates(cfg.cand_seed, cfg.L)
            ctx.extract(2, cfg.K, cfg.tol)
            torch.cuda.synchronize(); t0 = time.time()
            r = ctx.extract(cfg.N_out, cfg.K, cfg.tol)
            torch.cuda.synchronize(); dt = time.time() - t0
        comps = g["components"]
        match = sum(int(r.index[k]) == c["index"] for k, c in enumerate(comps))
        cos = min(abs(float(r.W[k] @ np.array(c["w"]))) for k, c in enumerate(comps))
        rel = max(abs(r.alpha[k] - c["alpha"]) / (c["alpha"] + 3) for k, c in enumerate(comps))
        print(name, "prec", prec, "time", round(dt, 4), "match", match, "/", len(comps), "min cos", cos, "max rel", rel,
              "unconv", int(r.n_unconverged.sum()), flush=True)
