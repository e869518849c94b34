import time, torch, numpy as np, sys
sys.path.insert(0, "/root/repo")
import datagen
from paper_2408_17118_b200 import oica
cfg = datagen.get(sys.argv[1])
dev = torch.device("cuda:0")
st = torch.cuda.Stream()
with oica.Context(0, oica.PREC_AUTO, stream=st) as ctx:
    ds = datagen.make_dataset(cfg, device=dev, dtype=torch.float32, keep_sources=False)
    X = ds.X.contiguous(); Xw = torch.empty_like(X); ctx.whiten(X, Xw)
    ctx.set_data(Xw); ctx.init_candidates(cfg.cand_seed, cfg.L)
    Xh = torch.empty(Xw.shape, dtype=torch.float32, pin_memory=True); Xh.copy_(Xw)
    r = ctx.extract(1, cfg.K, cfg.tol)
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ctx.set_data_host_ptr(Xh.data_ptr(), cfg.N, cfg.M, cfg.M)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        r = ctx.extract(2, cfg.K, cfg.tol, W_prefix=np.array(r.W[:1]))
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        print(f"set_data_host call {1e3*(t1-t0):.3f} ms, upload done {1e3*(t2-t0):.3f} ms, extract {1e3*(t3-t2):.3f} ms")
    # the bench's e2e leg: no per-step synchronisation, CUDA events on the context stream
    W = np.array(ctx.extract(6, cfg.K, cfg.tol).W[:6])
    for leg in ("device", "host"):
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(st)
        t0 = time.perf_counter()
        for k in range(3, 6):
            if leg == "host":
                ctx.set_data_host_ptr(Xh.data_ptr(), cfg.N, cfg.M, cfg.M)
            ctx.extract(k + 1, cfg.K, cfg.tol, W_prefix=W[:k])
        f1.record(st)
        torch.cuda.synchronize()
        print(leg, "events", f0.elapsed_time(f1) / 3, "ms/step; wall", 1e3 * (time.perf_counter() - t0) / 3)
