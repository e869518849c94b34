#!/usr/bin/env python
"""Benchmark of the Fast Ordering ICA hot path on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg4_scaling] [--impl oica|reference]

A STEP is one pass of the whole hot path for one component:
candidate draw + projection, the fixed-point do-while over the active set (fused
GEMM-cube-GEMM + fp64 epilogue + compaction) and the device-side selection/accept.  Warm-up
steps extract components 1..W, timed steps W+1..W+K (each step is the next component, as in
the paper's outer loop).  value = algorithmic TFLOP/s of the timed steps,
sum_i sum_t L_act(i,t) (4 N M + 3 M) / device time (max over ranks); inputs (X, 4 N M bytes)
are larger than L2, so no flush is needed between steps.

--impl reference times the float64 CPU oracle (the reference arm for this tier) on a bounded
sample of the same workload.  Multi-GPU: launch under torchrun; L-shard (candidates split,
one NCCL exchange per component).  One JSON line is printed by rank 0.

Data (--data): `golden` (default) regenerates on the host exactly the raw signals of the
config's stored oracle golden (tests/golden/oracle_<cfg>.json, written by scripts/make_golden.py
from oracle/ + datagen/), whitens them on the device (oica_whiten) and, after the run, compares
the all-components leg's accepted indices / rows / objectives with the stored oracle results
(`golden_match`; the file is read as data, no oracle code runs).  `device` draws the same recipe
with the device generator (faster set-up, a different draw, no golden).  Under torchrun rank 0
prepares the data and oica_distribute_data broadcasts it (C3).

The product library only: bench.py refuses to run when OICA_LIB or an experiment variable of
the -DOICA_EXPERIMENTS build is set.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ordering-ICA fixed-point TFLOP/s (% tensor peak) and seconds to extract all N"
DEFAULT_CONFIG = "cfg4_scaling"
REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
           0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
           0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}


# experiment knobs of the -DOICA_EXPERIMENTS build (compiled out of liboica.so); OICA_LIB selects
# another library build.  A bench line is only ever taken on the product library with none set.
EXPERIMENT_VARS = ("OICA_LIB", "OICA_TC_EPI", "OICA_TC_CL", "OICA_TC_RING", "OICA_TC_FORCE_LO", "OICA_TC_MIXED",
                   "OICA_TC_MIXED_SMS", "OICA_TC_GREEN", "OICA_GREEN_SMS", "OICA_SLOT_TARGET", "OICA_MIN_SLOTS",
                   "OICA_PROMOTE_D", "OICA_PROMOTE_RATIO", "OICA_PROMOTE_T")


def refuse_experiments():
    bad = [v for v in EXPERIMENT_VARS if os.environ.get(v) is not None]
    if bad:
        sys.stderr.write(f"bench.py: refusing to run with experiment variables set: {bad}\n")
        sys.exit(2)


def golden_path(cfg):
    """The stored oracle golden whose data seed is the config's own (tier A full L, tier B L'=256)."""
    import glob
    for p in sorted(glob.glob(os.path.join(ROOT, "tests", "golden", "oracle_*.json"))):
        try:
            with open(p) as f:
                head = json.loads(f.read())
        except Exception:
            continue
        if head.get("config") == cfg.name and head.get("data_seed") == cfg.data_seed and \
                head.get("cand_seed") == cfg.cand_seed:
            return p
    return None


def golden_match(path, W, index, alpha, n, sum_active=None, L=None):
    """Compare the all-components leg with the stored oracle results (north_star gates).  When the
    golden ran the same L (tier A), also the ratio of row-iterations (sum_t L_act) the GPU needed to
    the fp64 oracle's: the algorithmic TFLOP/s count the GPU's own iterations."""
    import numpy as np
    g = json.load(open(path))
    comps = g["components"][:n]
    same = sum(int(index[k]) == c["index"] for k, c in enumerate(comps))
    cos = [abs(float(np.dot(W[k], c["w"]))) for k, c in enumerate(comps)]
    rel = [abs((alpha[k] + 3.0) - (c["alpha"] + 3.0)) / abs(c["alpha"] + 3.0) for k, c in enumerate(comps)]
    out = {"golden": os.path.relpath(path, ROOT), "golden_L": g["L"], "components": len(comps),
           "index_match": same, "min_abs_cos": min(cos) if cos else None, "max_objective_rel_err": max(rel) if rel else None,
           "pass": bool(same == len(comps) and comps and min(cos) >= 0.9999 and max(rel) <= 1e-4)}
    if sum_active is not None and L == g["L"] and all("sum_active" in c for c in comps):
        out["row_iterations_gpu_over_oracle"] = float(sum(int(v) for v in sum_active[: len(comps)])) / \
            float(sum(c["sum_active"] for c in comps))
    return out


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


class ClockSampler:
    """SM clocks, power and clock-event (throttle) reasons sampled DURING the timed region: NVML
    every ~5 ms from a thread (plus one sample at entry and one at exit, so a region shorter than
    the period still has a record), falling back to `nvidia-smi -lms 200`."""

    def __init__(self, gpu: int):
        self.gpu, self.rows, self.proc, self.nvml, self.stop = gpu, [], None, None, None

    def _nvml_sample(self):
        m = self.nvml
        try:
            h = self.handle
            self.rows.append((float(m.nvmlDeviceGetClockInfo(h, m.NVML_CLOCK_SM)),
                              float(m.nvmlDeviceGetMaxClockInfo(h, m.NVML_CLOCK_SM)),
                              m.nvmlDeviceGetPowerUsage(h) / 1000.0,
                              int(m.nvmlDeviceGetCurrentClocksEventReasons(h))))
        except Exception:
            pass

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.handle = pynvml.nvmlDeviceGetHandleByIndex(self._physical_index())
            self.stop = threading.Event()
            self._nvml_sample()

            def loop():
                while not self.stop.wait(0.005):
                    self._nvml_sample()
            self.t = threading.Thread(target=loop, daemon=True)
            self.t.start()
            return self
        except Exception:
            self.nvml = None
        q = "clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active"
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                          "-lms", "200", "-i", str(self.gpu)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _physical_index(self):
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        if vis:
            try:
                return int(vis.split(",")[self.gpu])
            except (ValueError, IndexError):
                pass
        return self.gpu

    def _read(self):
        for line in self.proc.stdout:
            p = [s.strip() for s in line.split(",")]
            if len(p) >= 4:
                try:
                    self.rows.append((float(p[0]), float(p[1]), float(p[2]), int(p[3], 16)))
                except ValueError:
                    pass

    def __exit__(self, *a):
        if self.nvml is not None:
            self.stop.set()
            self.t.join(timeout=1)
            self._nvml_sample()
            try:
                self.nvml.nvmlShutdown()
            except Exception:
                pass
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        load = [r for r in self.rows if not (r[3] & 0x1)] or self.rows
        reasons = set()
        for r in load:
            for bit, name in REASONS.items():
                if r[3] & bit and bit != 0x1:
                    reasons.add(name)
        return {"sm_mhz": statistics.median(r[0] for r in load), "sm_max_mhz": max(r[1] for r in load),
                "power_w_max": max(r[2] for r in load), "samples": len(load), "reasons": sorted(reasons),
                "sampler": "nvml 5 ms" if self.nvml is not None else "nvidia-smi 200 ms"}


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def load_traffic(workload: str, precision: str):
    """dram bytes per launch of the step kernel from the committed ncu summary (or None)."""
    import glob
    best = None
    for p in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", "ncu_step_summary.json"))):
        try:
            d = json.load(open(p))
        except Exception:
            continue
        e = d.get(f"{workload}:{precision}")
        if e:
            best = e
    return best


def cpu_baseline(cfg, n_steps: int = 1, M_sample: int = 200_000, L_sample: int = 64):
    """Time the float64 oracle (as it stands) on a bounded sample of the workload.

    The sample's raw signals come from the seeded generator (on the GPU when present, only for
    speed); whitening and the extraction are the oracle's.  BLAS threads: every core of the
    process's affinity set (reported as `cores`)."""
    import numpy as np
    import torch
    from threadpoolctl import threadpool_info, threadpool_limits

    import datagen
    from oracle import ordering, whiten

    M_s = min(cfg.M, M_sample)
    L_s = min(cfg.L, L_sample)
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    ds = datagen.make_dataset(cfg, M=M_s, keep_sources=False, device=dev)
    Xraw = ds.X.cpu().numpy()
    threads = max(1, len(os.sched_getaffinity(0)))   # every host core the process may use
    with threadpool_limits(threads, user_api="blas"):
        Xw, _, _, _ = whiten.whiten(Xraw)
        X = Xw.astype(np.float32).astype(np.float64)
        W = np.zeros((0, cfg.N))
        flops, secs = 0.0, 0.0
        per = []
        for k in range(n_steps):
            t0 = time.perf_counter()
            Wk, res = ordering.extract(X, L_s, cfg.K, cfg.tol, k + 1, cfg.cand_seed, W_prefix=W if k else None)
            dt = time.perf_counter() - t0
            f = ordering.algorithmic_flops(res[-1:], cfg.N, M_s)
            per.append((f, dt))
            W = Wk
            flops += f
            secs += dt
        blas = [(i.get("internal_api"), i.get("num_threads")) for i in threadpool_info() if i.get("user_api") == "blas"]
    return dict(value=flops / secs / 1e12, unit="TFLOP/s", cores=threads, kind="oracle",
                sample=f"{cfg.name} N={cfg.N} with M'={M_s} samples, L'={L_s} candidates (ids 0..{L_s - 1}), "
                       f"{n_steps} component(s), float64 numpy, BLAS {blas}, host has "
                       f"{len(os.sched_getaffinity(0))} cores",
                seconds=secs, per_step=per)


def run_reference(args, cfg):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    n = args.warmup + args.steps
    cb = cpu_baseline(cfg, n_steps=n, M_sample=args.ref_M, L_sample=args.ref_L)
    per = cb.pop("per_step")
    timed = per[args.warmup:]
    f = sum(p[0] for p in timed)
    t = sum(p[1] for p in timed)
    val = f / t / 1e12
    cb["value"] = val
    out = {"impl": "reference", "metric": METRIC, "value": val, "unit": "TFLOP/s", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": cfg.name, "N": cfg.N, "M": cfg.M, "L": cfg.L, "sample_M": min(cfg.M, args.ref_M),
                      "sample_L": min(cfg.L, args.ref_L), "parallelism": "cpu oracle"},
           "cpu_baseline": cb, "e2e": {"value": val, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def fp32_peak():
    """Best measured FFMA throughput (scripts/fp32_peak.cu) with its clock, or None."""
    path = os.path.join(ROOT, "profiles", "r02", "microbench", "fp32_peak.jsonl")
    try:
        recs = [json.loads(l) for l in open(path) if l.strip()]
        recs = [r for r in recs if r.get("max_sm_mhz")]
        return max(recs, key=lambda r: r["tflops"]) if recs else None
    except (OSError, ValueError):
        return None


def run_oica(args, cfg):
    import numpy as np
    import torch
    import torch.distributed as dist

    import datagen
    from paper_2408_17118_b200 import oica

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("gloo")
    nid = None
    if world > 1:
        box = [oica.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(box, src=0)
        nid = box[0]
    stream = torch.cuda.Stream(device=dev)
    prec = {"auto": oica.PREC_AUTO, "fp32": oica.PREC_FP32, "tc": oica.PREC_TC,
            "tc_split": oica.PREC_TC_SPLIT}[args.precision]
    shard = {"l": oica.SHARD_L, "m": oica.SHARD_M, "hybrid": oica.SHARD_HYBRID}[args.shard]
    t_ctx = time.perf_counter()
    ctx = oica.Context(local, prec, rank, world, shard, stream=stream, nccl_id=nid)

    comm_init_s = time.perf_counter() - t_ctx
    # synthetic inputs of the config's recipe (not timed): rank 0 draws the raw signals (the
    # golden's host draw, or the device generator), whitens them on the device with oica_whiten
    # and distributes Xw to every rank (oica_distribute_data, C3)
    t0 = time.perf_counter()
    gpath = golden_path(cfg) if args.data == "golden" else None
    if args.data == "golden" and gpath is None:
        raise SystemExit(f"bench.py: no stored golden for {cfg.name}; use --data device")
    M_local = cfg.M
    if shard == oica.SHARD_M and world > 1:
        M_local = cfg.M * (rank + 1) // world - cfg.M * rank // world
    Xw_root = None
    if rank == 0:
        if gpath is not None:   # host draw of the golden's raw signals (fp64 generator, fp32 upload)
            ds = datagen.make_dataset(cfg, keep_sources=False)
            X = ds.X.to(torch.float32).contiguous().to(dev)
        else:
            ds = datagen.make_dataset(cfg, device=dev, dtype=torch.float32, keep_sources=False)
            X = ds.X.contiguous()
        del ds
        Xw_root = torch.empty_like(X)
        ctx.whiten(X, Xw_root)
        del X
        torch.cuda.synchronize()
    if shard == oica.SHARD_M and world > 1:
        Xw = torch.empty(cfg.N, M_local, dtype=torch.float32, device=dev)
    else:
        Xw = Xw_root if rank == 0 else torch.empty(cfg.N, cfg.M, dtype=torch.float32, device=dev)
    ctx.distribute_data(Xw_root, cfg.N, cfg.M, Xw)
    if Xw_root is not None and Xw_root.data_ptr() != Xw.data_ptr():
        del Xw_root
    ctx.set_data(Xw, M_global=cfg.M)
    ctx.init_candidates(cfg.cand_seed, cfg.L)
    setup_s = time.perf_counter() - t0

    if args.all_components:   # time the whole extraction: components 1..N_out after a warm-up pass
        args.steps = cfg.N_out
    xflags = (oica.REDUCE_X if args.reduce else 0) | (oica.EAGER if args.eager else 0)
    N_out = args.warmup + args.steps
    assert args.all_components or N_out <= cfg.N_out, "warmup + steps exceeds the config's N_out"
    Wacc = np.zeros((cfg.N_out, cfg.N))
    recs = []

    def step(k):
        if args.all_components and k >= args.warmup:
            k -= args.warmup   # timed pass restarts at component 1
        r = ctx.extract(k + 1, cfg.K, cfg.tol, flags=xflags, W_prefix=Wacc[:k] if k else None)
        Wacc[k] = r.W[k]
        recs.append(dict(i=k + 1, index=int(r.index[k]), alpha=float(r.alpha[k]), upsilon=float(r.upsilon[k]),
                         sum_active=int(r.sum_active[k]), n_iter=int(r.n_iter[k]), cluster=int(r.cluster_size[k]),
                         n_conv=int(r.n_converged[k]), n_unconv=int(r.n_unconverged[k]), near_tie=int(r.near_tie[k]),
                         dim=int(r.dim[k])))
        return r

    for k in range(args.warmup):
        step(k)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    ctx.reset_stats()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize(dev)
        e0.record(stream)
        for k in range(args.warmup, N_out):
            step(k)
        e1.record(stream)
        torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    ms_local = e0.elapsed_time(e1)
    ms = ms_local
    st = ctx.stats()
    timed = recs[args.warmup:]
    M = cfg.M
    # algorithmic work of the timed steps: the iteration of component i runs in dim_i = N (or
    # N - i + 1 with --reduce)
    flops = sum(r["sum_active"] * (4.0 * r["dim"] * M + 3.0 * M) for r in timed)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = flops / (ms / 1e3) / 1e12

    # end-to-end leg: the same components re-extracted through host buffers each step
    e2e = None
    if not args.no_e2e:
        Xh = torch.empty(Xw.shape, dtype=torch.float32, pin_memory=True)
        Xh.copy_(Xw)
        # one untimed upload: the context's upload buffer, copy stream and events are set up once
        ctx.set_data_host_ptr(Xh.data_ptr(), cfg.N, M_local, M_local, M_global=cfg.M)
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        d2h = 0
        for k in range(args.warmup, N_out):
            if args.all_components:
                k -= args.warmup
            ctx.set_data_host_ptr(Xh.data_ptr(), cfg.N, M_local, M_local, M_global=cfg.M)
            r = ctx.extract(k + 1, cfg.K, cfg.tol, flags=xflags, W_prefix=Wacc[:k] if k else None)
            d2h += 8 * cfg.N + 112 + 4 * int(r.n_iter[k])
        f1.record(stream)
        torch.cuda.synchronize(dev)
        ems = f0.elapsed_time(f1)
        if world > 1:
            t = torch.tensor([ems], dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        e2e = {"value": flops / (ems / 1e3) / 1e12, "unit": "TFLOP/s", "h2d_bytes_per_step": 4 * cfg.N * M_local,
               "d2h_bytes_per_step": d2h // max(1, args.steps), "ms_per_step": ems / args.steps}
        ctx.set_data(Xw, M_global=cfg.M)

    # all-components leg (BASELINE.json's metric also names "seconds to extract all N"): one fresh
    # extraction of components 1..N_out, device-timed (max over ranks); not part of `value`
    all_leg = None
    if not args.all_components and not args.no_all:
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        ra = ctx.extract(cfg.N_out, cfg.K, cfg.tol, flags=xflags)
        a1.record(stream)
        torch.cuda.synchronize(dev)
        ams = a0.elapsed_time(a1)
        if world > 1:
            t = torch.tensor([ams], dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ams = float(t.item())
        dims = [int(v) for v in ra.dim[: ra.n_extracted]]
        aflops = sum(int(ra.sum_active[k]) * (4.0 * dims[k] * cfg.M + 3.0 * cfg.M) for k in range(ra.n_extracted))
        all_leg = {"seconds": ams / 1e3, "components": int(ra.n_extracted), "value": aflops / (ams / 1e3) / 1e12,
                   "unit": "TFLOP/s", "indices": [int(v) for v in ra.index[: ra.n_extracted]]}
        if gpath is not None:
            all_leg["golden_match"] = golden_match(gpath, ra.W, ra.index, ra.alpha, int(ra.n_extracted), ra.sum_active,
                                                   cfg.L)

    # per-rank breakdown (multi-GPU diagnosis: step kernel / NCCL exchange / tail, communicator init)
    st_now = ctx.stats()
    mine = {"rank": rank, "comm_init_s": comm_init_s, "setup_s": setup_s, "timed_ms": ms_local,
            "step_ms": st["step_ms"], "graph_ms": st["graph_ms"], "graph_iterations": st["graph_iterations"],
            "exchange_ms": st["exchange_ms"], "exchange_calls": st["exchange_calls"],
            "iterations": st["iterations"], "tail_iterations": st["tail_iterations"],
            "kernel_launches": st["kernel_launches"], "all_leg_exchange_ms": st_now["exchange_ms"] - st["exchange_ms"]}
    per_rank = [mine]
    if world > 1:
        per_rank = [None] * world
        dist.all_gather_object(per_rank, mine)

    if rank != 0:
        ctx.close()
        if world > 1:
            dist.destroy_process_group()
        return

    peaks = measured_peaks()
    clocks = clk.summary()
    precision = {oica.PREC_TC: "tc", oica.PREC_TC_SPLIT: "tc_split"}.get(st["precision"], "fp32")
    kern_tflops = st["step_flops"] / (st["step_ms"] / 1e3) / 1e12 if st["step_ms"] > 0 else None
    issued_tflops = st["step_issued_flops"] / (st["step_ms"] / 1e3) / 1e12 if st["step_ms"] > 0 else None
    loop_only = kern_tflops is None and st["graph_ms"] > 0   # short iterations: the device-side loop
    if loop_only:
        kern_tflops = st["graph_flops"] / (st["graph_ms"] / 1e3) / 1e12
    if precision.startswith("tc"):
        peak = peaks.get("bf16_tflops_sustained") or 1404.1
        passes = 3 if precision == "tc_split" else 2
        roof = {"bound": "tensor",
                "peak_source": "MEASURED_PEAKS.json bf16_tflops_sustained (kind::f16 fp16 dense = bf16 rate); "
                               f"{passes} fp16 MMA passes per 2 algorithmic GEMMs; frac = algorithmic / peak, "
                               "issued_frac = issued (128-row tiles x padded N, all passes) / peak"}
    else:
        mhz = clocks.get("sm_mhz") or peaks.get("clocks_under_load", {}).get("sm_mhz_median", 1357.0)
        fp = fp32_peak()
        if fp:   # measured FFMA throughput (scripts/fp32_peak.cu) scaled to the sampled clock
            peak = fp["tflops"] * mhz / fp["max_sm_mhz"]
            roof = {"bound": "alu", "peak_source": f"measured FP32 FFMA peak {fp['tflops']:.1f} TFLOP/s at "
                                                   f"{fp['max_sm_mhz']:.0f} MHz (profiles/r02/microbench/fp32_peak.jsonl) "
                                                   f"scaled to {mhz:.0f} MHz (median SM clock under load)"}
        else:
            peak = 148 * 128 * 2 * mhz * 1e6 / 1e12
            roof = {"bound": "alu", "peak_source": f"148 SMs x 128 FP32 lanes x 2 flop x {mhz:.0f} MHz (median SM clock under load)"}
    tr = load_traffic(cfg.name, precision)
    roof.update({"achieved": kern_tflops, "peak": peak, "unit": "TFLOP/s",
                 "frac": (kern_tflops / peak) if kern_tflops else None,
                 "issued": issued_tflops, "issued_frac": (issued_tflops / peak) if issued_tflops else None,
                 "fine_row_frac": st["fine_rows"] / st["sum_active"] if st["sum_active"] else None,
                 "traffic": tr.get("dram_bytes_per_launch") if tr else None,
                 "traffic_launch": tr if tr else None,
                 "kernel": "fused fixed-point step (GEMM-cube-GEMM)", "launches": st["step_launches"],
                 "kernel_ms": st["step_ms"], "share_of_step": st["step_ms"] / ms if ms else None})
    if loop_only:
        roof.update({"kernel": "device-side iteration loop (CUDA-graph WHILE node: fused step + fused update per "
                               "iteration; steps not timed one by one -- run with --eager for the step alone)",
                     "launches": 2 * st["graph_iterations"], "kernel_ms": st["graph_ms"],
                     "share_of_step": st["graph_ms"] / ms if ms else None})
    if precision.startswith("tc") and kern_tflops:
        # transparency: the sustained figure is cuBLAS bf16 under the power cap (at its own, lower
        # clock); also the burst figure and the dense peak at the clock sampled in this run
        burst = peaks.get("bf16_tflops") or 1635.4
        mhz = clocks.get("sm_mhz") or 0
        per_clock = 148 * 8192 * mhz * 1e6 / 1e12 if mhz else None   # fp16 dense: 8192 flop/clk/SM
        roof.update({"peak_burst": burst, "frac_burst": kern_tflops / burst,
                     "peak_at_sampled_clock": per_clock,
                     "frac_at_sampled_clock": (kern_tflops / per_clock) if per_clock else None})
    cb = None
    if not args.no_cpu_baseline and world == 1:
        cb = cpu_baseline(cfg, 1, args.ref_M, args.ref_L)
        cb.pop("per_step", None)
    sec_per_comp = ms / 1e3 / args.steps
    sec_all = ms / 1e3 if args.all_components else (all_leg["seconds"] if all_leg else None)
    out = {"metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong",
           "vs_baseline": None, "dtype": "f16" if precision.startswith("tc") else "f32", "data": "synthetic",
           "config": {"workload": cfg.name, "N": cfg.N, "M": cfg.M, "L": cfg.L, "K": cfg.K, "tol": cfg.tol,
                      "N_out": cfg.N_out, "components_timed": [r["i"] for r in timed],
                      "parallelism": f"{args.shard}shard{world}",
                      "l2": f"inputs larger than L2 (X = {4 * cfg.N * cfg.M / 1e9:.2f} GB fp32), no flush",
                      "precision": precision, "slots": st["slots"],
                      "reduced_x": bool(args.reduce), "data_draw": args.data, "eager": bool(args.eager),
                      "library": "liboica.so (release build: no experiment modes)",
                      "seconds_all_components": sec_all,
                      "golden_match": (all_leg or {}).get("golden_match")},
           "seconds_per_component": sec_per_comp, "seconds_all_components": sec_all, "all_components": all_leg,
           "gpu_launches": st["kernel_launches"], "roofline": roof, "e2e": e2e, "cpu_baseline": cb,
           "clocks": clocks, "components": timed, "setup_s": setup_s, "per_rank": per_rank}
    print(json.dumps(out), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="oica", choices=["oica", "reference"])
    ap.add_argument("--config", default=DEFAULT_CONFIG)
    ap.add_argument("--precision", default="auto", choices=["auto", "fp32", "tc", "tc_split"])
    ap.add_argument("--shard", default="l", choices=["l", "m", "hybrid"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--reduce", action="store_true",
                    help="iterate on the reduced data X~ = G X (PAPER.md §3.3, OICA_REDUCE_X)")
    ap.add_argument("--all-components", action="store_true",
                    help="time all N_out components (seconds to extract all N); --steps is ignored")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--eager", action="store_true",
                    help="host-launched iterations (times every step launch; default: device-side loop where short)")
    ap.add_argument("--no-all", action="store_true", help="skip the all-components leg")
    ap.add_argument("--data", default="golden", choices=["golden", "device"],
                    help="golden: the stored oracle golden's host draw (checked against it); device: device draw")
    ap.add_argument("--ref-M", type=int, default=1_000_000)
    ap.add_argument("--ref-L", type=int, default=256)
    args = ap.parse_args()
    refuse_experiments()
    import datagen
    cfg = datagen.get(args.config)
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_oica(args, cfg)


if __name__ == "__main__":
    main()
