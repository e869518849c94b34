#!/usr/bin/env python
"""Summaries of ncu outputs for profiles/.

  ncu_summary.py launches <launches.csv> [--only-oica]   per-kernel launch count, time, share
  ncu_summary.py full <report.ncu-rep>                    key counters of each profiled kernel
"""
import csv
import io
import json
import re
import subprocess
import sys
from collections import defaultdict

UNIT = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}


def short(name):
    name = re.sub(r"\(anonymous namespace\)::|<unnamed>::|void ", "", name)
    base = name.split("(")[0]
    return base[:90]


def launches(path, only_oica=False):
    text = open(path).read()
    lines = [l for l in text.splitlines() if l.startswith('"')]
    rows = list(csv.reader(io.StringIO("\n".join(lines))))
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        name = r[ki]
        if only_oica and "oica::" not in name and not re.search(r"\bk_\w+", name):
            continue
        us = float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1e-3)
        a = agg[short(name)]
        a[0] += 1
        a[1] += us
    tot = sum(a[1] for a in agg.values()) or 1.0
    out = [f"{'kernel':90s} {'launches':>8s} {'total_us':>14s} {'share':>7s}"]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"{k:90s} {n:8d} {t:14.1f} {t / tot:7.4f}")
    return "\n".join(out)


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_sleeping_per_issue_active.ratio"]


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    lines = [l for l in raw.splitlines() if l.startswith('"')]
    rows = list(csv.reader(io.StringIO("\n".join(lines))))
    h, u = rows[0], rows[1]
    res = []
    for v in rows[2:]:
        d = {"kernel": short(v[h.index("Kernel Name")])}
        for k in h:
            if any(k.startswith(w) for w in KEYS) or "tensor" in k and "pct" in k:
                i = h.index(k)
                d[k] = f"{v[i]} {u[i]}".strip()
        res.append(d)
    return json.dumps(res, indent=1)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        print(launches(sys.argv[2], "--only-oica" in sys.argv))
    else:
        print(full(sys.argv[2]))
