#!/usr/bin/env python
"""Aggregate an ncu --csv launch list (gpu__time_duration.sum) per kernel name; cases split at the
first launch of a marker kernel.  python scripts/ncu_agg.py file.csv [marker=k_step_simt]"""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
marker = sys.argv[2] if len(sys.argv) > 2 else "k_step_simt"
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, vi, mi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
agg = collections.OrderedDict()
cur = "case0"
for r in rows[hi + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    m = re.search(r"(k_\w+)", r[ki])
    n = m.group(1) if m else r[ki][:30]
    if n == marker and cur == "case0":
        cur = "case1"
    a = agg.setdefault(cur, collections.OrderedDict()).setdefault(n, [0, 0.0])
    a[0] += 1
    a[1] += float(r[vi].replace(",", ""))
for c, d in agg.items():
    print(c, "total kernel ms", round(sum(v[1] for v in d.values()) / 1e6, 3))
    for k, v in sorted(d.items(), key=lambda x: -x[1][1])[:10]:
        print(f"   {k:28s} {v[0]:6d} {v[1] / 1e6:8.3f} ms  avg {v[1] / v[0] / 1e3:7.2f} us")
