#!/usr/bin/env python
"""One-line summary of bench.py JSON output files: python scripts/show_line.py file.json [...]"""
import json
import os
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().splitlines()[-1])
    except Exception as e:
        print(os.path.basename(f), "unreadable:", e)
        continue
    r = d.get("roofline") or {}
    g = (d.get("config") or {}).get("golden_match") or {}
    rnd = lambda v, n=3: round(v, n) if isinstance(v, (int, float)) else v
    print(os.path.basename(f), "value", rnd(d.get("value"), 1), "ms/step", rnd(d.get("ms_per_step")),
          "all_s", rnd(d.get("seconds_all_components"), 4), "kern", rnd(r.get("achieved"), 1), "frac", rnd(r.get("frac")),
          "share", rnd(r.get("share_of_step")), "clk", (d.get("clocks") or {}).get("sm_mhz"),
          (d.get("clocks") or {}).get("reasons"), "golden", g.get("pass"))
