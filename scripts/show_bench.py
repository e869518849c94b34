#!/usr/bin/env python
"""One-line summaries of bench JSON files (development helper)."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(f, "unreadable", e)
        continue
    r = d.get("roofline") or {}
    comps = [(c["index"], c["n_iter"], c["sum_active"], c["cluster"]) for c in d.get("components", [])]
    e2e = (d.get("e2e") or {}).get("value")
    print(f"{f}: value={d['value']:.1f} kern={r.get('achieved') or 0:.1f} issued={r.get('issued') or 0:.1f} "
          f"frac={r.get('frac') or 0:.3f} fine={r.get('fine_row_frac')} s/comp={d.get('seconds_per_component', 0):.4f} "
          f"clk={d['clocks'].get('sm_mhz')} {d['clocks'].get('reasons')} e2e={e2e} comps={comps}")
