#!/usr/bin/env python
"""Refresh profiles/<round>/ncu_step_summary.json (the roofline `traffic` bench.py reports) from the
`ncu --set full` summaries `scripts/gpu_jobs.sh ncu-step` writes (ncu_full_<cfg>.json; round 1:
ncu_full_<cfg>_final.json).

    python scripts/update_step_summary.py profiles/r02/ncu profiles/r02/ncu_step_summary.json
"""
import json
import os
import sys

UNITS = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def value(s, unit_scale=None):
    v, u = s.split()[0], s.split()[1] if len(s.split()) > 1 else ""
    x = float(v.replace(",", ""))
    if u in UNITS:
        return x * UNITS[u]
    if u == "ms":
        return x
    if u == "us":
        return x / 1e3
    return x


def main():
    import datagen
    src, dst = sys.argv[1], sys.argv[2]
    out = json.load(open(dst)) if os.path.exists(dst) else {}
    for cfg_name in ("cfg4_scaling", "cfg3_large", "cfg2_eeg_shaped"):
        p = os.path.join(src, f"ncu_full_{cfg_name}.json")
        if not os.path.exists(p):
            p = os.path.join(src, f"ncu_full_{cfg_name}_final.json")
        if not os.path.exists(p):
            continue
        d = json.load(open(p))[0]
        cfg = datagen.get(cfg_name)
        rd = value(d["dram__bytes_read.sum"])
        wr = value(d["dram__bytes_write.sum"])
        grid = int(d["launch__grid_size"])
        NP = ((cfg.N + 15) // 16) * 16
        S = max(1, min(128, max(min(30, cfg.M // 128), cfg.M // 65536)))
        out[f"{cfg_name}:tc"] = {
            "kernel": d["kernel"].replace("unnamed>::", ""),
            "dram_bytes_per_launch": rd + wr,
            "dram_read": rd,
            "dram_write": wr,
            "launch": f"third step launch of bench.py --steps 1 --warmup 3 --eager (component 1, full L), grid {grid} CTAs",
            "duration_ms_under_ncu": value(d["gpu__time_duration.sum"]),
            "algorithmic_bytes_per_launch": 2 * cfg.N * cfg.M + 2 * cfg.L * NP + 4 * S * cfg.L * NP,
            "algorithmic_bytes_note": f"X fp16 once (2 N M) + fp16 operand rows in (2 L NP) + fp32 slot partials out "
                                      f"(4 S L NP, S={S})",
            "source": p,
            # the SM-clock counter (the "realtime" triage counter reads low for short launches:
            # cfg 2 17% against 60% on the SM clock)
            "tensor_pipe_active_pct": value(d["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"]
                                            if "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed" in d
                                            else d["TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime"
                                                   ".avg.pct_of_peak_sustained_elapsed"]),
            "tensor_memory_active_pct": value(d["sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"])
            if "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed" in d else None,
        }
    json.dump(out, open(dst, "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    main()
