"""bench.py keeps the driver's JSON contract (one line; keys and types), both arms.

Runs the benchmark on the small cfg 0 (and the reference arm on a tiny sample) as subprocesses.
"""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args, env=None):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=900, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_bench_line_contract():
    d = _run("--config", "cfg0_tiny", "--steps", "2", "--warmup", "3", "--ref-M", "2000", "--ref-L", "16")
    for k, t in [("metric", str), ("value", float), ("unit", str), ("n_gpus", int), ("steps", int), ("warmup", int),
                 ("ms_per_step", float), ("higher_is_better", bool), ("scaling", str), ("dtype", str), ("data", str),
                 ("config", dict), ("roofline", dict), ("e2e", dict), ("cpu_baseline", dict), ("gpu_launches", int),
                 ("clocks", dict)]:
        assert isinstance(d[k], t), (k, d.get(k))
    assert d["steps"] == 2 and d["warmup"] == 3 and d["n_gpus"] == 1 and d["value"] > 0
    assert "vs_baseline" in d and d["config"]["workload"] == "cfg0_tiny"
    r = d["roofline"]
    assert r["bound"] in ("tensor", "alu", "hbm") and r["unit"] == "TFLOP/s" and r["achieved"] > 0 and r["peak"] > 0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9 and "traffic" in r
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == 4 * 8 * 2000 and e["d2h_bytes_per_step"] > 0
    c = d["cpu_baseline"]
    assert c["kind"] == "oracle" and c["value"] > 0 and c["cores"] >= 1 and c["sample"]
    assert d["gpu_launches"] > 0
    a = d["all_components"]   # BASELINE metric's "seconds to extract all N"
    assert d["seconds_all_components"] == a["seconds"] > 0 and a["components"] == 8 and a["value"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    assert d["config"]["seconds_all_components"] == a["seconds"] and d["config"]["data_draw"] == "golden"
    g = a["golden_match"]   # the stored tier-A oracle golden of cfg 0 (same data seed, full L)
    assert g["pass"] and g["index_match"] == 8 == g["components"], g
    assert d["config"]["golden_match"] == g and len(d["per_rank"]) == 1
    pr = d["per_rank"][0]   # cfg 0: short iterations run in the device-side loop (graph_ms), not timed per step
    assert pr["step_ms"] + pr["graph_ms"] > 0 and pr["graph_iterations"] > 0


def test_reference_arm_contract():
    d = _run("--impl", "reference", "--config", "cfg0_tiny", "--steps", "1", "--warmup", "1", "--ref-M", "2000",
             "--ref-L", "16")
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "TFLOP/s"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["e2e"]["value"] == d["value"]
