"""Build liboica.so in-tree with nvcc for sm_100a (B200).

    python -m paper_2408_17118_b200.build [--force] [-j N] [--experiments]

Every .cu under csrc/ is compiled with -gencode arch=compute_100a,code=sm_100a (the 'a'
target is required for tcgen05) and linked into paper_2408_17118_b200/liboica.so.
`--experiments` builds a separate liboica_exp.so with -DOICA_EXPERIMENTS: the timing variants
of DESIGN.md §7 (modes that skip work, cluster / ring / slot / promotion overrides read from
OICA_* environment variables).  The product library never contains them; the experiment
library is loaded only when OICA_LIB points at it (scripts/tc_variants.py), and bench.py
refuses to run with OICA_LIB set.  `--debug-checks` builds liboica_dbg.so with -DOICA_DEBUG_CHECKS:
device-side bounds checks of the active lists / compaction counts and bounded mbarrier waits in
the tensor-core step (a lost arrival traps instead of hanging the GPU) -- run the GPU tests
against it with OICA_LIB (scripts/gpu_jobs.sh debug-checks; compute-sanitizer is closed on the pool).
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(ROOT, "build", "oica")
LIB = os.path.join(HERE, "liboica.so")
LIB_EXP = os.path.join(HERE, "liboica_exp.so")
LIB_DBG = os.path.join(HERE, "liboica_dbg.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-Xptxas", "-warn-spills", "-I" + os.path.join(ROOT, "include"), "-I" + CSRC]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def _deps(src):
    hdrs = glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.hpp")) + [os.path.join(ROOT, "include", "oica.h")]
    return [src] + hdrs


def _stale(obj, deps):
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, jobs: int = 8, verbose: bool = False, experiments: bool = False,
          debug_checks: bool = False) -> str:
    bdir = BUILD + ("_exp" if experiments else "") + ("_dbg" if debug_checks else "")
    out = LIB_EXP if experiments else LIB_DBG if debug_checks else LIB
    extra = (["-DOICA_EXPERIMENTS"] if experiments else []) + (["-DOICA_DEBUG_CHECKS"] if debug_checks else [])
    os.makedirs(bdir, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    cc = nvcc()
    objs = []
    todo = []
    for s in srcs:
        o = os.path.join(bdir, os.path.basename(s) + ".o")
        objs.append(o)
        if force or _stale(o, _deps(s)):
            todo.append((s, o))

    def comp(so):
        s, o = so
        cmd = [cc, *ARCH, *FLAGS, *extra, "-c", s, "-o", o]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {os.path.basename(s)}:\n{r.stderr}")
        return s, r.stderr

    with cf.ThreadPoolExecutor(max_workers=max(1, jobs)) as ex:
        for s, err in ex.map(comp, todo):
            if verbose and err.strip():
                print(f"[{os.path.basename(s)}]\n{err}", file=sys.stderr)
    if todo or not os.path.exists(out) or any(os.path.getmtime(o) > os.path.getmtime(out) for o in objs):
        cmd = [cc, *ARCH, "-shared", "-o", out, *objs, "-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-j", type=int, default=8)
    ap.add_argument("-v", action="store_true")
    ap.add_argument("--experiments", action="store_true", help="build liboica_exp.so with -DOICA_EXPERIMENTS")
    ap.add_argument("--debug-checks", action="store_true",
                    help="build liboica_dbg.so with -DOICA_DEBUG_CHECKS (device bounds checks, bounded mbarrier waits)")
    a = ap.parse_args()
    print(build(a.force, a.j, a.v, a.experiments, a.debug_checks))
