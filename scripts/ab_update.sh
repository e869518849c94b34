#!/bin/bash
# A/B of liboica builds on the small problems (cfg 1, cfg 2 all components, Exp. 1), alternated:
#   variants = ab_libs/liboica_<name>.so for each name in $VARIANTS, "tree" = the working tree's build
set -u
mkdir -p gpurun_out/ab
for r in 1 2; do
  for v in ${VARIANTS:-base tree}; do
    lib=""; [ "$v" != tree ] && lib=$PWD/ab_libs/liboica_$v.so
    OICA_LIB=$lib python scripts/small_profile.py --reps ${REPS:-7} --cases ${CASES:-cfg1,cfg2,exp1_L20} \
      > gpurun_out/ab/${v}_r$r.json 2> gpurun_out/ab/${v}_r$r.err
    echo "== $v run $r"; cut -c1-60 gpurun_out/ab/${v}_r$r.json | head -0
    python - gpurun_out/ab/${v}_r$r.json <<'PY'
import json, sys
for l in open(sys.argv[1]):
    if l.startswith("{"):
        d = json.loads(l); print(f"  {d['case']:10s} {d['device_ms_median']:9.3f} ms  sha {d['result_sha']}")
PY
  done
done
