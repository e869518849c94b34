#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/promote_*.json
for cfgv in "1e-6 1e-3 40" "1e-6 0.3 40" "1e-8 0.3 40" "1e-7 0.1 40" "1e-8 0.5 60"; do
  set -- $cfgv
  OICA_PROMOTE_D=$1 OICA_PROMOTE_RATIO=$2 OICA_PROMOTE_T=$3 timeout 900 python bench.py --config cfg3_large --all-components --no-e2e --no-cpu-baseline > gpurun_out/promote_$1_$2_$3.json 2>/dev/null
done
