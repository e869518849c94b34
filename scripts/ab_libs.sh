#!/bin/bash
# A/B timing of two liboica builds (dev experiment), alternated twice on one box:
#   base = ab_libs/base_pkg (a complete older package: binding + library), new = the working tree
set -u
mkdir -p gpurun_out
for r in 1 2; do
  echo "== base run $r"; OICA_PKG_ROOT=$PWD/ab_libs/base_pkg timeout 600 python scripts/tc_variants.py 0 ${AB_SHAPES:-256 128 64} 2>&1 | grep '^{'
  echo "== new run $r"; timeout 600 python scripts/tc_variants.py 0 ${AB_SHAPES:-256 128 64} 2>&1 | grep '^{'
done
