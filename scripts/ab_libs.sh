#!/bin/bash
# A/B timing of two liboica builds (dev experiment): ab_libs/liboica_{base,new}.so, alternated twice
set -u
mkdir -p gpurun_out
for r in 1 2; do
  for v in base new; do
    cp ab_libs/liboica_$v.so paper_2408_17118_b200/liboica.so
    echo "== $v run $r"
    timeout 600 python scripts/tc_variants.py 0 ${AB_SHAPES:-256 128 64} 2>&1 | grep '^{'
  done
done
cp ab_libs/liboica_new.so paper_2408_17118_b200/liboica.so
