#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/spin.log
for N in 64 128 256; do for v in 0 8 6 14; do
  OICA_TC_EPI=$v timeout 300 python scripts/tc_variants.py $v $N >> gpurun_out/spin.log 2>&1
done; done
