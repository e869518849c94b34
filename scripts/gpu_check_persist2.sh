#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/persist2.log
for N in 256 128; do
for k in 0 1 4; do for m in 6 3 0; do
  OICA_TC_VERBOSE=1 OICA_TC_RING=1 OICA_TC_K=$k OICA_TC_EPI=$m timeout 300 python scripts/tc_variants.py $m $N 2>&1 | grep -v "^k_step" | sed "s/{/{\"K\": $k, /" >> gpurun_out/persist2.log
done; done; done
OICA_TC_VERBOSE=1 OICA_TC_RING=1 timeout 300 python scripts/tc_variants.py 0 128 2>&1 | grep "^k_step" | head -2 >> gpurun_out/persist2.log
OICA_TC_VERBOSE=1 timeout 300 python scripts/tc_variants.py 0 256 2>&1 | grep "^k_step" | head -2 >> gpurun_out/persist2.log
