#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/ring.log
for rep in 1 2; do for cl in 1 2; do for rg in 1 0; do
  OICA_TC_CL=$cl OICA_TC_RING=$rg timeout 300 python scripts/tc_variants.py 0 128 | sed "s/{/{\"cl\": $cl, \"ring\": $rg, /" >> gpurun_out/ring.log 2>&1
done; done; done
for m in 3 6; do for cl in 1 2; do
  OICA_TC_EPI=$m OICA_TC_CL=$cl OICA_TC_RING=1 timeout 300 python scripts/tc_variants.py $m 128 | sed "s/{/{\"cl\": $cl, \"ring\": 1, /" >> gpurun_out/ring.log 2>&1
done; done
