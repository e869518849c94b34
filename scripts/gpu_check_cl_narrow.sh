#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/cl_narrow.log
for N in 64 128; do for cl in 1 2; do for m in 0 3 6; do
  OICA_TC_CL=$cl OICA_TC_EPI=$m timeout 300 python scripts/tc_variants.py $m $N | sed "s/{/{\"cl\": $cl, /" >> gpurun_out/cl_narrow.log 2>&1
done; done; done
