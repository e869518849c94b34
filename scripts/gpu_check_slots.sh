#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/slots.log
for t in 8192 32768 8192 32768; do for m in 0 3; do
  OICA_SLOT_TARGET=$t OICA_TC_EPI=$m OICA_TC_RING=1 timeout 300 python scripts/tc_variants.py $m 128 | sed "s/{/{\"slot_target\": $t, /" >> gpurun_out/slots.log 2>&1
done; done
for m in 3 0; do OICA_TC_EPI=$m OICA_TC_RING=0 timeout 300 python scripts/tc_variants.py $m 128 | sed "s/{/{\"slot_target\": 8192, \"ring\": 0, /" >> gpurun_out/slots.log 2>&1; done
