#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/parity_persist.log 2>&1; echo parity=$?; tail -3 gpurun_out/parity_persist.log
rm -f gpurun_out/persist.log
for rg in 1 0; do OICA_TC_RING=$rg timeout 300 python scripts/tc_variants.py 0 128 | sed "s/{/{\"ring\": $rg, /" >> gpurun_out/persist.log 2>&1; done
OICA_TC_RING=1 OICA_TC_EPI=3 timeout 300 python scripts/tc_variants.py 3 128 | sed "s/{/{\"ring\": 1, /" >> gpurun_out/persist.log 2>&1
timeout 300 python scripts/tc_variants.py 0 256 | sed "s/{/{\"ring\": 0, /" >> gpurun_out/persist.log 2>&1
cat gpurun_out/persist.log | cut -c1-200
