#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/n64.log
for v in 0 3 4 5 6; do OICA_TC_EPI=$v timeout 300 python scripts/tc_variants.py $v 64 >> gpurun_out/n64.log 2>&1; done
for v in 0 3; do OICA_TC_CL=2 OICA_TC_EPI=$v timeout 300 python scripts/tc_variants.py $v 64 | sed 's/{/{"cl": 2, /' >> gpurun_out/n64.log 2>&1; done
