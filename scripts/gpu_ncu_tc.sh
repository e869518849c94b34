#!/bin/bash
# ncu evidence for the tensor-core step kernel (run each command plain first, then under ncu).
for CFG in cfg4_scaling cfg3_large; do
  CMD="python bench.py --config $CFG --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
  $CMD > gpurun_out/plain_$CFG.json 2> gpurun_out/plain_$CFG.err && \
  ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:oica:: -c 800 \
      --csv --log-file gpurun_out/launches_${CFG}_tc.csv $CMD > gpurun_out/ncu_list_$CFG.log 2>&1; echo list_$CFG=$?
  $CMD > gpurun_out/plain2_$CFG.json 2>&1 && \
  ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:k_step_tc -s 2 -c 1 \
      -o gpurun_out/prof_tc_$CFG $CMD > gpurun_out/ncu_full_$CFG.log 2>&1; echo full_$CFG=$?
done
