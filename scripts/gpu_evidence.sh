#!/bin/bash
# Round evidence: all-components timings, ncu launch list + full capture at cfg4 and cfg3.
mkdir -p gpurun_out
timeout 1200 python bench.py --all-components --no-e2e --no-cpu-baseline > gpurun_out/bench_cfg4_all.json 2> gpurun_out/bench_cfg4_all.err; echo b4all=$?
timeout 1200 python bench.py --all-components --no-e2e --no-cpu-baseline --reduce > gpurun_out/bench_cfg4_all_red.json 2> gpurun_out/bench_cfg4_all_red.err; echo b4allr=$?
timeout 600 python bench.py --config cfg1_artificial --all-components --no-e2e --no-cpu-baseline > gpurun_out/bench_cfg1_all.json 2> gpurun_out/bench_cfg1_all.err; echo b1all=$?
timeout 600 python bench.py --config cfg0_tiny --all-components --no-e2e --no-cpu-baseline > gpurun_out/bench_cfg0_all.json 2> gpurun_out/bench_cfg0_all.err; echo b0all=$?
for CFG in cfg4_scaling cfg3_large; do
  CMD="python bench.py --config $CFG --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
  $CMD > gpurun_out/plain_$CFG.json 2> gpurun_out/plain_$CFG.err && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:oica -c 4000 \
      --csv --log-file gpurun_out/launches_$CFG.csv $CMD > gpurun_out/ncu_list_$CFG.log 2>&1; echo list_$CFG=$?
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step_tc -s 2 -c 1 \
      -o gpurun_out/prof_tc_${CFG}_v7 $CMD > gpurun_out/ncu_full_$CFG.log 2>&1; echo full_$CFG=$?
done
