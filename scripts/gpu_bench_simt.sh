#!/bin/bash
# First measurement: SIMT step kernel on cfg3 (bench line, ncu launch list, ncu full capture).
set -x
CMD="python bench.py --config cfg3_large --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
python bench.py --config cfg3_large --steps 3 --warmup 3 > gpurun_out/bench_cfg3_simt.json 2> gpurun_out/bench_cfg3_simt.err; echo bench_rc=$?
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_cfg3_simt.csv $CMD > gpurun_out/ncu_list.log 2>&1; echo list_rc=$?
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_step_simt -s 6 -c 1 -o gpurun_out/prof_simt_cfg3 $CMD > gpurun_out/ncu_full.log 2>&1; echo full_rc=$?
tail -c 3000 gpurun_out/bench_cfg3_simt.json
