#!/bin/bash
# Full GPU suite + smoke + ncu evidence for the step kernel (cfg4).
python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
timeout 900 python -m pytest tests -q -m gpu -s > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$?
grep -E "passed|failed" gpurun_out/gpu_tests.log | tail -2
CMD="python bench.py --config cfg4_scaling --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_cfg4.json 2> gpurun_out/plain_cfg4.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:oica:: -c 800 \
    --csv --log-file gpurun_out/launches_cfg4_tc.csv $CMD > gpurun_out/ncu_list_cfg4.log 2>&1; echo list=$?
$CMD > gpurun_out/plain2_cfg4.json 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:k_step_tc -s 2 -c 1 \
    -o gpurun_out/prof_tc_cfg4 $CMD > gpurun_out/ncu_full_cfg4.log 2>&1; echo full=$?
