#!/bin/bash
# HEAD check focused on the headline config: GPU suite, default bench line, cfg4 all components,
# ncu launch list + one --set full capture (summaries only; gpurun_out is capped at 64 MiB).
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$?; tail -1 gpurun_out/gpu_tests.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
timeout 900 python bench.py > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; echo bench4_rc=$?
timeout 1200 python bench.py --all-components --no-e2e --no-cpu-baseline > gpurun_out/bench_cfg4_scaling_all.json 2>/dev/null; echo all_cfg4=$?
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_cfg4.json 2>/dev/null && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:oica -c 4000 \
    --csv --log-file gpurun_out/launches_cfg4_scaling.csv $CMD > /dev/null 2>&1; echo list=$?
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:k_step_tc -s 2 -c 1 \
    -o /tmp/prof_tc_cfg4_final $CMD > gpurun_out/ncu_full_cfg4.log 2>&1; echo full=$?
python scripts/ncu_summary.py full /tmp/prof_tc_cfg4_final.ncu-rep > gpurun_out/ncu_full_cfg4_scaling_final.json 2>&1
