#!/bin/bash
# Round evidence after a kernel change: smoke, GPU suite, bench lines (cfg4 default, cfg3, cfg2),
# all-components timing at cfg3, ncu launch list and one --set full capture of the step kernel.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build_rc=$?
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
timeout 1800 python -m pytest tests -q -m gpu -s > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$?
grep -E "passed|failed" gpurun_out/gpu_tests.log | tail -2
timeout 900 python bench.py > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; echo bench4_rc=$?
timeout 600 python bench.py --config cfg3_large --no-cpu-baseline > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err; echo bench3_rc=$?
timeout 600 python bench.py --config cfg2_eeg_shaped --no-cpu-baseline > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; echo bench2_rc=$?
timeout 900 python bench.py --config cfg3_large --all-components --no-e2e --no-cpu-baseline > gpurun_out/bench_cfg3_all.json 2> gpurun_out/bench_cfg3_all.err; echo bench3all_rc=$?
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_cfg4.json 2> gpurun_out/plain_cfg4.err && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:oica -c 4000 \
    --csv --log-file gpurun_out/launches_cfg4.csv $CMD > gpurun_out/ncu_list_cfg4.log 2>&1; echo list=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step_tc -s 2 -c 1 \
    -o gpurun_out/prof_tc_cfg4_v4 $CMD > gpurun_out/ncu_full_cfg4.log 2>&1; echo full=$?
