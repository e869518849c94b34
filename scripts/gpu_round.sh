#!/bin/bash
# GPU tests + TC bench lines (cfg4 default in both TC modes, cfg3), used during development.
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu -s > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$?
grep -E "passed|failed|Error" gpurun_out/gpu_tests.log | tail -5
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; echo bench4_rc=$?
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --precision tc_split > gpurun_out/bench_cfg4_split.json 2> gpurun_out/bench_cfg4_split.err; echo bench4s_rc=$?
timeout 600 python bench.py --config cfg3_large --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err; echo bench3_rc=$?
tail -3 gpurun_out/bench_cfg4.err
