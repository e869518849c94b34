#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -x -m gpu > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/gpu_tests.log
OICA_TC_RING=1 timeout 300 python scripts/tc_variants.py 0 128 > gpurun_out/slots2.log 2>&1
timeout 300 python scripts/tc_variants.py 0 128 >> gpurun_out/slots2.log 2>&1
cat gpurun_out/slots2.log | cut -c1-200
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; echo b4=$?
timeout 900 python bench.py --config cfg3_large --all-components --no-e2e --no-cpu-baseline > gpurun_out/bench_cfg3_all.json 2> gpurun_out/bench_cfg3_all.err; echo b3=$?
timeout 900 python bench.py --config cfg3_large --all-components --no-e2e --no-cpu-baseline --reduce > gpurun_out/bench_cfg3_all_red.json 2> gpurun_out/bench_cfg3_all_red.err; echo b3r=$?
timeout 900 python bench.py --config cfg2_eeg_shaped --all-components --no-e2e --no-cpu-baseline --reduce > gpurun_out/bench_cfg2_all_red.json 2> gpurun_out/bench_cfg2_all_red.err; echo b2r=$?
