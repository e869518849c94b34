#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_fullsize.py -q -x > gpurun_out/parity.log 2>&1; echo parity=$?; tail -1 gpurun_out/parity.log
timeout 900 python bench.py --config cfg2_eeg_shaped --all-components --no-e2e --no-cpu-baseline > gpurun_out/bench_cfg2_all.json 2>/dev/null; echo b2=$?
timeout 900 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/bench_cfg4.json 2>/dev/null; echo b4=$?
timeout 900 python bench.py --config cfg3_large --all-components --no-e2e --no-cpu-baseline --reduce > gpurun_out/bench_cfg3_all_red.json 2>/dev/null; echo b3r=$?
