#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/parity.log 2>&1; echo parity=$?; tail -3 gpurun_out/parity.log
timeout 600 python bench.py --config cfg1_artificial --all-components --no-e2e --no-cpu-baseline > gpurun_out/bench_cfg1_all.json 2> gpurun_out/bench_cfg1_all.err; echo b1all=$?
timeout 600 python bench.py --config cfg0_tiny --all-components --no-e2e --no-cpu-baseline > gpurun_out/bench_cfg0_all.json 2> gpurun_out/bench_cfg0_all.err; echo b0all=$?
timeout 600 python bench.py --config cfg2_eeg_shaped --all-components --no-e2e --no-cpu-baseline > gpurun_out/bench_cfg2_all.json 2> gpurun_out/bench_cfg2_all.err; echo b2all=$?
