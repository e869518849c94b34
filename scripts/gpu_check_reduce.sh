#!/bin/bash
# Reduced-X (§3.3) parity + timing.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -s -k "reduced or wide" > gpurun_out/parity_reduced.log 2>&1; echo parity_red=$?
tail -3 gpurun_out/parity_reduced.log
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/parity_all.log 2>&1; echo parity_all=$?
tail -2 gpurun_out/parity_all.log
timeout 900 python bench.py --config cfg3_large --all-components --no-e2e --no-cpu-baseline --reduce > gpurun_out/bench_cfg3_all_red.json 2> gpurun_out/bench_cfg3_all_red.err; echo b3r=$?
timeout 900 python bench.py --config cfg2_eeg_shaped --all-components --no-e2e --no-cpu-baseline > gpurun_out/bench_cfg2_all.json 2> gpurun_out/bench_cfg2_all.err; echo b2=$?
timeout 900 python bench.py --config cfg2_eeg_shaped --all-components --no-e2e --no-cpu-baseline --reduce > gpurun_out/bench_cfg2_all_red.json 2> gpurun_out/bench_cfg2_all_red.err; echo b2r=$?
timeout 900 python bench.py --no-e2e --no-cpu-baseline --reduce --warmup 20 --steps 3 > gpurun_out/bench_cfg4_red.json 2> gpurun_out/bench_cfg4_red.err; echo b4r=$?
