#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/parity.log 2>&1; echo parity=$?; tail -1 gpurun_out/parity.log
timeout 900 python bench.py --config cfg3_large --no-cpu-baseline > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err; echo b3=$?
timeout 900 python bench.py --config cfg3_large --all-components --no-e2e --no-cpu-baseline > gpurun_out/bench_cfg3_all.json 2> gpurun_out/bench_cfg3_all.err; echo b3a=$?
timeout 900 python bench.py --config cfg3_large --all-components --no-e2e --no-cpu-baseline --reduce > gpurun_out/bench_cfg3_all_red.json 2> gpurun_out/bench_cfg3_all_red.err; echo b3ar=$?
