#!/bin/bash
# Parity suite + cfg3 all-components timing (iteration batching / fine-row precision changes).
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x > gpurun_out/parity_iter.log 2>&1; echo parity=$?
tail -3 gpurun_out/parity_iter.log
timeout 900 python bench.py --config cfg3_large --all-components --no-e2e --no-cpu-baseline > gpurun_out/bench_cfg3_all.json 2> gpurun_out/bench_cfg3_all.err; echo bench3all_rc=$?
timeout 900 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; echo bench4_rc=$?
