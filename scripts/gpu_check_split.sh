#!/bin/bash
# dev check: GPU suite + iteration logs + all-components timings + full-L step timing
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
for c in cfg2_eeg_shaped cfg3_large cfg4_scaling; do
  timeout 300 python scripts/iteration_log.py $c --components 2 --out gpurun_out/iterlog_$c.json > gpurun_out/iterlog_$c.txt 2>&1
  tail -4 gpurun_out/iterlog_$c.txt
done
for c in cfg1_artificial cfg2_eeg_shaped cfg3_large; do
  OICA_TRACE=1 timeout 300 python bench.py --config $c --all-components --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/all_$c.json 2> gpurun_out/all_$c.err
  python scripts/show_bench.py gpurun_out/all_$c.json | cut -c1-160
done
timeout 300 python scripts/tc_variants.py 0 256 128 64 2>&1 | grep '^{'
