#!/bin/bash
# dev check: parity + iteration logs (tail cost) + all-components timings
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py -m gpu -x -q > gpurun_out/par.log 2>&1; tail -2 gpurun_out/par.log
for c in cfg4_scaling cfg3_large; do
  timeout 300 python scripts/iteration_log.py $c --components 2 --out gpurun_out/iterlog_$c.json > gpurun_out/iterlog_$c.txt 2>&1
  tail -6 gpurun_out/iterlog_$c.txt
done
for c in ${ALL_CFGS:-cfg2_eeg_shaped cfg3_large}; do
  OICA_TRACE=1 timeout 300 python bench.py --config $c --all-components --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/all_$c.json 2> gpurun_out/all_$c.err
  python scripts/show_bench.py gpurun_out/all_$c.json | cut -c1-160
done
