#!/bin/bash
# Session-3 A/B and check of the unrolled device-loop body (kLoopUnroll; OICA_LOOP_UNROLL overrides):
# small-problem timings and cfg 2 all components per unroll factor, then the -m gpu suite.
set -u
mkdir -p gpurun_out/unroll
for U in ${UNROLLS:-1 2 4}; do
  OICA_LOOP_UNROLL=$U python scripts/small_profile.py --reps 7 > gpurun_out/unroll/small_U$U.json 2>&1
  OICA_LOOP_UNROLL=$U timeout 600 python bench.py --config cfg2_eeg_shaped --all-components --warmup 3 --no-e2e \
    --no-cpu-baseline > gpurun_out/unroll/cfg2_all_U$U.json 2>gpurun_out/unroll/cfg2_all_U$U.err
done
for U in ${UNROLLS:-1 2 4}; do cat gpurun_out/unroll/small_U$U.json; python scripts/show_line.py gpurun_out/unroll/cfg2_all_U$U.json; done
[ -n "${NO_TESTS:-}" ] || NO_BENCH=1 bash scripts/gpu_jobs.sh tests
