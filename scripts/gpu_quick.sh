#!/bin/bash
# quick GPU validation: parity tests (no full-size goldens) + small-problem timings
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_contract.py -q -rf -x --durations=10 > gpurun_out/quick_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/quick_tests.log
tail -25 gpurun_out/quick_tests.log
python scripts/small_profile.py --reps 5 > gpurun_out/small.json 2> gpurun_out/small.err; echo "small rc=$?"
cat gpurun_out/small.json; tail -3 gpurun_out/small.err
