#!/bin/bash
# Round-2 GPU check: the gpu test suite (durations), then a short bench line.
# usage: gpurun -- 'bash scripts/gpu_r2.sh [pytest -k expr]'
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt 2>&1
K="${1:-}"
if [ -n "$K" ]; then
  timeout 2400 python -m pytest tests -m gpu -q -rf --durations=25 -k "$K" > gpurun_out/gpu_tests.log 2>&1
else
  timeout 2400 python -m pytest tests -m gpu -q -rf --durations=25 > gpurun_out/gpu_tests.log 2>&1
fi
echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
tail -30 gpurun_out/gpu_tests.log
if [ -z "$NO_BENCH" ]; then
  timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
  echo "bench rc=$?"
  python -c "import json;d=json.loads(open('gpurun_out/bench.json').read().splitlines()[-1]);print({k:d[k] for k in ('value','ms_per_step','seconds_all_components','clocks')}, d['roofline']['frac'])"
fi
