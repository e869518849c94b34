#!/bin/bash
mkdir -p gpurun_out
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -s -k "paper_experiment" > gpurun_out/parity_exp.log 2>&1; echo parity_exp=$?
grep -E "estimated|passed|failed|Error" gpurun_out/parity_exp.log | tail -10
timeout 1500 python scripts/paper_experiments.py --out gpurun_out/paper_experiments.json > gpurun_out/paper_experiments.log 2>&1; echo harness=$?
tail -25 gpurun_out/paper_experiments.log
