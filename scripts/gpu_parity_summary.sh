#!/bin/bash
# parity evidence with the printed worst cases (goldens tiers A/B, tier C certificate)
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_gpu_golden.py tests/test_gpu_certificate.py -q -s -rf > gpurun_out/parity_summary.log 2>&1
echo "rc=$?"; grep -E "precision|tier C|full L|passed|failed" gpurun_out/parity_summary.log | tail -20
