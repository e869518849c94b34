#!/bin/bash
# GPU parity tests against the debug-checks build (device bounds checks, bounded mbarrier waits):
# the pool has compute-sanitizer closed, so this is the memory/progress check of the kernels
mkdir -p gpurun_out
OICA_LIB=$PWD/paper_2408_17118_b200/liboica_dbg.so timeout 2400 python -m pytest tests/test_gpu_parity.py \
  tests/test_gpu_golden.py -q -rf -k "not cfg4 and not cfg3" > gpurun_out/debug_checks.log 2>&1
echo "rc=$?"; tail -3 gpurun_out/debug_checks.log
OICA_LIB=$PWD/paper_2408_17118_b200/liboica_dbg.so timeout 600 python scripts/sanitize_run.py >> gpurun_out/debug_checks.log 2>&1
echo "sanitize_run rc=$?"; tail -3 gpurun_out/debug_checks.log
