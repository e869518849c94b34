#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/parity.log 2>&1; echo parity=$?; tail -1 gpurun_out/parity.log
rm -f gpurun_out/xscale.log
for N in 64 128 256; do timeout 300 python scripts/tc_variants.py 0 $N >> gpurun_out/xscale.log 2>&1; OICA_TC_EPI=3 timeout 300 python scripts/tc_variants.py 3 $N >> gpurun_out/xscale.log 2>&1; done
cat gpurun_out/xscale.log | cut -c1-190
timeout 900 python bench.py --config cfg2_eeg_shaped --no-cpu-baseline > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; echo b2=$?
timeout 900 python bench.py --config cfg3_large --no-cpu-baseline > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err; echo b3d=$?
