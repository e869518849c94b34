#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python bench.py --config cfg3_large --all-components --no-e2e --no-cpu-baseline --precision fp32 > gpurun_out/bench_cfg3_all_fp32.json 2> gpurun_out/bench_cfg3_all_fp32.err; echo a=$?
timeout 900 python bench.py --config cfg3_large --all-components --no-e2e --no-cpu-baseline --precision tc_split > gpurun_out/bench_cfg3_all_split.json 2> gpurun_out/bench_cfg3_all_split.err; echo b=$?
