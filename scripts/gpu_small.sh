#!/bin/bash
# small-problem per-kernel durations (warm caches), eager launches under ncu
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none --cache-control none --csv \
  --log-file gpurun_out/small_eager.csv python scripts/small_profile.py --reps 1 --eager --cases ${CASES:-cfg1,exp1_L20} \
  > gpurun_out/small_ncu_eager.log 2>&1; echo "ncu eager rc=$?"
