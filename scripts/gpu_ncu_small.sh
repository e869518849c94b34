#!/bin/bash
# ncu --set full of the small-problem update and SIMT step kernels (exp. 1 shape, eager launches)
mkdir -p gpurun_out
for k in k_update k_step_simt; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k --launch-skip 60 -c 2 \
    -o gpurun_out/ncu_small_$k -f python scripts/small_profile.py --reps 1 --eager --cases exp1_L20 \
    > gpurun_out/ncu_small_$k.log 2>&1; echo "$k rc=$?"
done
