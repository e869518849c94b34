#!/bin/bash
mkdir -p gpurun_out/sanitizer
for tool in memcheck racecheck synccheck; do
  for c in san_fp32 san_tc san_wide; do
    timeout 900 compute-sanitizer --tool $tool --print-limit 50 --log-file gpurun_out/sanitizer/${tool}_$c.log \
      python scripts/sanitize_run.py $c > gpurun_out/sanitizer/${tool}_$c.out 2>&1
    echo "$tool $c rc=$? $(tail -1 gpurun_out/sanitizer/${tool}_$c.log)"
  done
done
