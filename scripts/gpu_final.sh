#!/bin/bash
# Final round evidence at HEAD: smoke, bench lines (cfg4 default, cfg3, cfg2, all-components),
# ncu launch lists + one --set full capture of the step kernel at cfg4 and cfg3.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$?; tail -1 gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build_rc=$?
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
timeout 900 python bench.py > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; echo bench4_rc=$?
timeout 600 python bench.py --config cfg3_large --no-cpu-baseline > gpurun_out/bench_cfg3.json 2>/dev/null; echo bench3_rc=$?
timeout 600 python bench.py --config cfg2_eeg_shaped --no-cpu-baseline > gpurun_out/bench_cfg2.json 2>/dev/null; echo bench2_rc=$?
timeout 600 python bench.py --config cfg1_artificial --no-cpu-baseline > gpurun_out/bench_cfg1.json 2>/dev/null; echo bench1_rc=$?
for C in cfg3_large cfg2_eeg_shaped cfg1_artificial cfg0_tiny; do
  timeout 900 python bench.py --config $C --all-components --no-e2e --no-cpu-baseline > gpurun_out/bench_${C}_all.json 2>/dev/null; echo all_$C=$?
  timeout 900 python bench.py --config $C --all-components --no-e2e --no-cpu-baseline --reduce > gpurun_out/bench_${C}_all_red.json 2>/dev/null; echo allr_$C=$?
done
timeout 1200 python bench.py --all-components --no-e2e --no-cpu-baseline > gpurun_out/bench_cfg4_scaling_all.json 2>/dev/null; echo all_cfg4=$?
timeout 1200 python bench.py --all-components --no-e2e --no-cpu-baseline --reduce > gpurun_out/bench_cfg4_scaling_all_red.json 2>/dev/null; echo allr_cfg4=$?
for CFG in cfg4_scaling cfg3_large; do
  CMD="python bench.py --config $CFG --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
  $CMD > gpurun_out/plain_$CFG.json 2> gpurun_out/plain_$CFG.err && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:oica -c 4000 \
      --csv --log-file gpurun_out/launches_$CFG.csv $CMD > gpurun_out/ncu_list_$CFG.log 2>&1; echo list_$CFG=$?
  timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:k_step_tc -s 2 -c 1 \
      -o /tmp/prof_tc_${CFG}_final $CMD > gpurun_out/ncu_full_$CFG.log 2>&1; echo full_$CFG=$?
  # keep gpurun_out small (64 MiB cap): summaries only
  python scripts/ncu_summary.py full /tmp/prof_tc_${CFG}_final.ncu-rep > gpurun_out/ncu_full_${CFG}_final.json 2>&1
  ncu -i /tmp/prof_tc_${CFG}_final.ncu-rep --page raw --csv > gpurun_out/ncu_raw_${CFG}_final.csv 2>/dev/null
done
ls -la gpurun_out | head -50
