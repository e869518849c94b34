#!/bin/bash
# GPU jobs of this repository (run through gpurun; outputs under gpurun_out/):
#   bash scripts/gpu_jobs.sh tests [pytest -k expr]   -m gpu suite (durations) + a short bench line
#   bash scripts/gpu_jobs.sh quick                    parity + bench-contract tests, small-problem timings
#   bash scripts/gpu_jobs.sh small                    per-kernel durations of small problems (ncu, warm caches)
#   bash scripts/gpu_jobs.sh ncu-small                ncu --set full of the update / FP32 step (Exp. 1 shape)
#   bash scripts/gpu_jobs.sh bench [CFG]              bench line + the ncu launch list of the same command
#   bash scripts/gpu_jobs.sh bench-all                bench lines of cfgs 0-3 (steps, all components, eager)
#   bash scripts/gpu_jobs.sh parity                   golden + tier-C parity with the printed worst cases
#   bash scripts/gpu_jobs.sh debug-checks             parity suite against liboica_dbg.so (bounds checks)
#   bash scripts/gpu_jobs.sh ncu-step CFG...          ncu --set full of one full-L step launch per config
#                                                     (summaries + raw csv; the roofline `traffic` source)
set -u
mkdir -p gpurun_out
job=${1:-tests}
shift || true
case $job in
tests)
  nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt 2>&1
  K="${1:-}"
  if [ -n "$K" ]; then
    timeout 2400 python -m pytest tests -m gpu -q -rf --durations=25 -k "$K" > gpurun_out/gpu_tests.log 2>&1
  else
    timeout 2400 python -m pytest tests -m gpu -q -rf --durations=25 > gpurun_out/gpu_tests.log 2>&1
  fi
  echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
  tail -30 gpurun_out/gpu_tests.log
  if [ -z "${NO_BENCH:-}" ]; then
    timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
    echo "bench rc=$?"
  fi
  ;;
quick)
  timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_contract.py -q -rf -x --durations=10 \
    > gpurun_out/quick_tests.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/quick_tests.log
  tail -25 gpurun_out/quick_tests.log
  python scripts/small_profile.py --reps 5 > gpurun_out/small.json 2> gpurun_out/small.err; echo "small rc=$?"
  cat gpurun_out/small.json
  ;;
small)
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
    --log-file gpurun_out/small_eager.csv python scripts/small_profile.py --reps 1 --eager --cases ${CASES:-cfg1,exp1_L20} \
    > gpurun_out/small_ncu_eager.log 2>&1
  echo "ncu eager rc=$?"
  ;;
ncu-small)
  for k in k_update k_step_simt; do
    timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k --launch-skip 60 -c 2 \
      -o gpurun_out/ncu_small_$k -f python scripts/small_profile.py --reps 1 --eager --cases exp1_L20 \
      > gpurun_out/ncu_small_$k.log 2>&1
    echo "$k rc=$?"
  done
  ;;
bench)
  CFG=${1:-cfg4_scaling}
  timeout 1200 python bench.py --config $CFG --steps ${STEPS:-3} --warmup ${WARMUP:-3} ${EXTRA:-} \
    > gpurun_out/bench_$CFG.json 2> gpurun_out/bench_$CFG.err
  echo "bench rc=$?"
  timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none -c ${NCU_C:-1200} --csv \
    --log-file gpurun_out/launches_$CFG.csv python bench.py --config $CFG --steps 1 --warmup ${WARMUP:-3} \
    --no-e2e --no-all --no-cpu-baseline ${EXTRA:-} > gpurun_out/ncu_$CFG.log 2>&1
  echo "ncu rc=$?"
  ;;
bench-all)
  mkdir -p gpurun_out/all
  for c in cfg0_tiny cfg1_artificial cfg2_eeg_shaped; do
    timeout 900 python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/all/bench_$c.json 2> gpurun_out/all/bench_$c.err
    timeout 900 python bench.py --config $c --all-components --warmup 3 --no-e2e --no-cpu-baseline \
      > gpurun_out/all/bench_${c}_all.json 2> gpurun_out/all/bench_${c}_all.err
    timeout 900 python bench.py --config $c --all-components --warmup 3 --no-e2e --no-cpu-baseline --eager \
      > gpurun_out/all/bench_${c}_all_eager.json 2> gpurun_out/all/bench_${c}_all_eager.err
  done
  timeout 1200 python bench.py --config cfg3_large --steps 3 --warmup 3 > gpurun_out/all/bench_cfg3_large.json \
    2> gpurun_out/all/bench_cfg3_large.err
  for f in gpurun_out/all/*.json; do python scripts/show_line.py $f; done
  ;;
parity)
  timeout 2400 python -m pytest tests/test_gpu_golden.py tests/test_gpu_certificate.py -q -s -rf \
    > gpurun_out/parity_summary.log 2>&1
  echo "rc=$?"; grep -E "precision|tier C|full L|passed|failed" gpurun_out/parity_summary.log | tail -20
  ;;
debug-checks)
  OICA_LIB=$PWD/paper_2408_17118_b200/liboica_dbg.so timeout 2400 python -m pytest tests/test_gpu_parity.py \
    tests/test_gpu_golden.py -q -rf -k "not cfg4 and not cfg3" > gpurun_out/debug_checks.log 2>&1
  echo "rc=$?"; tail -3 gpurun_out/debug_checks.log
  OICA_LIB=$PWD/paper_2408_17118_b200/liboica_dbg.so timeout 600 python scripts/sanitize_run.py \
    >> gpurun_out/debug_checks.log 2>&1
  echo "sanitize_run rc=$?"; tail -3 gpurun_out/debug_checks.log
  ;;
ncu-step)
  ncu --query-metrics 2>/dev/null | grep -i -E "tmem|tensor_mem|utc|pipe_tensor" > gpurun_out/ncu_tensor_metric_names.txt
  for CFG in "${@:-cfg4_scaling}"; do
    CMD="python bench.py --config $CFG --steps 1 --warmup 3 --no-e2e --no-all --no-cpu-baseline --data device --eager"
    timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:k_step_tc -s 2 -c 1 \
      -o /tmp/prof_step_$CFG $CMD > gpurun_out/ncu_full_$CFG.log 2>&1; echo "full_$CFG rc=$?"
    python scripts/ncu_summary.py full /tmp/prof_step_$CFG.ncu-rep > gpurun_out/ncu_full_${CFG}.json 2>&1
    ncu -i /tmp/prof_step_$CFG.ncu-rep --page raw --csv > gpurun_out/ncu_raw_${CFG}.csv 2>/dev/null
    ncu -i /tmp/prof_step_$CFG.ncu-rep --page details --csv > gpurun_out/ncu_details_${CFG}.csv 2>/dev/null
  done
  ;;
*)
  echo "unknown job $job"; exit 2
  ;;
esac
