#!/bin/bash
# bench line (no profiler) then the ncu launch list of the same command (per-kernel durations)
mkdir -p gpurun_out
CFG=${CFG:-cfg4_scaling}
timeout 1200 python bench.py --config $CFG --steps ${STEPS:-3} --warmup ${WARMUP:-3} ${EXTRA:-} > gpurun_out/bench_$CFG.json 2> gpurun_out/bench_$CFG.err
echo "bench rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/bench_$CFG.json').read().splitlines()[-1]);r=d['roofline'];print(d['value'],d['ms_per_step'],d['seconds_all_components'],r['achieved'],r['frac'],r['share_of_step'],d['clocks'])"
if [ -n "$NCU" ]; then
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none -c ${NCU_C:-800} --csv --log-file gpurun_out/launches_$CFG.csv \
  python bench.py --config $CFG --steps 1 --warmup ${WARMUP:-3} --no-e2e --no-all --no-cpu-baseline ${EXTRA:-} > gpurun_out/ncu_$CFG.log 2>&1
echo "ncu rc=$?"
fi
