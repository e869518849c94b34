#!/bin/bash
# bench lines of the small and mid configs: default step line + all components (device-side loop)
# and the eager variant (per-step timing), plus the cfg3 default line
mkdir -p gpurun_out/all
for c in cfg0_tiny cfg1_artificial cfg2_eeg_shaped; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/all/bench_$c.json 2> gpurun_out/all/bench_$c.err; echo "$c rc=$?"
  timeout 900 python bench.py --config $c --all-components --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/all/bench_${c}_all.json 2> gpurun_out/all/bench_${c}_all.err; echo "$c all rc=$?"
  timeout 900 python bench.py --config $c --all-components --warmup 3 --no-e2e --no-cpu-baseline --eager > gpurun_out/all/bench_${c}_all_eager.json 2> gpurun_out/all/bench_${c}_all_eager.err; echo "$c all eager rc=$?"
done
timeout 1200 python bench.py --config cfg3_large --steps 3 --warmup 3 > gpurun_out/all/bench_cfg3_large.json 2> gpurun_out/all/bench_cfg3_large.err; echo "cfg3 rc=$?"
for f in gpurun_out/all/*.json; do python -c "
import json,sys;d=json.loads(open('$f').read().splitlines()[-1]);r=d['roofline']
print('$f'.split('/')[-1], round(d['value'],1), 'ms/step', round(d['ms_per_step'],3), 'all_s', d['seconds_all_components'], 'kern', r['achieved'] and round(r['achieved'],1), 'frac', r['frac'] and round(r['frac'],3), 'share', r['share_of_step'] and round(r['share_of_step'],3), d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'), (d['config'].get('golden_match') or {}).get('pass'))
"; done
