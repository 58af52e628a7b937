#!/bin/bash
# planner knob sweep: events/s and us/round per setting (plan hash must not change)
mkdir -p gpurun_out
for w in ${SWEEP:-0 96}; do
  TIO_WARP_REFIT_MAX=$w timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-migration > gpurun_out/sweep_w$w.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/sweep_w$w.json')); p=d['planner']
print('warp_refit_max=$w', round(d['value']), 'us/round', round(p['us_per_round'],2), {k: v for k, v in p.items() if k not in ('kernel','bound')}, d['config']['plan_sha256'][:8])"
done
