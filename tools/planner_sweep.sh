#!/bin/bash
# planner knobs sweep + a source-level ncu capture of the round loop
mkdir -p gpurun_out
for w in 0 96 100000; do
  TIO_WARP_REFIT_MAX=$w timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-migration > gpurun_out/sweep_w$w.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/sweep_w$w.json')); p=d['planner']
print('warp_refit_max=$w', round(d['value']), 'us/round', round(p['us_per_round'],2), 'max_eval', round(p['max_evaluate_us_per_round'],2), p['phase_us_per_round_block0'], d['config']['plan_sha256'][:8])"
done
timeout 900 ncu --section SourceCounters --section WarpStateStats --section LaunchStats --section Occupancy \
  --clock-control none --import-source on -k regex:plan_loop_kernel -c 1 -o gpurun_out/prof_plan2 -f \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-migration > /dev/null 2> gpurun_out/ncu_plan2.err
echo "ncu rc=$?"
