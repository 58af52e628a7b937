#!/bin/bash
# validation + A/B batch (working tree = exp_all): GPU suite, planner/lifetime A/B, v3 lifetime, walk stats
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -4
bash tools/micro/ab.sh
bash tools/micro/lt_ab.sh
bash tools/micro/planprof.sh 2>&1 | head -12
# C4 plan-rate calibration: the measured bidirectional rate vs 0.92 of it (0.9 and 0.8 x peak)
for rs in 1.0 0.92; do timeout 1200 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --secondary "" --config c1 --c4-rate-scale $rs --c4-fracs 0.8 0.9 --no-identity 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); m=d['migration']
print('rate_scale', m['plan_rate_scale'], [(r['capacity_frac_of_trace_peak'], round(r['step_vs_ideal'],3), round(r['model_step_vs_ideal'],3), r['plan']['entries']) for r in m['runs']], 'ideal', round(m['ideal']['step_ms'],1))"; done
