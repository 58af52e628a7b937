# planner phase profile (debug build): wide (default) and narrow kernels at C3, C2
for w in default 0; do
  if [ $w = 0 ]; then export TIO_PLAN_WIDE_TILES=0; fi
  TIO_LIB_PATH=tools/micro/libtio_prof.so timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-migration > gpurun_out/bench_prof_$w.raw 2>/dev/null
  grep "plan-profile" gpurun_out/bench_prof_$w.raw | sort | uniq -c | head -4
  grep '^{' gpurun_out/bench_prof_$w.raw | tail -1 > gpurun_out/bench_prof_$w.json
  python -c "import json;d=json.load(open('gpurun_out/bench_prof_$w.json'));print('$w C3',json.dumps(d['planner'].get('debug_build')), d['planner']['us_per_round']);print('$w C2',json.dumps(d['c2']['planner'].get('debug_build')), d['c2']['planner']['us_per_round'])"
done
