#!/bin/bash
# Round measurement: smoke, GPU tests, default bench (C3 + C2 + C4), reference
# arm, launch list, ncu --set full of the planner (C3) and the lifetime kernels
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi -L
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
[ -z "$SKIP_TESTS" ] && timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -5
timeout 1800 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
[ -z "$SKIP_REF" ] && { timeout 1200 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"; }
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-migration > /dev/null 2>gpurun_out/ncu1.err
echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"plan_loop_kernel|k_events|k_kernels" -c 3 \
    -o gpurun_out/prof_final -f python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-migration --secondary "" > /dev/null 2>gpurun_out/ncu2.err
echo "ncu full rc=$?"
