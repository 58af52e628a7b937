#!/bin/bash
# One GPU session: smoke, parity tests, bench, launch list, ncu capture of one kernel (NCU_KERNEL, default k_events).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi -L
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
[ -z "$SKIP_TESTS" ] && timeout ${TEST_TIMEOUT:-900} python -m pytest tests -m gpu -q ${PYTEST_ARGS} 2>&1 | tail -40
[ -z "$SKIP_BENCH" ] && timeout 900 python bench.py --steps 3 --warmup 3 ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?"; cat gpurun_out/bench.json; tail -5 gpurun_out/bench.err
if [ -z "$NO_NCU" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-migration ${BENCH_ARGS} > /dev/null 2>gpurun_out/ncu1.err
echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${NCU_KERNEL:-k_events} -c 1 \
    -o gpurun_out/prof_${NCU_KERNEL:-k_events} -f python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-migration ${BENCH_ARGS} > /dev/null 2>gpurun_out/ncu2.err
echo "ncu full rc=$?"
fi
