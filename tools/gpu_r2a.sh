#!/bin/bash
# round-2 measurement batch A: lifetime (chain-free prefixes), RED floor,
# sharded planner (virtual + two processes), planner phase profile, cuFile
# probe, C4 determinism probe
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi -L
timeout 300 python tools/time_lifetime.py c3 paper_2506_06472_b200/_lib/libtio.so
timeout 300 python tools/time_lifetime.py c2 paper_2506_06472_b200/_lib/libtio.so
timeout 300 python tools/micro/red_floor.py c3
timeout 900 python -m pytest tests/test_gpu_sharded_plan.py tests/test_distributed.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -15
timeout 600 python tools/time_virtual.py c3 1 2 4
timeout 600 python tools/time_virtual.py c2 1 2 4
TIO_LIB_PATH=tools/micro/libtio_prof.so timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-migration > gpurun_out/bench_prof.json 2>gpurun_out/bench_prof.err
python -c "import json;d=json.load(open('gpurun_out/bench_prof.json'));print('C3',json.dumps(d['planner']));print('C2',json.dumps(d['c2']['planner']))"
df -hT /tmp /dev/shm /root 2>&1
for p in /tmp/tio_cufile.bin /dev/shm/tio_cufile.bin /root/tio_cufile.bin; do timeout 300 tools/micro/cufile_probe $p 1024; done
free -g | head -2; nproc
timeout 900 python tools/det_probe.py 8b efficient det 2>&1 | tail -4
timeout 900 python tools/det_probe.py 8b flash det 2>&1 | tail -4
