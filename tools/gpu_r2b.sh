#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TIO_LIB_PATH=tools/micro/libtio_vdbg.so timeout 120 python tools/vdebug.py 2 2>&1 | grep -v "^\[vdbg\]" | tail -5
timeout 900 python -m pytest tests/test_gpu_sharded_plan.py tests/test_distributed.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -8
timeout 600 python tools/time_virtual.py c3 1 2 4
timeout 600 python tools/time_virtual.py c2 1 2 4
