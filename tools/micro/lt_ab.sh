# lifetime v1 (working tree default) vs v3 (warp-contiguous, -DLT_V3): parity tests on v3, then timing
TIO_LIB_PATH=tools/micro/lt_v3.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "lifetime or period or golden or invalid or fuzz or random" 2>&1 | tail -3
timeout 600 python tools/time_lifetime.py c3 tools/micro/exp_all.so tools/micro/lt_v3.so tools/micro/exp_all.so tools/micro/lt_v3.so 2>&1 | grep lifetime
timeout 300 python tools/time_lifetime.py c2 tools/micro/exp_all.so tools/micro/lt_v3.so 2>&1 | grep lifetime
