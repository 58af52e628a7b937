# planner variants: us/round and plan sha at C3 / C2 (tools/time_virtual.py, 1 rank)
for v in ${VARIANTS:-base q}; do for c in c3 c2; do echo -n "$v "; TIO_LIB_PATH=tools/micro/pl_$v.so timeout 300 python tools/time_virtual.py $c 1 2>&1 | tail -1; done; done
