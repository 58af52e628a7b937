# A/B of two libtio builds: planner us/round at C3/C2 and lifetime time at C3/C2
A=${A:-tools/micro/base.so}; B=${B:-tools/micro/exp_all.so}
for lib in $A $B $A $B; do for c in c3 c2; do echo -n "$(basename $lib) "; TIO_LIB_PATH=$lib timeout 300 python tools/time_virtual.py $c 1 2>&1 | tail -1; done; done
timeout 600 python tools/time_lifetime.py c3 $A $B $A $B 2>&1 | grep lifetime
timeout 300 python tools/time_lifetime.py c2 $A $B 2>&1 | grep lifetime
