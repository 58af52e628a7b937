#!/bin/bash
# Build a libtio variant with extra nvcc defines (tuning experiments):
#   tools/build_variant.sh <out.so> -DNAME=VALUE ...
set -e
out=$1; shift
d=$(mktemp -d)
for f in paper_2506_06472_b200/csrc/*.cu; do
  /usr/local/cuda/bin/nvcc "$@" -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    -diag-suppress 177 -c "$f" -o "$d/$(basename "$f" .cu).o" &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$out" "$d"/*.o -lpthread
rm -rf "$d"
