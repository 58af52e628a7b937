#!/bin/bash
# Build libtio from the sources of a git revision (A/B timing against the
# working tree):  tools/build_rev.sh <rev> <out.so> [-DNAME=VALUE ...]
set -e
rev=$1; out=$2; shift 2
d=$(mktemp -d)
mkdir -p "$d/pkg/csrc" "$d/include"           # same relative layout (csrc/../../include/tio.h)
for f in $(git ls-tree --name-only "$rev" paper_2506_06472_b200/csrc/); do
  git show "$rev:$f" > "$d/pkg/csrc/$(basename "$f")"
done
git show "$rev:include/tio.h" > "$d/include/tio.h"
for f in "$d"/pkg/csrc/*.cu; do
  /usr/local/cuda/bin/nvcc "$@" -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
    -Xcompiler -fPIC -diag-suppress 177 -c "$f" -o "${f%.cu}.o" &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$out" "$d"/pkg/csrc/*.o -lpthread
rm -rf "$d"
