#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_cases.py;
# logs to gpurun_out/sanitizer/ (copied to profiles/ when judged)
cd "$(dirname "$0")/.."
out=gpurun_out/sanitizer
mkdir -p $out
CS=/usr/local/cuda/bin/compute-sanitizer
for case in ${CASES:-lifetime_plan virtual replay online}; do
  for tool in ${TOOLS:-memcheck racecheck synccheck}; do
    extra=""
    [ "$tool" = memcheck ] && extra="--leak-check no"
    # library kernels of PyTorch are not ours: only libtio kernels (namespace tio) are checked
    timeout ${SAN_TIMEOUT:-900} $CS --tool $tool $extra --kernel-name kns=tio --print-limit 50 \
        python tools/sanitize_cases.py $case > $out/${case}_${tool}.log 2>&1
    echo "$case $tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|ok' $out/${case}_${tool}.log | tr '\n' ' ')"
  done
done
