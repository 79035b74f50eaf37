#!/bin/bash
# compute-sanitizer over the step-GEMM protocols (run on the GPU box).
# Writes gpurun_out/sanitize_<tool>_<case>.log; summary lines on stdout.
set -u
mkdir -p gpurun_out
CS=${CS:-/usr/local/cuda/bin/compute-sanitizer}
for tool in memcheck synccheck racecheck; do
  for case in fused splitk flags f32; do
    env=""
    [ "$case" = flags ] && env="RTPB_FLAGS=1"
    log=gpurun_out/sanitize_${tool}_${case}.log
    timeout ${CASE_TIMEOUT:-900} env $env $CS --tool $tool --error-exitcode 9 --print-limit 50 \
      python tools/sanitize_driver.py $case 2 > $log 2>&1
    rc=$?
    echo "$tool $case rc=$rc :: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|sanitize case' $log | tr '\n' ' ')"
  done
done
