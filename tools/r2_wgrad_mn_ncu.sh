#!/bin/bash
# ncu full capture: dW on MN-major operands (wgrad) vs the same product on pre-transposed operands
# (wgrad_as_dgrad) at config (d) N = 1 and N = 8 shapes.
mkdir -p gpurun_out
for s in "16384 4096 16384" "16384 4096 2048"; do
  tag=$(echo $s | tr ' ' _)
  for k in wgrad wgrad_as_dgrad; do
    timeout 300 ncu --set full --clock-control none -k regex:rtp_gemm -s 3 -c 1 -o gpurun_out/mn_${k}_$tag \
      python tools/gemm_one.py $s $k > gpurun_out/mn_${k}_$tag.log 2>&1
    ncu -i gpurun_out/mn_${k}_$tag.ncu-rep --page raw --csv > gpurun_out/mn_${k}_$tag.csv 2>/dev/null
    ncu -i gpurun_out/mn_${k}_$tag.ncu-rep --page details --csv > gpurun_out/mn_${k}_${tag}_details.csv 2>/dev/null
    rm -f gpurun_out/mn_${k}_$tag.ncu-rep
  done
done
