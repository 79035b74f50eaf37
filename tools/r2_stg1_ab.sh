#!/bin/bash
# A/B: dW (WGRAD) epilogue with one fp32 staging buffer per warp (more mainloop stages) vs two.
out=gpurun_out/stg1_ab.txt; : > $out
for v in default stg1 default stg1; do
  if [ $v = default ]; then unset RTPB_LIB; else export RTPB_LIB=build/var_$v/librtpb.so; fi
  echo "== $v" >> $out
  for s in "16384 4096 16384" "16384 16384 4096" "16384 4096 2048" "16384 16384 512"; do
    timeout 120 python tools/gemm_one.py $s wgrad,wgrad_as_dgrad,dgrad 2>&1 | grep -v Warn >> $out
  done
done
for v in default stg1 default stg1; do
  if [ $v = default ]; then unset RTPB_LIB; else export RTPB_LIB=build/var_$v/librtpb.so; fi
  echo "== bench $v" >> $out
  timeout 300 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['clocks'], {k:round(v['tflops_per_gpu_time']) for k,v in d['roofline']['per_kernel'].items()})" >> $out 2>&1
done
