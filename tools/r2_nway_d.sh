#!/bin/bash
# config (d) (and (c)) at N = 8 shard shapes: dX || dW SM split forced (RTPB_NWAY_DX_SMS) vs default (no split).
out=gpurun_out/nway_d.txt; : > $out
run() { timeout 300 env "$@" python bench.py --solo 8 --blocks 4 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print(round(d['value'],1), d['config']['workload'][-10:], d['clocks']['sm_mhz'], {k:(round(v['tflops_per_gpu_time']),round(v['avg_us'],1)) for k,v in r['per_kernel'].items()})" >> $out; }
for v in 0 84 64 100 0 84; do
  echo "== d NWAY=$v" >> $out
  if [ $v = 0 ]; then run X=1; else run RTPB_NWAY_DX_SMS=$v; fi
done
