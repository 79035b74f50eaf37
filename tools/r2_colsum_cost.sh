#!/bin/bash
# dW kernel time with the bias column sum fused (default) vs without it (RTPB_NO_COLSUM: the separate
# column-sum kernel, listed apart), per kernel from an ncu launch list.
mkdir -p gpurun_out; out=gpurun_out/colsum_cost.txt; : > $out
for v in default nocolsum; do
  if [ $v = default ]; then unset RTPB_LIB; else export RTPB_LIB=build/var_$v/librtpb.so; fi
  for s in "16384 4096 16384" "16384 4096 2048"; do
    echo "== $v $s" >> $out
    timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/gemm_one.py $s wgrad,wgrad_as_dgrad 2>/dev/null \
      | python -c "
import csv,sys,collections
t=collections.defaultdict(list)
for r in csv.reader(l for l in sys.stdin if l.startswith('\"')):
    if len(r)>14 and r[12]=='gpu__time_duration.sum': t[r[4][:60]].append(float(r[14].replace(',','')))
for k,v in t.items(): print(f'   {len(v):3d} x {sum(v)/len(v):9.1f} {k}')" >> $out
  done
done
