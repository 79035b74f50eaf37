#!/bin/bash
# Round-end evidence refresh on the GPU box: solo / config (d) sweeps, the
# reference arm, the ncu launch list + full capture. Writes gpurun_out/.
set -u
mkdir -p gpurun_out
O=gpurun_out/solo_r1.jsonl; rm -f $O
timeout 300 python tools/rtp_sweep.py --config d --blocks 4 --steps 3 --warmup 2 --out $O > /dev/null 2>&1 || echo "fail d1"
timeout 300 python tools/rtp_sweep.py --config d --solo 8 --blocks 4 --steps 3 --warmup 2 --out $O > /dev/null 2>&1 || echo "fail d8"
for n in 2 4 8; do
  timeout 300 python bench.py --solo $n --steps 50 --no-cpu-baseline 2>/dev/null >> $O || echo "fail solo b$n"
done
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref_arm.json 2> gpurun_out/ref_arm.err || echo "fail ref arm"
bash tools/profile_round.sh ${1:-r1c} 12 3
