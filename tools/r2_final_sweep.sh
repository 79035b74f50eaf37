#!/bin/bash
# Simulated N-worker sweeps (workers share one GPU) with the final code: exposed rotation and per-worker memory.
mkdir -p gpurun_out
O=gpurun_out/sweep_r2z.jsonl; rm -f $O
for n in 2 4 8; do timeout 200 python tools/rtp_sweep.py --config b --simulate $n --out $O >> gpurun_out/sweep_r2z.log 2>&1 || echo b$n fail; done
for m in outofplace inplace; do timeout 300 python tools/rtp_sweep.py --config c --simulate 8 --mode $m --out $O >> gpurun_out/sweep_r2z.log 2>&1 || echo c8$m fail; done
timeout 400 python tools/rtp_sweep.py --config d --simulate 8 --blocks 2 --steps 3 --out $O >> gpurun_out/sweep_r2z.log 2>&1 || echo d8 fail
