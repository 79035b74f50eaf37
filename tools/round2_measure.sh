#!/bin/bash
# Round-2 evidence on the GPU box: bench lines for configs d (default), b, c;
# per-GPU compute at N-way shapes (solo) with events and with arrival flags;
# simulated N-worker sweeps (exposed rotation, per-worker memory). gpurun_out/.
set -u
mkdir -p gpurun_out
B=gpurun_out/bench_r2.jsonl; S=gpurun_out/solo_r2.jsonl; W=gpurun_out/sweep_r2.jsonl
rm -f $B $S $W
timeout 600 python bench.py --steps 10 --warmup 3 2>/dev/null | tail -1 >> $B || echo "fail bench d"
timeout 300 python bench.py --config b --steps 50 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 >> $B || echo "fail bench b"
timeout 300 python bench.py --config c --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 >> $B || echo "fail bench c"
for f in 0 1; do
  for n in 2 4 8; do
    RTPB_FLAGS=$f timeout 300 python bench.py --config b --solo $n --steps 50 --no-cpu-baseline --no-e2e 2>/dev/null \
      | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); d['flags']=$f; print(json.dumps(d))" >> $S \
      || echo "fail solo b$n f$f"
  done
  RTPB_FLAGS=$f timeout 600 python tools/rtp_sweep.py --config d --solo 8 --blocks 4 --steps 3 --warmup 2 --out $S \
    > /dev/null 2>&1 || echo "fail solo d8 f$f"
  RTPB_FLAGS=$f timeout 600 python tools/rtp_sweep.py --config c --solo 8 --steps 3 --warmup 2 --out $S \
    > /dev/null 2>&1 || echo "fail solo c8 f$f"
done
for n in 2 4 8; do timeout 300 python tools/rtp_sweep.py --config b --simulate $n --out $W > /dev/null 2>&1 || echo "fail sim b$n"; done
for m in outofplace inplace; do
  timeout 400 python tools/rtp_sweep.py --config c --simulate 8 --mode $m --out $W > /dev/null 2>&1 || echo "fail sim c8 $m"
done
timeout 600 python tools/rtp_sweep.py --config d --simulate 8 --blocks 2 --steps 3 --out $W > /dev/null 2>&1 || echo "fail sim d8"
echo done
