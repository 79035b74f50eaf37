# simulated N = 8 rings on one GPU: exposed rotation with the per-step event schedule vs the
# arrival-flag / pass-launch schedule (RTPB_SIM_FLAGS: each worker's grids on its share of the SMs)
mkdir -p gpurun_out
W=gpurun_out/sweep_r2b.jsonl; rm -f $W
for f in 0 1; do
  for m in outofplace; do
    RTPB_FLAGS=$f RTPB_SIM_FLAGS=$f timeout -s KILL 500 python tools/rtp_sweep.py --config c --simulate 8 --mode $m --steps 3 --warmup 2 --out $W > /dev/null 2>gpurun_out/simsweep_c_$f.err || echo "fail c8 $f" >> $W
  done
  RTPB_FLAGS=$f RTPB_SIM_FLAGS=$f timeout -s KILL 600 python tools/rtp_sweep.py --config d --simulate 8 --blocks 2 --steps 3 --warmup 2 --out $W > /dev/null 2>gpurun_out/simsweep_d_$f.err || echo "fail d8 $f" >> $W
  RTPB_FLAGS=$f RTPB_SIM_FLAGS=$f timeout -s KILL 300 python tools/rtp_sweep.py --config b --simulate 8 --steps 5 --warmup 2 --out $W > /dev/null 2>gpurun_out/simsweep_b_$f.err || echo "fail b8 $f" >> $W
done
python - <<'PY'
import json
for l in open("gpurun_out/sweep_r2b.jsonl"):
    try: d = json.loads(l)
    except Exception: print(l.strip()); continue
    print(d.get("config"), d.get("n"), d.get("rotation_mode"), d.get("ms_per_step"), d.get("exposed_comm_frac"), d.get("tflops_per_gpu"))
PY
