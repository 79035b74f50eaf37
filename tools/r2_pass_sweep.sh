# A/B: pass launches vs per-step at config (b) N = 2/4/8 and (d) N = 8 (solo); dX SM share sweep
mkdir -p gpurun_out
S=gpurun_out/solo_sweep2.jsonl; rm -f $S
run_b() {  # $1 = label, $2 = n, rest = env
  local lab=$1 n=$2; shift 2
  env RTPB_FLAGS=1 "$@" timeout -s KILL 90 python bench.py --config b --solo $n --steps 50 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 \
    | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'v':'$lab','cfg':'b','n':$n,'tf':round(d['tflops_per_gpu'],1),'ms':d['ms_per_step']}))" >> $S || echo "fail b$n $lab" >> $S
}
run_d() {
  local lab=$1; shift 1
  env RTPB_FLAGS=1 "$@" timeout -s KILL 200 python tools/rtp_sweep.py --config d --solo 8 --blocks 4 --steps 3 --warmup 2 --out gpurun_out/d8_tmp.jsonl > /dev/null 2>&1 \
     && tail -1 gpurun_out/d8_tmp.jsonl | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'v':'$lab','cfg':'d','n':8,'tf':round(d['tflops_per_gpu'],1),'ms':d['ms_per_step']}))" >> $S || echo "fail d8 $lab" >> $S
}
for n in 2 4 8; do run_b nopass $n RTPB_NO_PASS=1; run_b pass $n RTPB_NO_PASS=0; done
for d in 50 96 110; do run_b pass_dx$d 8 RTPB_PASS_DX_SMS=$d; done
run_b pass_fwdonly 8 RTPB_PASS_BWD=0
run_d nopass RTPB_NO_PASS=1
run_d pass RTPB_NO_PASS=0
run_d pass_bwd RTPB_PASS_BWD=1
GRAPH=1 SOLO=8 RTPB_FLAGS=1 timeout -s KILL 120 python tools/timeline.py > gpurun_out/tl_b8_pass3.txt 2>&1
cat $S
timeout -s KILL 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo "all rc=$?" >> gpurun_out/gputest.log
