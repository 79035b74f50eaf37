# configs (c) / (d) at N = 8 shapes: per-step backward (default) vs the backward pass launches
mkdir -p gpurun_out
S=gpurun_out/solo_bwd_big.jsonl; rm -f $S
for cfg in d c; do
  for v in "RTPB_PASS_BWD=0" "RTPB_PASS_BWD=1"; do
    B=""; [ $cfg = d ] && B="--blocks 4"
    env $v timeout -s KILL 400 python tools/rtp_sweep.py --config $cfg --solo 8 $B --steps 3 --warmup 2 --out gpurun_out/big_tmp.jsonl > /dev/null 2>&1 \
      && tail -1 gpurun_out/big_tmp.jsonl | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'v':'$v','cfg':'$cfg','n':8,'tf':round(d['tflops_per_gpu'],1),'ms':d['ms_per_step']}))" >> $S || echo "fail $cfg $v" >> $S
  done
done
cat $S
