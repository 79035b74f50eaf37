mkdir -p gpurun_out
S=gpurun_out/solo_split.jsonl; rm -f $S
run_b() {
  local lab=$1 n=$2; shift 2
  env "$@" timeout -s KILL 90 python bench.py --config b --solo $n --steps 50 --no-cpu-baseline --no-e2e 2>gpurun_out/err_$lab$n.txt | tail -1 \
    | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'v':'$lab','cfg':'b','n':$n,'tf':round(d['tflops_per_gpu'],1),'ms':d['ms_per_step'],'pl':[(l['kind'],round(l['us'],1),l['sms']) for l in d['roofline']['per_launch_in_step_order']]}))" >> $S || echo "fail b$n $lab" >> $S
}
for n in 8 4 2; do run_b split_model $n; done
for n in 8 4; do
  RTPB_FLAGS=1 timeout -s KILL 300 python tools/rtp_sweep.py --config c --solo $n --steps 3 --warmup 2 --out gpurun_out/c_tmp.jsonl > /dev/null 2>&1 \
     && tail -1 gpurun_out/c_tmp.jsonl | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'v':'default','cfg':'c','n':$n,'tf':round(d['tflops_per_gpu'],1),'ms':d['ms_per_step']}))" >> $S || echo "fail c$n" >> $S
done
RTPB_FLAGS=1 timeout -s KILL 300 python tools/rtp_sweep.py --config d --solo 8 --blocks 4 --steps 3 --warmup 2 --out gpurun_out/d8_tmp.jsonl > /dev/null 2>&1 \
     && tail -1 gpurun_out/d8_tmp.jsonl | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'v':'default','cfg':'d','n':8,'tf':round(d['tflops_per_gpu'],1),'ms':d['ms_per_step']}))" >> $S || echo "fail d8" >> $S
cat $S
