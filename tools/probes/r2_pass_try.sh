# pass launches: unit parity vs per-step launches, IPC parity (flags on = pass launches), then solo A/B
mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests/test_gpu_pass.py -x -q -p no:cacheprovider > gpurun_out/pass.log 2>&1; echo "pass rc=$?" >> gpurun_out/pass.log
timeout -s KILL 600 python -m pytest tests/test_gpu_ipc.py -x -q -p no:cacheprovider > gpurun_out/ipc.log 2>&1; echo "ipc rc=$?" >> gpurun_out/ipc.log
S=gpurun_out/solo_pass.jsonl; rm -f $S
for v in "RTPB_NO_PASS=1" "RTPB_NO_PASS=0"; do
  for n in 2 4 8; do
    env RTPB_FLAGS=1 $v timeout -s KILL 90 python bench.py --config b --solo $n --steps 50 --no-cpu-baseline --no-e2e 2>gpurun_out/err_b$n.txt | tail -1 \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'v':'$v','cfg':'b','n':$n,'tf':d['tflops_per_gpu'],'ms':d['ms_per_step'],'exec':d.get('step_execution')}))" >> $S || echo "fail b$n $v" >> $S
  done
  env RTPB_FLAGS=1 $v timeout -s KILL 200 python tools/rtp_sweep.py --config d --solo 8 --blocks 4 --steps 3 --warmup 2 --out gpurun_out/d8_tmp.jsonl > /dev/null 2>gpurun_out/err_d8.txt \
     && tail -1 gpurun_out/d8_tmp.jsonl | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'v':'$v','cfg':'d','n':8,'tf':d['tflops_per_gpu'],'ms':d['ms_per_step']}))" >> $S || echo "fail d8 $v" >> $S
done
cat $S
