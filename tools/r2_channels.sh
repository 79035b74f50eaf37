mkdir -p gpurun_out
S=gpurun_out/solo_channels.jsonl; rm -f $S
run_b() {
  local lab=$1 n=$2; shift 2
  env "$@" timeout -s KILL 90 python bench.py --config b --solo $n --steps 50 --no-cpu-baseline --no-e2e 2>gpurun_out/err_$lab$n.txt | tail -1 \
    | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'v':'$lab','cfg':'b','n':$n,'tf':round(d['tflops_per_gpu'],1),'ms':d['ms_per_step'],'pl':[(l['kind'],round(l['us'],1),l['sms']) for l in d['roofline']['per_launch_in_step_order']]}))" >> $S || echo "fail b$n $lab" >> $S
}
for n in 8 4 2; do
  run_b two_ch $n
  run_b one_ch $n RTPB_PASS_ONE_CHANNEL=1
  run_b two_ch_dx96 $n RTPB_PASS_DX_SMS=96
  run_b two_ch_dx110 $n RTPB_PASS_DX_SMS=110
done
cat $S
timeout -s KILL 600 python -m pytest tests/test_gpu_pass.py -x -q -p no:cacheprovider > gpurun_out/pass.log 2>&1; echo "rc=$?" >> gpurun_out/pass.log
