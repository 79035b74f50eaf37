mkdir -p gpurun_out
O=gpurun_out/colsum_ab.txt; rm -f $O
for v in "X=0" "RTPB_COLSUM_MAX_I=8192"; do
  echo "== $v" >> $O
  for s in "16384 4096 16384" "16384 16384 4096" "16384 4096 2048" "16384 16384 512"; do
    env $v timeout -s KILL 120 python tools/gemm_one.py $s wgrad >> $O 2>&1
  done
done
for i in 1 2; do
  for v in "X=0" "RTPB_COLSUM_MAX_I=8192"; do
    env $v timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); pk=d['roofline'].get('per_kernel',{}); print('bench d N=1 $v', round(d['value'],1), d['clocks']['sm_mhz'], {k:round(v['tflops_per_gpu_time']) for k,v in pk.items()})" >> $O 2>&1
  done
done
for v in "X=0" "RTPB_COLSUM_MAX_I=8192"; do
  env $v timeout -s KILL 300 python tools/rtp_sweep.py --config d --solo 8 --blocks 4 --steps 3 --warmup 2 --out gpurun_out/d8_tmp.jsonl > /dev/null 2>&1 \
     && tail -1 gpurun_out/d8_tmp.jsonl | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('d solo8 $v', round(d['tflops_per_gpu'],1))" >> $O
  env $v timeout -s KILL 90 python bench.py --config b --solo 8 --steps 50 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('b solo8 $v', round(d['tflops_per_gpu'],1))" >> $O
done
cat $O
