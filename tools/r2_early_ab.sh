mkdir -p gpurun_out
O=gpurun_out/early_ab.txt; rm -f $O
for i in 1 2; do
for v in default earlymath; do
  if [ $v = default ]; then unset RTPB_LIB; else export RTPB_LIB=build/var_earlymath/librtpb.so; fi
  for s in "16384 4096 16384" "16384 4096 2048" "8192 768 3072"; do
    echo "$v $(timeout -s KILL 120 python tools/gemm_one.py $s fwd_gelu 2>&1 | tail -1)" >> $O
  done
done
done
for i in 1 2; do
for v in default earlymath; do
  if [ $v = default ]; then unset RTPB_LIB; else export RTPB_LIB=build/var_earlymath/librtpb.so; fi
  timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); pk=d['roofline'].get('per_kernel',{}); print('bench d N=1 $v', round(d['value'],1), d['clocks']['sm_mhz'], {k:round(v['tflops_per_gpu_time']) for k,v in pk.items()})" >> $O 2>&1
done
done
unset RTPB_LIB
cat $O
