mkdir -p gpurun_out
O=gpurun_out/ab_n1.txt; rm -f $O
for i in 1 2; do
  for v in base cur; do
    if [ $v = base ]; then D=build/base_tree; else D=.; fi
    (cd $D && timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1) \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); pk=d['roofline'].get('per_kernel',{}); print('$v', round(d['value'],1), round(d['ms_per_step'],2), d['clocks']['sm_mhz'], {k:round(v['tflops_per_gpu_time']) for k,v in pk.items()})" >> $O 2>&1 || echo "fail $v" >> $O
  done
done
cat $O
