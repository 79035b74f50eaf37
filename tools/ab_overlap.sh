# A/B of the N=1 dX || dW overlap split (GPU box).
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$? ; tail -3 gpurun_out/gpu_tests.log
for v in none default 56 64 74 84 92; do
  if [ $v = none ]; then export RTPB_NO_OVERLAP=1; else unset RTPB_NO_OVERLAP; fi
  if [ $v = none ] || [ $v = default ]; then unset RTPB_OVERLAP_DX_SMS; else export RTPB_OVERLAP_DX_SMS=$v; fi
  timeout 300 python bench.py --steps 100 --no-cpu-baseline > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err
  python -c "import json;d=json.load(open('gpurun_out/ab_$v.json'));r=d['roofline'];print('$v', round(d['value'],1), round(d['ms_per_step']*1e3,1), 'eager', round(d['eager_ms_per_step']*1e3,1), 'ach', round(r['achieved'],1), [ (p['kind'],p['us'],p['start_us'],p['sms']) for p in r['per_launch_in_step_order']])" || tail -5 gpurun_out/ab_$v.err
done
