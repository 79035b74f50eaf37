mkdir -p gpurun_out
O=gpurun_out/sweep.jsonl; R=gpurun_out/rot.jsonl; rm -f $O $R
timeout 300 python tools/rotation_bench.py --simulate 2 --out $R > gpurun_out/rot2.log 2>&1 || echo rot2 fail
timeout 300 python tools/rotation_bench.py --simulate 8 --out $R > gpurun_out/rot8.log 2>&1 || echo rot8 fail
for n in 2 4 8; do timeout 200 python tools/rtp_sweep.py --config b --simulate $n --out $O >> gpurun_out/sweep.log 2>&1 || echo b$n fail; done
timeout 200 python tools/rtp_sweep.py --config b --out $O >> gpurun_out/sweep.log 2>&1 || echo b1 fail
for m in outofplace inplace; do timeout 300 python tools/rtp_sweep.py --config c --simulate 8 --mode $m --out $O >> gpurun_out/sweep.log 2>&1 || echo c8$m fail; done
timeout 300 python tools/rtp_sweep.py --config c --simulate 2 --out $O >> gpurun_out/sweep.log 2>&1 || echo c2 fail
timeout 400 python tools/rtp_sweep.py --config d --steps 3 --out $O >> gpurun_out/sweep.log 2>&1 || echo d1 fail
timeout 400 python tools/rtp_sweep.py --config d --simulate 8 --blocks 2 --steps 3 --out $O >> gpurun_out/sweep.log 2>&1 || echo d8 fail
tail -5 gpurun_out/sweep.log
