mkdir -p gpurun_out
GRAPH=1 SOLO=8 RTPB_FLAGS=1 timeout 300 python tools/timeline.py > gpurun_out/tl_b8_flags.txt 2>&1
RTPB_FLAGS=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launch_d8.csv python tools/rtp_sweep.py --config d --solo 8 --blocks 1 --steps 1 --warmup 1 > gpurun_out/launch_d8.log 2>&1
for f in 0 1; do RTPB_FLAGS=$f timeout 300 python bench.py --config b --solo 8 --steps 50 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/solo_b8_f$f.json; done
