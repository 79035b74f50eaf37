mkdir -p gpurun_out
RTPB_TRACE_HOST=1 timeout -s KILL 40 python tools/probes/sim_hang.py 4 > gpurun_out/sim_dbg.txt 2>&1
timeout -s KILL 900 python -m pytest tests/test_gpu_pass.py -x -q -p no:cacheprovider > gpurun_out/pass.log 2>&1; echo "rc=$?" >> gpurun_out/pass.log
