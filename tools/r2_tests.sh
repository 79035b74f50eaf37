mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_pass.py -x -q -p no:cacheprovider > gpurun_out/pass.log 2>&1; echo "pass rc=$?" >> gpurun_out/pass.log
timeout -s KILL 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo "all rc=$?" >> gpurun_out/gputest.log
