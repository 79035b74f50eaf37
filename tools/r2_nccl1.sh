mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "nccl or NCCL" > gpurun_out/nccl1.log 2>&1; echo "rc=$?" >> gpurun_out/nccl1.log
