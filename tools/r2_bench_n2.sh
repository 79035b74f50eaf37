#!/bin/bash
# The bench's multi-process path on one GPU: torchrun N = 2 with --same-device (IPC transport, both ranks on
# GPU 0; a plumbing/parity check, not a throughput number), and the reference arm under torchrun.
mkdir -p gpurun_out
timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 2 --same-device --config b --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_n2_same.log 2>&1; echo "rc=$?" >> gpurun_out/bench_n2_same.log
timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29535 \
  bench.py --gpus 2 --same-device --config d --blocks 2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_n2_same_d.log 2>&1; echo "rc=$?" >> gpurun_out/bench_n2_same_d.log
timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 \
  bench.py --impl reference --gpus 2 --steps 3 --warmup 3 > gpurun_out/bench_n2_ref.log 2>&1; echo "rc=$?" >> gpurun_out/bench_n2_ref.log
