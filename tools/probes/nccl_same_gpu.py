"""Probe: can two NCCL ranks share one GPU here? (torchrun --nproc-per-node 2)"""
import os
import torch
import torch.distributed as dist
rank = int(os.environ["RANK"])
torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
t = torch.full((4,), float(rank), device="cuda")
dist.all_reduce(t)
print("rank", rank, "allreduce ok", t.tolist(), flush=True)
dist.destroy_process_group()
