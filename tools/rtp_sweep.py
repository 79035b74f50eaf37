"""RTP MLP sweep over BASELINE.json configs (b), (c), (d): step throughput,
exposed rotation time and per-GPU peak memory against the paper's model.

    python tools/rtp_sweep.py --config b --simulate 8 [--mode inplace]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 tools/rtp_sweep.py --config d

Simulated: N workers share GPU 0 (Lockstep transport; a ring shift is N
device-local copies). Throughput is then the whole group's work on ONE GPU
and the exposed-comm figure says whether the copies hide under the step
GEMMs; NVLink numbers need the distributed launch. Memory is per worker
(the device ledger is kept per worker), i.e. what one GPU would hold.

Exposed rotation time = T(step) - T(step with rtpb_debug_skip_comm), where
the skip run keeps the schedule, events and bookkeeping but moves no bytes.
Configs:
  b  MLP 768->3072->768, 8192 tokens per worker
  c  MLP 8192->28672->8192, 32768 global tokens (4096 per worker at N=8)
  d  stack of L MLP blocks 4096->16384->4096 (L=32 by default; fewer with
     --blocks), 16384 tokens per worker (seq 2048 x batch 64 over 8 GPUs)
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2311_01635_b200 import _lib, rtp  # noqa: E402

CONFIGS = {"b": (768, 3072, 8192, None, 1), "c": (8192, 28672, None, 32768, 1), "d": (4096, 16384, 16384, None, 32)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="b", choices=sorted(CONFIGS))
    ap.add_argument("--simulate", type=int, default=0)
    ap.add_argument("--solo", type=int, default=0,
                    help="one rank of an N-way ring on GPU 0, shifts skipped: per-GPU compute at N-way shapes")
    ap.add_argument("--mode", default="outofplace", choices=["inplace", "outofplace"])
    ap.add_argument("--blocks", type=int, default=None)
    ap.add_argument("--tokens-per-worker", type=int, default=None)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--out", default=None)
    ap.add_argument("--no-chain", action="store_true",
                    help="do not link the blocks (no block-to-block prefetch of the first shift)")
    args = ap.parse_args()

    h, f, tpw, tglobal, blocks = CONFIGS[args.config]
    if args.blocks:
        blocks = args.blocks
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if args.solo:
        n = args.solo
        torch.cuda.set_device(0)
        grp = rtp.WorkerGroup.solo(n, 0, 0)
        how = f"solo: rank 0 of a {n}-way ring on one GPU, shifts skipped (per-GPU compute only)"
    elif args.simulate:
        n = args.simulate
        torch.cuda.set_device(0)
        grp = rtp.WorkerGroup(n, "lockstep", devices=[0] * n)
        how = f"simulated: {n} workers on one GPU"
    else:
        n = world
        torch.cuda.set_device(local)
        dev = torch.device("cuda", local)
        if world > 1:
            import torch.distributed as dist
            dist.init_process_group("nccl", device_id=dev)
            uid = torch.zeros(128, dtype=torch.uint8, device=dev)
            if rank == 0:
                uid.copy_(torch.frombuffer(bytearray(rtp.WorkerGroup.nccl_unique_id()), dtype=torch.uint8))
            dist.broadcast(uid, 0)
            grp = rtp.WorkerGroup.nccl(n, rank, local, bytes(uid.cpu().numpy().tobytes()))
            how = f"nccl: {n} processes, one GPU each"
        else:
            grp = rtp.WorkerGroup(1)
            how = "single GPU"
    M = args.tokens_per_worker or tpw or (tglobal // n)
    T = M * n
    ranks = grp.local_ranks
    dev = grp.stream(ranks[0]).device
    cur = torch.cuda.current_stream(dev)

    per_block_params = 2 * h * f + f + h
    mlps = []
    for b in range(blocks):
        m = rtp.RtpMlp(grp, f"block{b}", h, f, "bf16", seed=42, stream_base=b * per_block_params)
        m.set_rotation_mode(args.mode)
        m.begin_step()
        mlps.append(m)
    if not args.no_chain:
        for a, b in zip(mlps, mlps[1:]):
            a.chain(b)  # each block posts its neighbour's first shift under its own last step
    g = torch.Generator(device=dev).manual_seed(42 + rank)
    xs = [(torch.rand(M, h, device=dev, generator=g) * 2 - 1).to(torch.bfloat16) for _ in ranks]
    dys = [(torch.rand(M, h, device=dev, generator=g) * 2 - 1).to(torch.bfloat16) for _ in ranks]
    acts = [[torch.empty(M, h, dtype=torch.bfloat16, device=dev) for _ in ranks] for _ in range(blocks)]
    grads = [[torch.empty(M, h, dtype=torch.bfloat16, device=dev) for _ in ranks] for _ in range(2)]

    def step():
        for m in mlps:
            m.zero_grads()
        inp = xs
        for b, m in enumerate(mlps):  # x_{b+1} = mlp_b(x_b)
            m.forward(inp, out=acts[b])
            inp = acts[b]
        up = dys
        for b in range(blocks - 1, -1, -1):
            out = grads[b % 2]
            mlps[b].backward(up, out=out)
            up = out

    def tmax(ms):
        if dist is None:
            return ms
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def timed(k):
        torch.cuda.synchronize(dev)
        if dist is not None:
            dist.barrier()
        a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(cur)
        for _ in range(k):
            step()
        b_.record(cur)
        torch.cuda.synchronize(dev)
        return tmax(a.elapsed_time(b_) / k)

    for _ in range(args.warmup):
        step()
    grp.reset_ledger_peaks()
    ms = timed(args.steps)
    _lib.lib.rtpb_debug_skip_comm(1)
    try:
        step()
        ms_nocomm = timed(args.steps)
    finally:
        _lib.lib.rtpb_debug_skip_comm(0)

    flops = 12.0 * T * h * f * blocks
    if args.solo:
        flops /= n  # one rank's share
    wb = (h * f + f + f * h + h) * 2 * blocks  # bf16 weights, whole model
    gb = (h * f + f + f * h + h) * 4 * blocks  # fp32 gradients
    led = [grp.ledger(r) for r in ranks]
    worst = max(led, key=lambda d: d["peak_total"])
    pgc = worst["peak_param"] + worst["peak_grad"] + worst["peak_comm"]
    bytes_sent = (n - 1) / n * (2 * wb + gb) if n > 1 else 0.0  # per GPU per step
    line = {"config": args.config, "how": how, "n": n, "rotation_mode": args.mode, "chained": not args.no_chain, "h": h, "f": f, "blocks": blocks,
            "tokens_per_worker": M, "global_tokens": T, "steps": args.steps,
            "ms_per_step": ms, "ms_per_step_compute_only": ms_nocomm,
            "exposed_comm_ms": max(0.0, ms - ms_nocomm), "exposed_comm_frac": max(0.0, ms - ms_nocomm) / ms,
            "tflops_whole_group" if not args.solo else "tflops_per_gpu": flops / (ms * 1e-3) / 1e12,
            "rotation_bytes_sent_per_gpu": bytes_sent,
            "memory_per_worker": {
                "peak_param": worst["peak_param"], "peak_grad": worst["peak_grad"], "peak_comm": worst["peak_comm"],
                "peak_activation": worst["peak_activation"], "peak_other": worst["peak_other"],
                "peak_total_ledger": worst["peak_total"], "param_grad_comm": pgc,
                "model_inplace": (wb + gb) / n, "model_outofplace": (wb + gb + max(wb, gb)) / n,
                "vs_model": pgc / ((wb + gb + (max(wb, gb) if args.mode == "outofplace" and n > 1 else 0)) / n)}}
    if args.solo:
        # projected N-GPU step from the measured per-GPU compute and the ring
        # bytes over NVLink 5 (900 GB/s per direction): perfect / no overlap
        t_nvl = bytes_sent / 900e9 * 1e3
        line["projection"] = {"nvlink_ms": t_nvl, "step_ms_overlapped": max(ms, t_nvl),
                              "step_ms_serial": ms + t_nvl,
                              "tflops_per_gpu_overlapped": flops / (max(ms, t_nvl) * 1e-3) / 1e12,
                              "note": "measured compute of one rank; rotation bytes modelled, not measured"}
    if rank == 0:
        print(json.dumps(line), flush=True)
        if args.out:
            with open(args.out, "a") as fh:
                fh.write(json.dumps(line) + "\n")
    for m in mlps:
        m.close()
    grp.close()
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
