"""Rotation-primitive micro-bench (BASELINE.json config (e)): ring shifts of
one shard per worker, 1 MB - 1 GB, clockwise / counter-clockwise, out-of-place
(double-buffered: receive into the spare) and in-place (chunked through one
staging chunk), plus the ring allgather of the same per-rank chunk as the
comparison collective (the paper's "custom NCCL-test"), and the
overlap of a rotation with a step GEMM running on another stream.

Distributed (one process per GPU, NCCL send/recv over NVLink):
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 tools/rotation_bench.py
Simulated (N workers sharing GPU 0; a shift is N device-local copies, so the
numbers are HBM copy rates, not NVLink):
    python tools/rotation_bench.py --simulate N

Prints one JSON line per measurement; GB/s are bytes SENT per rank per
second (a shift sends and receives one shard per rank). Times are CUDA
events on the issuing stream, max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2311_01635_b200 import rtp  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--simulate", type=int, default=0, help="N workers on GPU 0 (no NCCL)")
    ap.add_argument("--sizes-mb", default="1,4,16,64,256,1024")
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--allgather-max-mb", type=int, default=256)
    ap.add_argument("--out", default=None, help="also append the JSON lines to this file")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if args.simulate:
        n = args.simulate
        torch.cuda.set_device(0)
        grp = rtp.WorkerGroup(n, "lockstep", devices=[0] * n)
        mode = f"simulated: {n} workers on one GPU (device-local copies)"
    else:
        import torch.distributed as dist
        n = world
        torch.cuda.set_device(local)
        dev = torch.device("cuda", local)
        dist.init_process_group("nccl", device_id=dev)
        uid = torch.zeros(128, dtype=torch.uint8, device=dev)
        if rank == 0:
            uid.copy_(torch.frombuffer(bytearray(rtp.WorkerGroup.nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(uid, 0)
        grp = rtp.WorkerGroup.nccl(n, rank, local, bytes(uid.cpu().numpy().tobytes()))
        mode = f"nccl: {n} processes, one GPU each"
    ranks = grp.local_ranks
    dev = grp.stream(ranks[0]).device
    cur = torch.cuda.current_stream(dev)

    def tmax(ms):
        if dist is None:
            return ms
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def timed(fn, iters):
        fn()
        torch.cuda.synchronize(dev)
        if dist is not None:
            dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(cur)
        for _ in range(iters):
            fn()
        b.record(cur)
        torch.cuda.synchronize(dev)
        return tmax(a.elapsed_time(b) / iters)

    lines = []

    def emit(d):
        d["mode"] = mode
        d["n"] = n
        lines.append(d)
        if rank == 0:
            print(json.dumps(d), flush=True)

    # A step GEMM for the overlap measurement (config (d) ffn1 step at N=8:
    # M=16384, I=4096, per=2048 -> 275 GFLOP), on a side stream.
    gm, gi, gp = 16384, 4096, 2048
    gx = torch.randn(gm, gi, device=dev).to(torch.bfloat16)
    gw = (torch.randn(gi * gp + gp, device=dev) * 0.01).to(torch.bfloat16)
    gy = torch.empty(gm, gp, dtype=torch.bfloat16, device=dev)
    side = torch.cuda.Stream(dev)

    def gemm():
        side.wait_stream(cur)
        for r in ranks:
            rtp.fwd_step(gx, gw, gy, 0, gp, stream=side)
        cur.wait_stream(side)

    t_gemm = timed(gemm, 5)
    emit({"what": "gemm_alone", "ms": t_gemm, "gemms_per_rank": 1, "local_workers": len(ranks),
          "shape": [gm, gi, gp]})

    for mb in (int(v) for v in args.sizes_mb.split(",")):
        nbytes = mb << 20
        nel = nbytes // 2
        W = [torch.randn(nel, device=dev).to(torch.bfloat16) for _ in ranks]
        SP = [torch.empty_like(w) for w in W]
        G = [torch.zeros(nel, dtype=torch.float32, device=dev) for _ in ranks]  # fp32 grads: 2x bytes
        state = {"W": W, "SP": SP}

        def cw_oop():
            grp.rotate("cw", state["W"], spares=state["SP"], keep_spare=True)
            state["W"], state["SP"] = state["SP"], state["W"]

        def ccw_wg_oop():
            grp.rotate("ccw", state["W"], grads=G, spares=state["SP"], keep_spare=True)
            state["W"], state["SP"] = state["SP"], state["W"]

        def cw_inplace():
            grp.rotate("cw", state["W"])

        def ccw_wg_inplace():
            grp.rotate("ccw", state["W"], grads=G)

        iters = max(2, min(args.iters, int(4096 / mb)))
        for name, fn, sent in (("cw_outofplace", cw_oop, nbytes), ("cw_inplace_chunked", cw_inplace, nbytes),
                               ("ccw_wg_outofplace", ccw_wg_oop, 3 * nbytes),
                               ("ccw_wg_inplace_chunked", ccw_wg_inplace, 3 * nbytes)):
            ms = timed(fn, iters)
            emit({"what": name, "shard_mb": mb, "bytes_sent_per_rank": sent, "ms": ms,
                  "gbs_per_rank": sent / (ms * 1e-3) / 1e9,
                  "aggregate_gbs": sent * n / (ms * 1e-3) / 1e9})

        # overlap of one out-of-place shift with the step GEMM on another stream
        def both():
            side.wait_stream(cur)
            for r in ranks:
                rtp.fwd_step(gx, gw, gy, 0, gp, stream=side)
            cw_oop()
            cur.wait_stream(side)

        t_rot = timed(cw_oop, iters)
        t_both = timed(both, max(2, iters // 2))
        hidden = (t_gemm + t_rot - t_both) / min(t_gemm, t_rot)
        emit({"what": "overlap_cw_outofplace_vs_gemm", "shard_mb": mb, "ms_rotation": t_rot, "ms_gemm": t_gemm,
              "ms_both": t_both, "overlap_frac": max(0.0, min(1.0, hidden)),
              "exposed_ms": max(0.0, t_both - t_gemm)})

        if mb <= args.allgather_max_mb:
            out = [torch.empty(n * nel, dtype=torch.bfloat16, device=dev) for _ in ranks]
            ms = timed(lambda: grp.allgather(W, out), max(2, iters // 2))
            sent = (n - 1) * nbytes
            emit({"what": "ring_allgather", "shard_mb": mb, "bytes_sent_per_rank": sent, "ms": ms,
                  "gbs_per_rank": sent / (ms * 1e-3) / 1e9})
            if dist is not None:
                flat = torch.empty(n * nel, dtype=torch.bfloat16, device=dev)
                ms = timed(lambda: dist.all_gather_into_tensor(flat, W[0]), max(2, iters // 2))
                emit({"what": "nccl_allgather", "shard_mb": mb, "bytes_sent_per_rank": sent, "ms": ms,
                      "gbs_per_rank": sent / (ms * 1e-3) / 1e9})
            del out
        del W, SP, G, state
        torch.cuda.empty_cache()

    if args.out and rank == 0:
        with open(args.out, "a") as f:
            for d in lines:
                f.write(json.dumps(d) + "\n")
    grp.close()
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
