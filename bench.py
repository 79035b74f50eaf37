"""RTP MLP fwd+bwd benchmark (BASELINE.json metric: "RTP MLP fwd+bwd TFLOP/s/GPU
& peak HBM/GPU at 1/2/4/8 B200 vs CPU ref").

Workloads (BASELINE.json configs), bf16, Flyweight init
(SplitMix64 seed 42, SerialModel parameter order), synthetic activations:
  d (default)  stack of 32 RTP MLP blocks 4096 -> 16384 -> 4096, 16384 tokens
               per GPU (seq 2048 x global batch 64 over 8 GPUs), weak scaling:
               north_star's roofline target config; fits one GPU (~62 GB)
  b            one MLP block 768 -> 3072 -> 768, 8192 tokens per GPU, weak
  c            one MLP block 8192 -> 28672 -> 8192, 32768 global tokens
               (strong scaling), in-place vs out-of-place peak memory
A step = zero_grads + forward through every block + backward in reverse,
through the library's public API (RtpMlp, C ABI). FLOPs per step =
12 * T * h * f * blocks (fwd, dX, dW at 2*T*h*f per linear).

python bench.py [--config d] [--gpus N --steps K --warmup W] [--impl reference]
N > 1: launch with torch.distributed.run, one process per GPU, NCCL ring.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SEED = 42
METRIC = "RTP MLP fwd+bwd TFLOP/s/GPU & peak HBM/GPU at 1/2/4/8 B200 vs CPU ref"
UNIT = "TFLOP/s"

# name: (h, f, blocks, tokens per GPU (weak) or None, global tokens (strong) or None, label)
CONFIGS = {
    "b": (768, 3072, 1, 8192, None, "rtp_mlp_768x3072x768 (config b)"),
    "c": (8192, 28672, 1, None, 32768, "rtp_mlp_8192x28672x8192 (config c)"),
    "d": (4096, 16384, 32, 16384, None, "rtp_mlp_stack32_4096x16384 (config d)"),
}


def flops_per_step(tokens: int, h: int, f: int, blocks: int) -> float:
    return 12.0 * tokens * h * f * blocks


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["bf16_tflops"]), float(p.get("bf16_tflops_sustained", p["bf16_tflops"])), "measured"
    except Exception:
        return 1590.0, 1400.0, "fallback"


def host_info():
    model = platform.processor() or ""
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        affinity = len(os.sched_getaffinity(0))
    except Exception:
        affinity = os.cpu_count()
    return {"nproc": affinity, "cpu_count": os.cpu_count(), "cpu_model": model}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.samples = []
        self._proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self._proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                           "--format=csv,noheader,nounits", "-lms", "100"],
                                          stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self._proc = None
        return self

    def _read(self):
        for line in self._proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.samples.append(parts)

    def __exit__(self, *a):
        if self._proc:
            time.sleep(0.25)
            self._proc.terminate()
            try:
                self._proc.wait(timeout=5)
            except Exception:
                self._proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no-samples"], "samples": 0}

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        sm = [num(s[0]) for s in self.samples if num(s[0]) is not None]
        mx = [num(s[1]) for s in self.samples if num(s[1]) is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[3 + i].lower().startswith("active")})
        loaded = [v for v in sm if v and v > 600] or sm
        loaded.sort()
        return {"sm_mhz": loaded[len(loaded) // 2] if loaded else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples),
                "power_w_max": max((num(s[2]) or 0) for s in self.samples)}


def dist_env():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), \
        int(os.environ.get("LOCAL_RANK", "0"))


# ------------------------------------------------------------------ reference arm
def _cpu_workers(h, f):
    cores = host_info()["nproc"] or 1
    workers = 1
    while workers * 2 <= cores and f % (workers * 2) == 0 and h % (workers * 2) == 0:
        workers *= 2
    return workers


def cpu_reference(cfg, sample_rows=None, target_s=12.0, iters=1):
    """Times the reference's own CPU implementation of the path (oracle/_ref:
    the reference sources compiled by path; two RtpLinear + gelu composed as
    model.cpp:77-105, Concurrent transport, one worker thread per host core,
    fp64) on ONE block of the config at a bounded row sample. A stack's step
    is linear in FLOPs, so the rate extrapolates to the whole workload
    (labelled). Falls back to the C restatement when oracle/_ref is absent."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as orc
    h, f, blocks = CONFIGS[cfg][:3]
    workers = _cpu_workers(h, f)
    try:
        R = orc.Reference()
        kind = "reference"

        def run(rows, k=1):
            return R.time_mlp(workers, rows, h, f, SEED, iters=k, concurrent=True)
    except Exception:
        O = orc.Oracle()
        kind = "port"
        import numpy as np
        rng = np.random.default_rng(SEED)
        w1, b1 = rng.uniform(-0.1, 0.1, (h, f)), rng.uniform(-0.1, 0.1, f)
        w2, b2 = rng.uniform(-0.1, 0.1, (f, h)), rng.uniform(-0.1, 0.1, h)

        def run(rows, k=1):
            t = 0.0
            for _ in range(k):
                x, dy = rng.uniform(-1, 1, (rows, h)), rng.uniform(-1, 1, (rows, h))
                t0 = time.perf_counter()
                O.rtp_mlp(workers, w1, b1, w2, b2, x, dy)
                t += time.perf_counter() - t0
            return t
    if sample_rows is None:
        probe = 8 * workers
        t = run(probe)
        rate = flops_per_step(probe, h, f, 1) / max(t, 1e-6)
        sample_rows = int(target_s * rate / flops_per_step(1, h, f, 1))
        cap = CONFIGS[cfg][3] or CONFIGS[cfg][4]
        sample_rows = max(workers, min(cap, (sample_rows // workers) * workers))
    secs = run(sample_rows, iters)
    value = flops_per_step(sample_rows, h, f, 1) * iters / secs / 1e12
    info = host_info()
    return {"value": value, "unit": UNIT, "cores": workers, "kind": kind,
            "sample": f"{iters}x one {h}->{f}->{h} MLP block fwd+bwd over {sample_rows} rows (fp64, {workers} "
                      f"Concurrent-transport worker threads), {secs:.1f} s"
                      + (f"; extrapolated to the {blocks}-block stack (step time linear in FLOPs)" if blocks > 1
                         else ""),
            "extrapolated": blocks > 1 or sample_rows < (CONFIGS[cfg][3] or CONFIGS[cfg][4]),
            "rows": sample_rows, "seconds": secs, "host": info}


def run_reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    h, f, blocks, tpg, tglob, label = CONFIGS[args.config]
    per_step_target = max(1.5, 60.0 / max(1, args.steps + args.warmup))
    base = cpu_reference(args.config, target_s=per_step_target)
    rows = base["rows"]
    if args.warmup:
        cpu_reference(args.config, sample_rows=rows, iters=args.warmup)
    timed = cpu_reference(args.config, sample_rows=rows, iters=args.steps)
    value = timed["value"]
    ms = flops_per_step(rows, h, f, 1) / (value * 1e12) * 1e3
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak" if tpg else "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": label, "h": h, "f": f, "blocks": blocks, "sample_tokens": rows,
                       "tokens_per_gpu": tpg or (tglob // max(1, args.gpus)),
                       "note": "each step: one block over a bounded row sample on host cores; TFLOP/s "
                               "extrapolates to the whole stack (linear in FLOPs)"},
            "impl": "reference",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": timed["cores"], "kind": timed["kind"],
                             "sample": timed["sample"], "host": timed["host"]},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ ring self-check
def ring_self_check(rtp, grp, ring, rank, mode, world):
    """Before timing: the committed reference golden tests/golden/mlp_ring.npz
    (the reference's own RtpMlp, N in {1,2,4,8}) through THIS group's transport
    and ring size; every local rank's Y / dX rows and gradient shards within
    the bf16 tolerance (normwise 2e-2). Returns (ok, detail)."""
    import numpy as np
    import torch
    path = os.path.join(ROOT, "tests", "golden", "mlp_ring.npz")
    try:
        g = np.load(path)
    except OSError as exc:
        return None, f"fixture missing: {exc}"
    if f"n{ring}_y" not in g:
        return None, f"no golden for a ring of {ring}"
    rows = g["x"].shape[0]
    M = rows // ring
    m = rtp.RtpMlp(grp, "selfcheck", g["w1"].shape[0], g["w1"].shape[1], "bf16", w1=g["w1"], b1=g["b1"],
                   w2=g["w2"], b2=g["b2"])
    m.set_rotation_mode(mode)
    m.begin_step()
    m.zero_grads()

    def dev(a, r):
        return torch.from_numpy(np.ascontiguousarray(a[r * M:(r + 1) * M])).to(torch.bfloat16).to(
            grp.device_of(r)).contiguous()
    ranks = grp.local_ranks
    ys = m.forward([dev(g["x"], r) for r in ranks])
    dxs = m.backward([dev(g["dy"], r) for r in ranks])
    grp.synchronize()

    def nerr(a, ref):
        ref = np.asarray(ref, np.float64)
        return float(np.max(np.abs(np.asarray(a, np.float64) - ref)) / max(np.max(np.abs(ref)), 1e-300))
    worst = 0.0
    for k, r in enumerate(ranks):
        sl = slice(r * M, (r + 1) * M)
        worst = max(worst, nerr(ys[k].double().cpu().numpy(), g[f"n{ring}_y"][sl]),
                    nerr(dxs[k].double().cpu().numpy(), g[f"n{ring}_dx"][sl]),
                    nerr(m.ffn1.grad_shard(r).double().cpu().numpy(), g[f"n{ring}_grads1"][r]),
                    nerr(m.ffn2.grad_shard(r).double().cpu().numpy(), g[f"n{ring}_grads2"][r]))
        home = (m.ffn1.slot(r)["logical_id"], m.ffn2.slot(r)["logical_id"])
        if home != (r, r):
            worst = float("inf")
    m.close()
    return worst < 2e-2, f"max normwise error {worst:.3e} over Y, dX, dW1|db1, dW2|db2 (tolerance 2e-2)"


# ------------------------------------------------------------------ our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="d", choices=sorted(CONFIGS))
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mode", default="outofplace", choices=["inplace", "outofplace"])
    ap.add_argument("--blocks", type=int, default=None, help="override the config's block count")
    ap.add_argument("--tokens-per-gpu", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="skip the host-buffer e2e leg (profiling runs)")
    ap.add_argument("--no-profile", action="store_true", help="skip the profiled per-launch replay")
    ap.add_argument("--eager", action="store_true", help="time host-issued launches instead of a CUDA graph")
    ap.add_argument("--exact-gelu", action="store_true",
                    help="bf16 epilogues evaluate the exact-erf GELU (default: the tanh.approx form)")
    ap.add_argument("--no-paired-dx", action="store_true",
                    help="per-step dX sums (the reference's order; out-of-place == in-place bitwise)")
    ap.add_argument("--transport", default="nccl", choices=["nccl", "ipc"],
                    help="N > 1 ring shift: ncclSend/ncclRecv (default) or copy-engine pushes through CUDA IPC")
    ap.add_argument("--solo", type=int, default=0,
                    help="measurement: rank 0 of an N-way ring on this GPU, shifts skipped (per-GPU compute at "
                         "N-way shapes, plus the rotation bytes over NVLink as a model)")
    ap.add_argument("--same-device", action="store_true",
                    help="test mode: every rank on GPU 0 (IPC transport, gloo plumbing); numbers not meaningful")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference_arm(args)
        return
    if args.warmup < 3:
        args.warmup = 3

    import torch
    import torch.distributed as dist

    from paper_2311_01635_b200 import _lib, rtp

    H, F, BLOCKS, TPG, TGLOB, LABEL = CONFIGS[args.config]
    if args.blocks:
        BLOCKS = args.blocks
    rank, world, local = dist_env()
    if args.same_device:
        local = 0
        args.transport = "ipc"
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    graph_fallback = None
    if world > 1:
        # plumbing only (barriers, max over ranks, the id broadcast)
        if args.same_device:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
        make_uid = rtp.WorkerGroup.ipc_unique_id if args.transport == "ipc" else rtp.WorkerGroup.nccl_unique_id
        box = [make_uid() if rank == 0 else None]
        dist.broadcast_object_list(box, 0)
        make = rtp.WorkerGroup.ipc if args.transport == "ipc" else rtp.WorkerGroup.nccl
        grp = make(world, rank, local, box[0])
        if args.transport == "ipc":
            args.eager = True  # the IPC flags carry per-shift sequence numbers: no graph replay
            graph_fallback = "IPC transport: shift flags carry per-shift sequence numbers (not replayable)"
    elif args.solo > 1:
        grp = rtp.WorkerGroup.solo(args.solo, 0, local)
    else:
        grp = rtp.WorkerGroup(1)

    def allmax(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cpu" if args.same_device else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    ring = args.solo if args.solo > 1 else world  # ring size the layers are sharded for
    if args.tokens_per_gpu:
        M = args.tokens_per_gpu
    else:
        M = TPG if TPG else TGLOB // ring
    T = M * world  # tokens processed by the whole job per step
    fl_step = flops_per_step(T, H, F, BLOCKS)

    # ---- self-check through the same transport and ring size (reference golden)
    parity_ok, parity_detail = (None, "solo: no peers, shifts skipped") if args.solo > 1 else \
        ring_self_check(rtp, grp, ring, rank, args.mode, world)
    if parity_ok is not None and world > 1:
        parity_ok = allmax(0.0 if parity_ok else 1.0) == 0.0

    # ---- the model: BLOCKS Flyweight blocks, SerialModel stream order, chained
    per_block_params = 2 * H * F + F + H
    mlps = []
    for b in range(BLOCKS):
        m = rtp.RtpMlp(grp, f"block{b}", H, F, "bf16", seed=SEED, stream_base=b * per_block_params)
        m.set_rotation_mode(args.mode)
        if args.exact_gelu:
            m.set_option("exact_gelu", True)
        if args.no_paired_dx:
            m.set_option("paired_dx", False)
        m.begin_step()
        mlps.append(m)
    paired = (not args.no_paired_dx) and os.environ.get("RTPB_DX_PAIR", "1") != "0"
    numerics = {"gelu": "exact erf" if args.exact_gelu else
                "tanh form on tanh.approx.f32 in the bf16 epilogues (|d| <= 4.7e-4; --exact-gelu for exact erf)",
                "paired_dx": bool(paired and args.mode == "outofplace" and ring > 1),
                "accumulation": "fp32 (TMEM), fp32 gradient shards and cross-step dX accumulator"}
    for a, b in zip(mlps, mlps[1:]):
        a.chain(b)  # a block posts its neighbour's first weight shift under its own last step

    g = torch.Generator(device=dev).manual_seed(SEED + rank)
    x = (torch.rand(M, H, device=dev, generator=g) * 2 - 1).to(torch.bfloat16)
    dy = (torch.rand(M, H, device=dev, generator=g) * 2 - 1).to(torch.bfloat16)
    outs = [torch.empty(M, H, dtype=torch.bfloat16, device=dev) for _ in range(BLOCKS)]
    grads = [torch.empty(M, H, dtype=torch.bfloat16, device=dev) for _ in range(2)]
    dx = torch.empty(M, H, dtype=torch.bfloat16, device=dev)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # 512 MiB > 126 MB L2
    flush_sink = torch.zeros((), dtype=torch.float32, device=dev)

    def step(x_in=None, dy_in=None, dx_out=None):
        for m in mlps:
            m.zero_grads()
        inp = [x if x_in is None else x_in]
        for b, m in enumerate(mlps):
            m.forward(inp, out=[outs[b]])
            inp = [outs[b]]
        up = [dy if dy_in is None else dy_in]
        for b in range(BLOCKS - 1, -1, -1):
            o = (dx if dx_out is None else dx_out) if b == 0 else grads[b % 2]
            mlps[b].backward(up, out=[o])
            up = [o]

    t0 = time.perf_counter()
    for _ in range(args.warmup):
        step()
    barrier()
    est_ms = (time.perf_counter() - t0) * 1e3 / args.warmup

    stream = torch.cuda.current_stream(dev)
    # ---- eager timing (host-issued launches), for the record
    eager_ms = None
    if not args.eager:
        k = max(2, min(20, int(3000 / max(est_ms, 1e-3))))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        e0.record(stream)
        for _ in range(k):
            step()
        e1.record(stream)
        barrier()
        eager_ms = allmax(e0.elapsed_time(e1) / k)

    # ---- capture one step (zero_grads + forward + backward through the public
    # API, every library launch incl. PDL edges, CTA-pair clusters and the
    # NCCL shifts) into a CUDA graph. The timed graph carries no profiling
    # events (event nodes between launches break their programmatic overlap);
    # the per-launch roofline numerator comes from a second, profiled capture.
    def capture(profiled):
        _lib.lib.rtpb_profile_enable(1 if profiled else 0)
        _lib.lib.rtpb_profile_read(None, None, None, None, None, 1 << 30)  # drop older records
        l0 = rtp.launch_count()
        g_ = torch.cuda.CUDAGraph()
        cs = torch.cuda.Stream(dev)
        cs.wait_stream(stream)
        with torch.cuda.graph(g_, stream=cs):
            step()
        stream.wait_stream(cs)
        n_launch = rtp.launch_count() - l0
        for _ in range(2):
            g_.replay()
        barrier()
        return g_, n_launch

    graph = None
    graph_note = "eager (--eager)" if graph_fallback is None else f"eager ({graph_fallback})"
    _lib.lib.rtpb_profile_enable(0)
    launches_per_step = None
    if not args.eager:
        try:
            graph, launches_per_step = capture(False)
            graph_note = "CUDA graph replay of the captured step (no profiling events in the timed graph)"
        except Exception as exc:  # noqa
            graph = None
            graph_fallback = f"graph capture failed: {exc!r}"
            graph_note = f"eager ({graph_fallback})"
            _lib.lib.rtpb_profile_enable(0)
            barrier()

    # ---- timed region: exactly K steps, L2 flushed before each, CUDA events on the stream
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launches0 = rtp.launch_count()
    grp.reset_ledger_peaks()
    torch.cuda.reset_peak_memory_stats(dev)
    with ClockSampler(local) as clocks:
        barrier()
        for i in range(args.steps):
            # cold L2: write 512 MiB (> 126 MB L2), then read it back so the
            # flush's dirty lines are written back before, not inside, the step
            flush.zero_()
            flush_sink.copy_(flush.sum())
            ev[i][0].record(stream)
            if graph is not None:
                graph.replay()
            else:
                step()
            ev[i][1].record(stream)
        barrier()
    launches = (launches_per_step * args.steps) if graph is not None else rtp.launch_count() - launches0
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = allmax(sum(step_ms))
    ms_per_step = total_ms / args.steps
    value = fl_step / (ms_per_step * 1e-3) / 1e12  # whole-job aggregate over all GPUs
    burst, sustained, peak_src = load_peaks()

    # ---- profiled pass (per-launch CUDA events on each launching stream), same L2 flush
    roofline = {"bound": "tensor", "achieved": None, "peak": burst, "unit": "TFLOP/s", "frac": None,
                "traffic": None}
    if not args.no_profile:
        roofline = profiled_roofline(args, torch, _lib, rtp, dev, stream, step, capture, graph, flush, flush_sink,
                                     barrier, burst, sustained, peak_src)

    # ---- memory: device ledger (params, grads, comm, activations, workspace) + caller tensors
    led = grp.ledger(rank)
    torch_peak = torch.cuda.max_memory_allocated(dev) - flush.numel() * 4
    shard_w = sum(m.ffn1.shard_len() * 2 + m.ffn2.shard_len() * 2 for m in mlps)
    shard_g = sum(m.ffn1.shard_len() * 4 + m.ffn2.shard_len() * 4 for m in mlps)
    W_total, G_total = shard_w * ring, shard_g * ring
    pgc = led["peak_param"] + led["peak_grad"] + led["peak_comm"]
    model_in = (W_total + G_total) // ring
    model_oop = (W_total + G_total + max(W_total, G_total)) // ring
    mem = {"peak_hbm_bytes_per_gpu": led["peak_total"] + torch_peak,
           "ledger_peak": {k[5:]: v for k, v in led.items() if k.startswith("peak_")},
           "caller_activations_bytes": torch_peak,
           "model_inplace_bytes": model_in, "model_outofplace_bytes": model_oop,
           "param_grad_comm_bytes": pgc,
           "param_grad_comm_vs_model": pgc / (model_oop if (args.mode == "outofplace" and ring > 1) else model_in),
           "note": "model rows: the paper's (W+G)/N and (W+G+max(W,G))/N with bf16 W, fp32 G; out of place the "
                   "spare is one W shard per layer (G moves in place, ring.cpp:314,328), so the measured "
                   "Param+Grad+Comm sits below the W+G+max(W,G) row"}

    # ---- exposed rotation time: T(step) - T(step without moving bytes)
    exposed = {"ms_per_step": 0.0, "frac": 0.0, "method": "N=1: no rotation, nothing to expose"}
    shift = None
    if world > 1:
        def eager_step_ms(k):
            barrier()
            a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a_.record(stream)
            for _ in range(k):
                step()
            b_.record(stream)
            barrier()
            return allmax(a_.elapsed_time(b_) / k)
        k = max(2, min(10, int(2000 / max(ms_per_step, 1e-3))))
        t_with = eager_step_ms(k)
        _lib.lib.rtpb_debug_skip_comm(1)
        try:
            step()
            t_without = eager_step_ms(k)
        finally:
            _lib.lib.rtpb_debug_skip_comm(0)
        exposed = {"ms_per_step": max(0.0, t_with - t_without), "frac": max(0.0, t_with - t_without) / t_with,
                   "ms_step_eager": t_with, "ms_step_compute_only": t_without,
                   "method": "eager steps with and without rtpb_debug_skip_comm (same schedule, no bytes moved), "
                             "max over ranks"}
        shift = measure_shift(torch, grp, mlps[0], stream, barrier, allmax, args.transport)
    nvl_bw = 900e9  # NVLink 5 per direction per GPU
    w_all = sum(m.ffn1.shard_len() + m.ffn2.shard_len() for m in mlps) * ring
    sent = (ring - 1) / ring * (2 * w_all * 2 + w_all * 4) if ring > 1 else 0.0  # bf16 W fwd+bwd, fp32 G bwd
    t_gemm_peak = fl_step / world / (burst * 1e12) * 1e3
    t_nvl = sent / nvl_bw * 1e3
    step_roofline = {"gemm_ms_at_peak": t_gemm_peak, "nvlink_ms": t_nvl, "bytes_sent_per_gpu": sent,
                     "bound": "tensor" if t_gemm_peak >= t_nvl else "nvlink",
                     "roofline_ms": max(t_gemm_peak, t_nvl), "frac": max(t_gemm_peak, t_nvl) / ms_per_step,
                     "note": "north_star roofline: slower of the step's GEMM flops at the bf16 peak and its "
                             "rotation bytes over NVLink (900 GB/s/direction)"}

    # ---- e2e through the public API with host buffers (pinned), copies timed
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e_leg(torch, dev, stream, step, x, dy, dx, M, H, barrier, allmax, ms_per_step, fl_step,
                          args.steps)

    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline and not args.solo:
            try:
                cpu = cpu_reference(args.config, target_s=12.0)
            except Exception as exc:  # noqa
                cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "unavailable", "sample": repr(exc)}
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
                "scaling": "weak" if (TPG or args.tokens_per_gpu) else "strong",
                "vs_baseline": None, "dtype": "bf16",
                "data": "synthetic (uniform activations, Flyweight SplitMix64 weights, seed 42)",
                "value_scope": "whole job: TFLOP/s summed over all n_gpus (per GPU: tflops_per_gpu)",
                "config": {"workload": LABEL, "h": H, "f": F, "blocks": BLOCKS,
                           "tokens_per_gpu": M, "global_tokens": T, "rotation_mode": args.mode,
                           "parallelism": f"rtp{world}", "transport": args.transport if world > 1 else None,
                           "same_device_test": bool(args.same_device and world > 1),
                           "solo_ring": args.solo if args.solo > 1 else None,
                           "l2": "flushed before every timed step (512 MiB written, then read back)",
                           "flops_per_step": fl_step},
                "tflops_per_gpu": value / world,
                "parity_ok": parity_ok, "parity_check": parity_detail, "numerics": numerics,
                "gpu_launches": int(launches),
                "step_execution": graph_note,
                "ring_schedule": ring_schedule(ring, args.mode, H, F, M, bool(args.same_device and world > 1)),
                "eager_ms_per_step": eager_ms,
                "roofline": roofline,
                "step_roofline": step_roofline,
                "exposed_comm": exposed,
                "shift": shift,
                "memory": mem,
                "cpu_baseline": cpu,
                "e2e": e2e,
                "clocks": clocks.summary()}
        print(json.dumps(line), flush=True)
    for m in mlps:
        m.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def ring_schedule(ring, mode, h, f, rows, shared_gpu=False):
    """How the N > 1 passes are launched (rtp_layers.cpp pass_launch_ok /
    backward_pass_pays): one persistent launch per layer pass ordered by
    arrival flags, or one event-ordered launch per rotation step."""
    import os
    if ring < 2:
        return "N = 1: no rotation"
    env = os.environ.get("RTPB_FLAGS")
    flags = (env != "0") if env is not None else not shared_gpu  # the library's default (use_flags)
    passes_ok = not shared_gpu
    passes = passes_ok and flags and mode == "outofplace" and os.environ.get("RTPB_NO_PASS", "0") in ("", "0")
    out = {}
    for name, i, o in (("ffn1", h, f), ("ffn2", f, h)):
        per = o // ring
        if not passes or per % 32:
            out[name] = "one launch per rotation step (" + ("arrival flags" if flags else "stream events") + ")"
            continue
        bwd = os.environ.get("RTPB_PASS_BWD")
        # the library's rule (RtpLinear::backward_pass_pays): a step's dX under 40 GFLOP
        small = 2.0 * rows * i * per < 40e9
        both = bwd == "1" or (bwd != "0" and small)
        out[name] = "one launch per pass: forward" + (", dX and dW side by side" if both else
                                                      "; backward one launch per step")
    return out


def profiled_roofline(args, torch, _lib, rtp, dev, stream, step, capture, graph, flush, flush_sink, barrier,
                      burst, sustained, peak_src):
    """Per-launch GEMM timing from a separately profiled replay: algorithmic
    FLOPs per launch (2*M*I*per per product) over each launch's CUDA-event
    duration x its share of the SMs."""
    import ctypes as C
    prof_graph = None
    if graph is not None:
        try:
            prof_graph, _ = capture(True)
        except Exception:  # noqa
            prof_graph = None
    if prof_graph is None:
        _lib.lib.rtpb_profile_enable(1)
        _lib.lib.rtpb_profile_read(None, None, None, None, None, 1 << 30)
    prof_steps = 3
    pev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    for i in range(prof_steps):
        flush.zero_()
        flush_sink.copy_(flush.sum())
        if i == prof_steps - 1:
            pev[0].record(stream)
        if prof_graph is not None:
            prof_graph.replay()
        else:
            step()
        if i == prof_steps - 1:
            pev[1].record(stream)
    barrier()
    prof_step_ms = pev[0].elapsed_time(pev[1])
    _lib.lib.rtpb_profile_enable(0)
    cnt = _lib.lib.rtpb_profile_read(None, None, None, None, None, 0)
    kinds = (C.c_int * cnt)()
    fl = (C.c_double * cnt)()
    ms = (C.c_float * cnt)()
    st = (C.c_float * cnt)()
    smc = (C.c_int * cnt)()
    _lib.lib.rtpb_profile_read(kinds, fl, ms, st, smc, cnt)
    per_step = cnt if prof_graph is not None else max(1, cnt // prof_steps)
    recs = list(zip(kinds, fl, ms, st, smc))[cnt - per_step:]
    t_first = min(r[3] for r in recs) if recs else 0.0
    names = {0: "fwd", 1: "dgrad", 2: "wgrad"}
    all_sms = torch.cuda.get_device_properties(dev).multi_processor_count
    per_launch = [{"kind": names[k], "us": round(m_ * 1e3, 2), "start_us": round((t0 - t_first) * 1e3, 2),
                   "sms": int(sm_), "tflops": round(f_ / (m_ * 1e-3) / 1e12, 1) if m_ else None}
                  for k, f_, m_, t0, sm_ in recs]
    per_kind = {}
    for k, f_, m_, t0, sm_ in recs:
        d = per_kind.setdefault(names[k], [0.0, 0.0, 0, 0.0])
        d[0] += f_
        d[1] += m_
        d[2] += 1
        d[3] += m_ * sm_ / all_sms  # GPU-time: duration x share of the SMs the launch was sized for
    gemm_flops = sum(d[0] for d in per_kind.values())
    gemm_gpu_ms = sum(d[3] for d in per_kind.values())
    iv = sorted((t0, t0 + m_) for _, _, m_, t0, _ in recs)
    busy, cur_a, cur_b = 0.0, None, None
    for a_, b_ in iv:
        if cur_b is None or a_ > cur_b:
            if cur_b is not None:
                busy += cur_b - cur_a
            cur_a, cur_b = a_, b_
        else:
            cur_b = max(cur_b, b_)
    if cur_b is not None:
        busy += cur_b - cur_a
    achieved = gemm_flops / (gemm_gpu_ms * 1e-3) / 1e12 if gemm_gpu_ms else 0.0
    traffic, traffic_src = None, None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            tj = json.load(fh)
        entry = tj.get("configs", {}).get(args.config)
        if entry:
            traffic, traffic_src = entry.get("dram_bytes_per_launch"), entry.get("source")
    except Exception:
        pass
    if len(per_launch) > 24:  # keep the line readable: first block's launches + the last
        shown = per_launch[:6] + per_launch[-3:]
    else:
        shown = per_launch
    return {"bound": "tensor", "achieved": achieved, "peak": burst, "unit": "TFLOP/s",
            "frac": achieved / burst, "traffic": traffic, "traffic_source": traffic_src,
            "kernel": "rtp_gemm_kernel (tcgen05 step GEMMs: fwd, dgrad, wgrad)",
            "peak_source": f"{peak_src} bf16 burst; sustained {sustained}",
            "frac_of_sustained": achieved / sustained,
            "achieved_over_gemm_wall": gemm_flops / (busy * 1e-3) / 1e12 if busy else None,
            "gemm_busy_share_of_step": busy / prof_step_ms if prof_step_ms else None,
            "profiled_step_ms": prof_step_ms, "launches_per_step": len(per_launch),
            "note": "per-launch numbers from a separately captured, profiled replay of the step (event "
                    "nodes between launches break programmatic overlap, so the timed graph has none)",
            "per_kernel": {k: {"tflops_per_gpu_time": v[0] / (v[3] * 1e-3) / 1e12, "launches": v[2],
                               "avg_us": v[1] / v[2] * 1e3} for k, v in per_kind.items()},
            "per_launch_in_step_order": shown}


def measure_shift(torch, grp, mlp, stream, barrier, allmax, transport):
    """One ring shift of the model's largest weight shard (out of place, into a
    spare) and one counter-clockwise W+G shift, timed with CUDA events on the
    caller's stream (the library orders its comm stream inside it), max over
    ranks: NVLink GB/s sent per GPU against 900 GB/s per direction."""
    ranks = grp.local_ranks
    dev = grp.device_of(ranks[0])
    L = mlp.ffn1.shard_len()
    W = [torch.empty(L, dtype=torch.bfloat16, device=dev).normal_() for _ in ranks]
    SP = [torch.empty_like(w) for w in W]
    G = [torch.zeros(L, dtype=torch.float32, device=dev) for _ in ranks]
    out = {"transport": transport, "shard_bytes": L * 2}
    for name, kw, nbytes in (("cw_w_outofplace", dict(spares=SP, keep_spare=True), L * 2),
                             ("ccw_wg_outofplace", dict(grads=G, spares=SP, keep_spare=True), L * 6)):
        op = "cw" if name.startswith("cw") else "ccw"
        grp.rotate(op, W, **kw)
        barrier()
        iters = 10
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(iters):
            grp.rotate(op, W, **kw)
        b.record(stream)
        barrier()
        ms = allmax(a.elapsed_time(b) / iters)
        out[name] = {"ms": ms, "bytes_sent_per_gpu": nbytes, "gbs": nbytes / (ms * 1e-3) / 1e9,
                     "frac_of_nvlink_900": nbytes / (ms * 1e-3) / 900e9}
    return out


def run_e2e_leg(torch, dev, stream, step, x, dy, dx, M, H, barrier, allmax, ms_per_step, fl_step, steps):
    """The same step through RtpMlp.forward/backward from pinned host X / dY
    with dX read back, copies inside the timed region. Training-loop shape:
    step i+1's inputs are copied host->device on copy streams while step i
    computes, and step i's dX goes device->host on another while step i+1
    computes (double-buffered)."""
    hx = [x.cpu().pin_memory() for _ in range(2)]
    hdy = [dy.cpu().pin_memory() for _ in range(2)]
    hdx = [torch.empty(M, H, dtype=torch.bfloat16).pin_memory() for _ in range(2)]
    xd = [torch.empty_like(x) for _ in range(2)]
    dyd = [torch.empty_like(dy) for _ in range(2)]
    dxd = [torch.empty_like(dx) for _ in range(2)]
    h2d, h2d_b, d2h = torch.cuda.Stream(dev), torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    EV = lambda: torch.cuda.Event()  # noqa: E731
    e2e_steps = max(5, min(steps, 100, int(4000 / max(ms_per_step, 1e-3))))

    def run(nsteps):
        landed, landed_b = [EV(), EV()], [EV(), EV()]
        computed, drained = [EV(), EV()], [EV(), EV()]
        done_with_inputs = [None, None]

        def issue_h2d(i):
            b = i % 2
            with torch.cuda.stream(h2d):
                if done_with_inputs[b] is not None:
                    h2d.wait_event(done_with_inputs[b])  # step i-2 finished reading these buffers
                xd[b].copy_(hx[b], non_blocking=True)
                landed[b].record(h2d)
            with torch.cuda.stream(h2d_b):
                if done_with_inputs[b] is not None:
                    h2d_b.wait_event(done_with_inputs[b])
                dyd[b].copy_(hdy[b], non_blocking=True)
                landed_b[b].record(h2d_b)

        h2d.wait_stream(stream)
        h2d_b.wait_stream(stream)
        d2h.wait_stream(stream)
        issue_h2d(0)
        for i in range(nsteps):
            b = i % 2
            if i + 1 < nsteps:
                issue_h2d(i + 1)
            stream.wait_event(landed[b])
            stream.wait_event(landed_b[b])
            if i >= 2:
                stream.wait_event(drained[b])  # dxd[b] read back before it is overwritten
            step(xd[b], dyd[b], dxd[b])
            computed[b].record(stream)
            done_with_inputs[b] = computed[b]
            with torch.cuda.stream(d2h):
                d2h.wait_event(computed[b])
                hdx[b].copy_(dxd[b], non_blocking=True)
                drained[b].record(d2h)
        stream.wait_stream(d2h)
        stream.wait_stream(h2d)
        stream.wait_stream(h2d_b)

    run(2)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    run(e2e_steps)
    e1.record(stream)
    barrier()
    e2e_ms = allmax(e0.elapsed_time(e1) / e2e_steps)
    return {"value": fl_step / (e2e_ms * 1e-3) / 1e12, "unit": UNIT,
            "h2d_bytes_per_step": 2 * M * H * 2, "d2h_bytes_per_step": M * H * 2, "ms_per_step": e2e_ms,
            "steps": e2e_steps,
            "path": "RtpMlp.forward/backward over every block (C ABI, eager launches) from pinned host X, dY; "
                    "dX read back; step i+1 H2D and step i-1 D2H overlap step i on copy streams"}


if __name__ == "__main__":
    main()
