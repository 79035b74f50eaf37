"""RTP MLP fwd+bwd benchmark (BASELINE.json metric: "RTP MLP fwd+bwd TFLOP/s/GPU
& peak HBM/GPU at 1/2/4/8 B200 vs CPU ref").

Workload (config (b) of BASELINE.json, the metric's single-GPU config): one
RTP MLP block ffn1 768->3072 -> GELU -> ffn2 3072->768, bf16, Flyweight init
(SplitMix64 seed 42), 8192 tokens per GPU (GPT-2 seq 512 x 16, SURVEY §8d;
global T = 8192 x N, batch-major row shards: weak scaling). A step = zero
grads + forward + backward of the block through the library's public API.
FLOPs per step = 12 * T * h * f (fwd, dX, dW at 2*T*h*f per linear).

python bench.py [--gpus N --steps K --warmup W] [--impl reference]
N > 1: launch with torch.distributed.run, one process per GPU, NCCL ring.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

H, F, TOKENS_PER_GPU, SEED = 768, 3072, 8192, 42
METRIC = "RTP MLP fwd+bwd TFLOP/s/GPU & peak HBM/GPU at 1/2/4/8 B200 vs CPU ref"
UNIT = "TFLOP/s"


def flops_per_step(tokens: int) -> float:
    return 12.0 * tokens * H * F


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["bf16_tflops"]), float(p.get("bf16_tflops_sustained", p["bf16_tflops"])), "measured"
    except Exception:
        return 1590.0, 1400.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.samples = []
        self._stop = threading.Event()
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
def cpu_reference(sample_rows: int | None = None, target_s: float = 12.0, iters: int = 1):
    """Times the reference's own CPU implementation of the path (oracle/_ref:
    the reference sources compiled by path; RtpLinear x2 + gelu on the
    Concurrent transport, one worker thread per host core, fp64) on a bounded
    row sample of the same workload. Falls back to the C restatement."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as orc
    cores = os.cpu_count() or 1
    workers = 1
    while workers * 2 <= cores and (F % (workers * 2) == 0) and (H % (workers * 2) == 0):
        workers *= 2
    try:
        R = orc.Reference()
        kind = "reference"

        def run(rows):
            return R.time_mlp(workers, rows, H, F, SEED, iters=1, concurrent=True)
    except Exception:
        O = orc.Oracle()
        kind = "port"
        import numpy as np
        rng = np.random.default_rng(SEED)
        w1, b1 = rng.uniform(-0.1, 0.1, (H, F)), rng.uniform(-0.1, 0.1, F)
        w2, b2 = rng.uniform(-0.1, 0.1, (F, H)), rng.uniform(-0.1, 0.1, H)

        def run(rows):
            x, dy = rng.uniform(-1, 1, (rows, H)), rng.uniform(-1, 1, (rows, H))
            t0 = time.perf_counter()
            O.rtp_mlp(workers, w1, b1, w2, b2, x, dy)
            return time.perf_counter() - t0
    if sample_rows is None:
        probe = 32 * workers
        t = run(probe)
        rate = flops_per_step(probe) / max(t, 1e-6)
        sample_rows = int(target_s * rate / flops_per_step(1))
        sample_rows = max(workers, min(TOKENS_PER_GPU, (sample_rows // workers) * workers))
    secs = sum(run(sample_rows) for _ in range(iters))
    value = flops_per_step(sample_rows) * iters / secs / 1e12
    return {"value": value, "unit": UNIT, "cores": workers, "kind": kind,
            "sample": f"{iters}x MLP fwd+bwd over {sample_rows} of {TOKENS_PER_GPU} tokens (768->3072->768, fp64, "
                      f"{workers} Concurrent-transport workers), {secs:.1f} s"}


def run_reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    steps = []
    # bounded sample per step so --steps K --warmup W ends within minutes
    per_step_target = max(2.0, 60.0 / max(1, args.steps + args.warmup))
    base = cpu_reference(target_s=per_step_target)
    rows = int(base["sample"].split(" over ")[1].split(" ")[0])
    for _ in range(args.warmup):
        cpu_reference(sample_rows=rows)
    for _ in range(args.steps):
        steps.append(cpu_reference(sample_rows=rows))
    value = sum(s["value"] for s in steps) / len(steps)
    ms = flops_per_step(rows) / (value * 1e12) * 1e3
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "rtp_mlp_768x3072x768", "tokens": rows, "tokens_per_gpu": TOKENS_PER_GPU,
                       "note": "bounded row sample of the same workload on host cores"},
            "impl": "reference",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": steps[0]["cores"], "kind": steps[0]["kind"],
                             "sample": steps[0]["sample"]},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mode", default="outofplace", choices=["inplace", "outofplace"])
    ap.add_argument("--tokens-per-gpu", type=int, default=TOKENS_PER_GPU)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--eager", action="store_true", help="time host-issued launches instead of a CUDA graph")
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

    rank, world, local = dist_env()
    if args.same_device:
        local = 0
        args.transport = "ipc"
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
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
    M = args.tokens_per_gpu
    T = M * world
    ring = args.solo if args.solo > 1 else world  # ring size the layers are sharded for
    mlp = rtp.RtpMlp(grp, "block0", H, F, "bf16", seed=SEED, stream_base=0)  # Flyweight init on device
    mlp.set_rotation_mode(args.mode)
    mlp.begin_step()

    g = torch.Generator(device=dev).manual_seed(SEED + rank)
    x = (torch.rand(M, H, device=dev, generator=g) * 2 - 1).to(torch.bfloat16)
    dy = (torch.rand(M, H, device=dev, generator=g) * 2 - 1).to(torch.bfloat16)
    y = torch.empty(M, H, dtype=torch.bfloat16, device=dev)
    dx = torch.empty(M, H, dtype=torch.bfloat16, device=dev)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # 512 MiB > 126 MB L2
    flush_sink = torch.zeros((), dtype=torch.float32, device=dev)

    def step():
        mlp.zero_grads()
        mlp.forward([x], out=[y])
        mlp.backward([dy], out=[dx])

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    barrier()

    stream = torch.cuda.current_stream(dev)
    # ---- eager reference timing (host-issued launches), for the record
    eager_ms = None
    if not args.eager:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        e0.record(stream)
        for _ in range(20):
            step()
        e1.record(stream)
        barrier()
        eager_ms = e0.elapsed_time(e1) / 20

    # ---- capture one step (zero_grads + forward + backward through the public
    # API, every library launch incl. PDL edges and CTA-pair clusters) into a
    # CUDA graph. The timed graph carries no profiling events (event nodes
    # between launches break their programmatic overlap: measured 16 us per
    # config (b) step); the per-launch roofline numerator comes from a second,
    # profiled capture replayed after the timed region.
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
        for _ in range(3):
            g_.replay()
        barrier()
        return g_, n_launch

    graph = None
    graph_note = "eager (--eager)"
    _lib.lib.rtpb_profile_enable(0)
    launches_per_step = None
    if not args.eager:
        try:
            graph, launches_per_step = capture(False)
            graph_note = "CUDA graph replay of the captured step (no profiling events in the timed graph)"
        except Exception as exc:  # noqa
            graph = None
            graph_note = f"eager (graph capture failed: {exc!r})"
            _lib.lib.rtpb_profile_enable(0)

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

    # ---- profiled pass (per-launch CUDA events on each launching stream), same L2 flush
    prof_graph = None
    if graph is not None:
        try:
            prof_graph, _ = capture(True)
        except Exception:  # noqa
            prof_graph = None
    if prof_graph is None:
        _lib.lib.rtpb_profile_enable(1)
        _lib.lib.rtpb_profile_read(None, None, None, None, None, 1 << 30)
    prof_steps = 5
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
    total_ms = sum(step_ms)
    total_ms = allmax(total_ms)
    ms_per_step = total_ms / args.steps
    value = flops_per_step(T) / (ms_per_step * 1e-3) / 1e12  # whole-job aggregate

    # ---- per-launch GEMM timing (the roofline numerator), last timed step
    import ctypes as C
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
    # wall time with at least one step GEMM running (union of launch intervals)
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
    burst, sustained, peak_src = load_peaks()
    # achieved: algorithmic flops per unit of GPU time the GEMM launches held
    # (duration x their share of the SMs: two GEMMs side by side on halves of
    # the machine are each compared with half the peak)
    achieved = gemm_flops / (gemm_gpu_ms * 1e-3) / 1e12 if gemm_gpu_ms else 0.0
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            traffic = json.load(fh).get("dram_bytes_per_launch")
    except Exception:
        pass
    roofline = {"bound": "tensor", "achieved": achieved, "peak": burst, "unit": "TFLOP/s",
                "frac": achieved / burst, "traffic": traffic,
                "kernel": "rtp_gemm_kernel (tcgen05 step GEMMs: fwd, dgrad, wgrad)",
                "peak_source": f"{peak_src} bf16 burst; sustained {sustained}",
                "frac_of_sustained": achieved / sustained,
                "achieved_over_gemm_wall": gemm_flops / (busy * 1e-3) / 1e12 if busy else None,
                "gemm_busy_share_of_step": busy / prof_step_ms if prof_step_ms else None,
                "profiled_step_ms": prof_step_ms,
                "note": "per-launch numbers from a separately captured, profiled replay of the step (event "
                        "nodes between launches cost ~16 us per step, so the timed graph has none)",
                "per_kernel": {k: {"tflops_per_gpu_time": v[0] / (v[3] * 1e-3) / 1e12, "launches": v[2],
                                   "avg_us": v[1] / v[2] * 1e3} for k, v in per_kind.items()},
                "per_launch_in_step_order": per_launch}

    # ---- memory: device ledger (params, grads, comm, activations, workspace) + caller tensors
    led = grp.ledger(rank)
    torch_peak = torch.cuda.max_memory_allocated(dev) - flush.numel() * 4
    shard_w = mlp.ffn1.shard_len() * 2 + mlp.ffn2.shard_len() * 2
    shard_g = mlp.ffn1.shard_len() * 4 + mlp.ffn2.shard_len() * 4
    W_total, G_total = shard_w * ring, shard_g * ring
    mem = {"peak_hbm_bytes_per_gpu": led["peak_total"] + torch_peak,
           "ledger_peak": {k[5:]: v for k, v in led.items() if k.startswith("peak_")},
           "caller_activations_bytes": torch_peak,
           "model_inplace_bytes": (W_total + G_total) // ring,
           "model_outofplace_bytes": (W_total + G_total + max(W_total, G_total)) // ring,
           "param_grad_comm_bytes": led["peak_param"] + led["peak_grad"] + led["peak_comm"]}

    # ---- exposed rotation time: T(step) - T(step without moving bytes)
    exposed = {"ms_per_step": 0.0, "frac": 0.0, "method": "N=1: no rotation, nothing to expose"}
    if world > 1:
        def eager_step_ms(k=10):
            barrier()
            a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a_.record(stream)
            for _ in range(k):
                step()
            b_.record(stream)
            barrier()
            return allmax(a_.elapsed_time(b_) / k)
        t_with = eager_step_ms()
        _lib.lib.rtpb_debug_skip_comm(1)
        try:
            step()
            t_without = eager_step_ms()
        finally:
            _lib.lib.rtpb_debug_skip_comm(0)
        exposed = {"ms_per_step": max(0.0, t_with - t_without), "frac": max(0.0, t_with - t_without) / t_with,
                   "ms_step_eager": t_with, "ms_step_compute_only": t_without,
                   "method": "eager steps with and without rtpb_debug_skip_comm (same schedule, no bytes moved), "
                             "max over ranks"}
    nvl_bw = 900e9  # NVLink 5 per direction per GPU
    w_all = (mlp.ffn1.shard_len() + mlp.ffn2.shard_len()) * ring
    sent = (ring - 1) / ring * (2 * w_all * 2 + w_all * 4) if ring > 1 else 0.0  # bf16 W fwd+bwd, fp32 G bwd
    t_gemm_peak = flops_per_step(T) / world / (burst * 1e12) * 1e3
    t_nvl = sent / nvl_bw * 1e3
    step_roofline = {"gemm_ms_at_peak": t_gemm_peak, "nvlink_ms": t_nvl, "bytes_sent_per_gpu": sent,
                     "bound": "tensor" if t_gemm_peak >= t_nvl else "nvlink",
                     "roofline_ms": max(t_gemm_peak, t_nvl), "frac": max(t_gemm_peak, t_nvl) / ms_per_step,
                     "note": "north_star roofline: slower of the step's GEMM flops at the bf16 peak and its "
                             "rotation bytes over NVLink (900 GB/s/direction)"}

    # ---- e2e through the public API with host buffers (pinned), copies timed
    e2e = None
    if rank == 0 or world > 1:
        # Training-loop shape: step i+1's inputs are copied host->device on a
        # copy stream while step i computes, and step i's dX goes device->host
        # on another while step i+1 computes (double-buffered). Every step's
        # H2D and D2H happen inside the timed region.
        hx = [x.cpu().pin_memory() for _ in range(2)]
        hdy = [dy.cpu().pin_memory() for _ in range(2)]
        hdx = [torch.empty(M, H, dtype=torch.bfloat16).pin_memory() for _ in range(2)]
        xd = [torch.empty_like(x) for _ in range(2)]
        dyd = [torch.empty_like(dy) for _ in range(2)]
        dxd = [torch.empty_like(dx) for _ in range(2)]
        # X and dY travel on two H2D streams (two copy engines in flight)
        h2d, h2d_b, d2h = torch.cuda.Stream(dev), torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        EV = lambda: torch.cuda.Event()  # noqa: E731
        e2e_steps = max(10, min(args.steps, 100))

        def run_e2e(nsteps):
            landed = [EV(), EV()]
            computed = [EV(), EV()]
            drained = [EV(), EV()]
            done_with_inputs = [None, None]

            landed_b = [EV(), EV()]

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
                mlp.zero_grads()
                mlp.forward([xd[b]], out=[y])
                mlp.backward([dyd[b]], out=[dxd[b]])
                computed[b].record(stream)
                done_with_inputs[b] = computed[b]
                with torch.cuda.stream(d2h):
                    d2h.wait_event(computed[b])
                    hdx[b].copy_(dxd[b], non_blocking=True)
                    drained[b].record(d2h)
            stream.wait_stream(d2h)
            stream.wait_stream(h2d)
            stream.wait_stream(h2d_b)

        run_e2e(4)
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        run_e2e(e2e_steps)
        e1.record(stream)
        barrier()
        e2e_ms = e0.elapsed_time(e1) / e2e_steps
        e2e_ms = allmax(e2e_ms)
        e2e = {"value": flops_per_step(T) / (e2e_ms * 1e-3) / 1e12, "unit": UNIT,
               "h2d_bytes_per_step": 2 * M * H * 2, "d2h_bytes_per_step": M * H * 2, "ms_per_step": e2e_ms,
               "path": "RtpMlp.forward/backward (C ABI, eager launches) from pinned host X, dY; dX read "
                       "back; step i+1 H2D and step i-1 D2H overlap step i on copy streams"}

    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline and not args.solo:
            try:
                cpu = cpu_reference(target_s=12.0)
            except Exception as exc:  # noqa
                cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "unavailable", "sample": repr(exc)}
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "bf16", "data": "synthetic (uniform activations, Flyweight "
                                                             "SplitMix64 weights, seed 42)",
                "config": {"workload": "rtp_mlp_768x3072x768 (config b)", "h": H, "f": F,
                           "tokens_per_gpu": M, "global_tokens": T, "rotation_mode": args.mode,
                           "parallelism": f"rtp{world}", "transport": args.transport if world > 1 else None,
                           "same_device_test": bool(args.same_device and world > 1),
                           "solo_ring": args.solo if args.solo > 1 else None, "l2": "flushed before every timed step (512 MiB written, then read back)",
                           "flops_per_step": flops_per_step(T)},
                "tflops_per_gpu": value / world,
                "gpu_launches": int(launches),
                "step_execution": graph_note,
                "eager_ms_per_step": eager_ms,
                "roofline": roofline,
                "step_roofline": step_roofline,
                "exposed_comm": exposed,
                "memory": mem,
                "cpu_baseline": cpu,
                "e2e": e2e,
                "clocks": clocks.summary()}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
