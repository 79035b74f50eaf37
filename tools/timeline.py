"""Dev probe (not a test): per-CTA timeline of the step GEMMs in one RTP MLP
fwd+bwd (config (b), N=1, L2 flushed first), from the %globaltimer stamps the
kernel writes when rtpb_debug_trace is set (layout: gemm_sm100.cuh GemmArgs::trace).

python tools/timeline.py [tokens h f]
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2311_01635_b200 import _lib, rtp  # noqa: E402

STRIDE, UNITS = 80, 12
M = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
H = int(sys.argv[2]) if len(sys.argv) > 2 else 768
F = int(sys.argv[3]) if len(sys.argv) > 3 else 3072
import os
NAMES = (["fwd1", "fwd2"] if os.environ.get("RTPB_NO_FUSED_FWD") else ["fwd1+fwd2"]) + \
    (["dgrad2", "wgrad2", "dgrad1", "wgrad1"] if os.environ.get("RTPB_NO_FUSED_BWD") else ["dgrad2+dgrad1", "wgrad2+wgrad1"])

dev = torch.device("cuda", 0)
SOLO = int(os.environ.get("SOLO", "0"))  # rank 0 of an N-way ring, shifts skipped (per-GPU schedule)
grp = rtp.WorkerGroup.solo(SOLO, 0, 0) if SOLO else rtp.WorkerGroup(1)
if SOLO:
    NAMES = [f"L{i}" for i in range(64)]
mlp = rtp.RtpMlp(grp, "tl", H, F, "bf16", seed=42, stream_base=0)
mlp.set_rotation_mode("outofplace")
mlp.begin_step()
x = (torch.rand(M, H, device=dev) * 2 - 1).to(torch.bfloat16)
dy = (torch.rand(M, H, device=dev) * 2 - 1).to(torch.bfloat16)
y = torch.empty_like(x)
dx = torch.empty_like(x)
flush = torch.empty(512 * 1024 * 1024 // 4, device=dev)


def step():
    mlp.zero_grads()
    mlp.forward([x], out=[y])
    mlp.backward([dy], out=[dx])


for _ in range(5):
    step()
torch.cuda.synchronize()
buf = torch.zeros((64 if SOLO else 6) * 148 * STRIDE + 1024, dtype=torch.int64, device=dev)
if os.environ.get("GRAPH"):
    # GRAPH=1: the step captured in a CUDA graph (as bench.py times it); the
    # trace pointers are baked into the captured launches
    cs = torch.cuda.Stream(dev)
    cs.wait_stream(torch.cuda.current_stream(dev))
    gph = torch.cuda.CUDAGraph()
    _lib.lib.rtpb_debug_trace(buf.data_ptr(), buf.numel() * 8)
    with torch.cuda.graph(gph, stream=cs):
        step()
    _lib.lib.rtpb_debug_trace(None, 0)
    for rep in range(3):
        buf.zero_()
        flush.zero_()
        flush.sum().item()
        gph.replay()
        torch.cuda.synchronize()
else:
    for rep in range(3):
        buf.zero_()
        flush.zero_()
        flush.sum().item()
        _lib.lib.rtpb_debug_trace(buf.data_ptr(), buf.numel() * 8)
        step()
        torch.cuda.synchronize()
        _lib.lib.rtpb_debug_trace(None, 0)
tr = buf.cpu().numpy().astype(np.float64)
# locate launches: consecutive blocks, grid unknown -> infer from nonzero entries
t_origin = None
off = 0
print(f"M={M} h={H} f={F}: times in us relative to the first kernel's first CTA entry")
for li, name in enumerate(NAMES):
    # grid: count CTAs with nonzero entry stamp, scanning blocks of STRIDE
    if off + STRIDE > tr.size or tr[off] == 0:
        break
    g = int(tr[off + STRIDE - 1])
    blk = tr[off:off + g * STRIDE].reshape(g, STRIDE)
    off += g * STRIDE
    if t_origin is None:
        t_origin = blk[:, 0].min()
    rel = lambda v: (v - t_origin) / 1e3  # noqa: E731
    entry, gdw = blk[:, 0], blk[:, 1]
    u = blk[:, 2:2 + 6 * UNITS].reshape(g, UNITS, 6)
    mma_lead = u[:, :, 2] > 0
    epi = u[:, :, 4] > 0
    last_epi = np.where(epi, u[:, :, 5], 0).max()
    first_mma = np.where(mma_lead, u[:, :, 2], np.inf).min()
    ml = (u[:, :, 3] - u[:, :, 2])[mma_lead]          # first stage -> last commit issued
    accw = (u[:, :, 1] - u[:, :, 0])[mma_lead]        # wait for a free accumulator
    ep = (u[:, :, 5] - u[:, :, 4])[epi]               # epilogue per unit
    lat = []
    for c in range(g):
        for i in range(UNITS):
            if mma_lead[c, i] and epi[c, i]:
                lat.append(u[c, i, 4] - u[c, i, 3])
    units_per_cta = epi.sum(1)
    if os.environ.get("UNITS") and str(li) in os.environ.get("UNITS").split(","):
        for c in range(0, g, 2):
            print("   cta", c, " ".join(f"[{rel(u[c, i, 2]):.1f}>{rel(u[c, i, 4]):.1f}:{rel(u[c, i, 5]):.1f}]"
                                      for i in range(UNITS) if u[c, i, 2] > 0))
    print(f"{name:7s} grid {g:3d} entry {rel(entry.min()):7.1f}..{rel(entry.max()):7.1f}  griddep_wait done "
          f"{rel(gdw.min()):7.1f}..{rel(gdw.max()):7.1f}  first stage {rel(first_mma):7.1f}  last epi done "
          f"{rel(last_epi):7.1f}  span {(last_epi - entry.min()) / 1e3:6.1f}")
    print(f"        units/CTA {units_per_cta.min()}..{units_per_cta.max()}  mainloop issue {ml.mean() / 1e3:5.2f} "
          f"(min {ml.min() / 1e3:5.2f} max {ml.max() / 1e3:5.2f})  acc wait {accw.mean() / 1e3:5.2f} "
          f"(max {accw.max() / 1e3:5.2f})  epilogue {ep.mean() / 1e3:5.2f} (max {ep.max() / 1e3:5.2f})  "
          f"commit->epi {np.mean(lat) / 1e3 if lat else 0:5.2f}")
    # per-unit epilogue end times of the last units (tail)
    ends = np.sort(np.where(epi, u[:, :, 5], 0).max(1))
    print(f"        CTA finish spread: p10 {rel(np.percentile(ends, 10)):7.1f} p50 {rel(np.percentile(ends, 50)):7.1f} "
          f"p90 {rel(np.percentile(ends, 90)):7.1f} max {rel(ends.max()):7.1f}")
