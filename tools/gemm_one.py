"""Dev probe (not a test): launch each step GEMM kind a few times at one shape,
for ncu captures (-k regex:rtp_gemm -s 3 -c 3) and quick timing.

python tools/gemm_one.py M I per [kinds=fwd,dgrad,wgrad] [tile code]
"""
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2311_01635_b200 import _lib, rtp  # noqa: E402

M, I, per = (int(v) for v in sys.argv[1:4])
kinds = sys.argv[4].split(",") if len(sys.argv) > 4 else ["fwd", "dgrad", "wgrad"]
code = int(sys.argv[5]) if len(sys.argv) > 5 else 0
_lib.lib.rtpb_debug_force_bn(code)
dev = "cuda"
X = torch.randn(M, I, device=dev).to(torch.bfloat16)
sh = (torch.randn(I * per + per, device=dev) * 0.01).to(torch.bfloat16)
Y = torch.empty(M, per, dtype=torch.bfloat16, device=dev)
dY = torch.randn(M, per, device=dev).to(torch.bfloat16)
dX = torch.empty(M, I, dtype=torch.bfloat16, device=dev)
G = torch.zeros(I * per + per, dtype=torch.float32, device=dev)
Hh = torch.empty(M, per, dtype=torch.bfloat16, device=dev)
pre = torch.randn(M, I, device=dev).to(torch.bfloat16)
fns = {"fwd": lambda: rtp.fwd_step(X, sh, Y, 0, per),
       "fwd_gelu": lambda: rtp.fwd_step(X, sh, Y, 0, per, act=Hh),
       "fwd_actonly": lambda: rtp.fwd_step(X, sh, None, 0, per, act=Hh, store_pre=False),
       "dgrad_gelu": lambda: rtp.dgrad_step(dY, 0, sh, None, dX, M, I, per, True, True, pre=pre),
       "dgrad": lambda: rtp.dgrad_step(dY, 0, sh, None, dX, M, I, per, True, True),
       "wgrad": lambda: rtp.wgrad_step(X, dY, 0, G, G, per)}
if any(k.startswith("dgrad_") and k != "dgrad_gelu" for k in kinds):  # cross-step fp32 accumulator kinds
    ACC = torch.zeros(M, I, dtype=torch.float32, device=dev)
    fns["dgrad_first"] = lambda: rtp.dgrad_step(dY, 0, sh, ACC, dX, M, I, per, True, False)
    fns["dgrad_mid"] = lambda: rtp.dgrad_step(dY, 0, sh, ACC, dX, M, I, per, False, False)
    fns["dgrad_last"] = lambda: rtp.dgrad_step(dY, 0, sh, ACC, dX, M, I, per, False, True)
    fns["dgrad_last_gelu"] = lambda: rtp.dgrad_step(dY, 0, sh, ACC, dX, M, I, per, False, True, pre=pre)
if "wgrad_as_dgrad" in kinds:  # the dW product on the dgrad kernel: X^T (I x M) . (dY^T (per x M))^T
    XT2 = X.t().contiguous()
    WT = torch.empty(per * M + M, dtype=torch.bfloat16, device=dev)
    WT[:per * M].view(per, M).copy_(dY.t())
    OUT = torch.empty(I, per, dtype=torch.bfloat16, device=dev)
    fns["wgrad_as_dgrad"] = lambda: rtp.dgrad_step(XT2, 0, WT, None, OUT, I, per, M, True, True)
if "wgrad_as_fwd" in kinds:  # the dW product on the forward kernel: A = X^T K-major, B = dY MN-major
    XT1 = X.t().contiguous()
    DYS = torch.zeros(M * per + per, dtype=torch.bfloat16, device=dev)
    DYS[:M * per].view(M, per).copy_(dY)
    OUTF = torch.empty(I, per, dtype=torch.bfloat16, device=dev)
    fns["wgrad_as_fwd"] = lambda: rtp.fwd_step(XT1, DYS, OUTF, 0, per)
fl = 2.0 * M * I * per
for k in kinds:
    f = fns[k]
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        f()
    b.record()
    torch.cuda.synchronize()
    us = a.elapsed_time(b) / 10 * 1e3
    hbm = {"dgrad_first": 4, "dgrad_mid": 8, "dgrad_last": 6, "dgrad_last_gelu": 8}.get(k, 0) * M * I
    extra = f" {hbm / us / 1e3:6.0f} GB/s acc traffic" if hbm else ""
    print(f"{k:6s} M={M} I={I} per={per} tile={code}: {us:8.1f} us {fl / us / 1e6:6.0f} TF/s{extra}", flush=True)

if os.environ.get("TRACE"):
    import numpy as np
    STRIDE, UNITS = 80, 12
    for k in kinds:
        buf = torch.zeros(148 * STRIDE + 64, dtype=torch.int64, device=dev)
        torch.cuda.synchronize()
        _lib.lib.rtpb_debug_trace(buf.data_ptr(), buf.numel() * 8)
        fns[k]()
        torch.cuda.synchronize()
        _lib.lib.rtpb_debug_trace(None, 0)
        tr = buf.cpu().numpy().astype(np.float64)
        g = int(tr[STRIDE - 1]) if 0 < tr[STRIDE - 1] <= 148 else 148
        blk = tr[:g * STRIDE].reshape(g, STRIDE)
        t0 = blk[:, 0].min()
        u = blk[:, 2:2 + 6 * UNITS].reshape(g, UNITS, 6)
        lead = u[:, :, 2] > 0
        epi = u[:, :, 4] > 0
        ml = (u[:, :, 3] - u[:, :, 2])[lead] / 1e3
        ep = (u[:, :, 5] - u[:, :, 4])[epi] / 1e3
        accw = (u[:, :, 1] - u[:, :, 0])[lead] / 1e3
        # gap between a unit's last commit and the next unit's first stage (same CTA)
        ends = np.where(epi, u[:, :, 5], 0).max(1)
        print(f"  trace {k}: grid {g} units/CTA {epi.sum(1).min()}..{epi.sum(1).max()} mainloop {ml.mean():.2f} "
              f"(min {ml.min():.2f} max {ml.max():.2f}) us  epilogue {ep.mean():.2f} (max {ep.max():.2f})  acc-wait "
              f"{accw.mean():.2f} (max {accw.max():.2f})  span {(ends.max() - t0) / 1e3:.1f}  first-stage "
              f"{(np.where(lead, u[:, :, 2], np.inf).min() - t0) / 1e3:.2f}")
