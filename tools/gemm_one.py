"""Dev probe (not a test): launch each step GEMM kind a few times at one shape,
for ncu captures (-k regex:rtp_gemm -s 3 -c 3) and quick timing.

python tools/gemm_one.py M I per [kinds=fwd,dgrad,wgrad] [tile code]
"""
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
fns = {"fwd": lambda: rtp.fwd_step(X, sh, Y, 0, per),
       "dgrad": lambda: rtp.dgrad_step(dY, 0, sh, None, dX, M, I, per, True, True),
       "wgrad": lambda: rtp.wgrad_step(X, dY, 0, G, G, per)}
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
    print(f"{k:6s} M={M} I={I} per={per} tile={code}: {us:8.1f} us {fl / us / 1e6:6.0f} TF/s", flush=True)
