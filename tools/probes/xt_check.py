"""Dev probe: the dW with A = X^T (RTPB_WGRAD_XT=1, transposed copy, K-major) against the default
MN-major dW: run once per setting (the switch is read once per process), save / compare G bitwise and
against an fp32 torch product. python tools/probes/xt_check.py save|check out.pt"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2311_01635_b200 import rtp  # noqa: E402

mode, path = sys.argv[1], sys.argv[2]
res = {}
for (M, I, per) in [(16384, 4096, 16384), (1024, 512, 2048), (2048, 1024, 768)]:
    g = torch.Generator(device="cuda").manual_seed(M + I + per)
    X = torch.randn(M, I, device="cuda", generator=g).to(torch.bfloat16)
    dY = torch.randn(M, per, device="cuda", generator=g).to(torch.bfloat16)
    G = torch.zeros(I * per + per, dtype=torch.float32, device="cuda")
    rtp.wgrad_step(X, dY, 0, None, G, per)
    torch.cuda.synchronize()
    ref = X.float().t() @ dY.float()
    err = ((G[:I * per].view(I, per) - ref).norm() / ref.norm()).item()
    db = (G[I * per:] - dY.float().sum(0)).abs().max().item()
    res[(M, I, per)] = G.cpu()
    print(f"{mode} M={M} I={I} per={per}: normwise vs fp32 {err:.3e}, db max abs {db:.3e}")
if mode == "save":
    torch.save(res, path)
else:
    old = torch.load(path)
    for k, v in res.items():
        print(f"check {k}: bitwise equal to the MN-major dW: {torch.equal(old[k], v)}, max |d| {(old[k] - v).abs().max().item():.3e}")
