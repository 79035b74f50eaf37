"""Dev probe (ncu target): config (b) at N = 8 shard shapes on a Solo group
(rank 0's schedule, shifts skipped), one warm-up step then one profiled step
of pass launches — fwd(ffn1), fwd(ffn2), dX(ffn2) || dW(ffn2), dX(ffn1) ||
dW(ffn1). Run under ncu with --replay-mode application (the pass grids spin on
flags another stream raises; kernel replay serialises them)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2311_01635_b200 import rtp  # noqa: E402

N, M, H, F = 8, 8192, 768, 3072
g = rtp.WorkerGroup.solo(N, 0, 0)
mlp = rtp.RtpMlp(g, "probe", H, F, "bf16", seed=42, stream_base=0)
mlp.set_rotation_mode("outofplace")
mlp.begin_step()
x = (torch.rand(M, H, device="cuda") * 2 - 1).to(torch.bfloat16)
dy = (torch.rand(M, H, device="cuda") * 2 - 1).to(torch.bfloat16)
y, dx = torch.empty_like(x), torch.empty_like(x)
for _ in range(2):
    mlp.zero_grads()
    mlp.forward([x], out=[y])
    mlp.backward([dy], out=[dx])
torch.cuda.synchronize()
print("ok", float(dx.float().abs().mean()))
