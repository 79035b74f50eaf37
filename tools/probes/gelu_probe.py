"""Dev: config-(b) GELU-fused step kernels (fwd+gelu for ffn1, dX*gelu' for ffn2)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2311_01635_b200 import rtp  # noqa: E402
M, h, f = 8192, 768, 3072
X = torch.randn(M, h, device="cuda").to(torch.bfloat16)
W1 = (torch.randn(h * f + f, device="cuda") * 0.05).to(torch.bfloat16)
PRE = torch.empty(M, f, dtype=torch.bfloat16, device="cuda")
ACT = torch.empty(M, f, dtype=torch.bfloat16, device="cuda")
dY = torch.randn(M, h, device="cuda").to(torch.bfloat16)
W2 = (torch.randn(f * h + h, device="cuda") * 0.05).to(torch.bfloat16)
DPRE = torch.empty(M, f, dtype=torch.bfloat16, device="cuda")
for _ in range(3):
    rtp.fwd_step(X, W1, PRE, 0, f, act=ACT)
    rtp.dgrad_step(dY, 0, W2, None, DPRE, M, f, h, True, True, pre=PRE)
torch.cuda.synchronize()
