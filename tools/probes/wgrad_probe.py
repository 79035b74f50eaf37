"""Dev: run the config-(b) WGRAD shapes with a forced tile code (argv[1])."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2311_01635_b200 import _lib, rtp  # noqa: E402
code = int(sys.argv[1]) if len(sys.argv) > 1 else 0
_lib.lib.rtpb_debug_force_bn(code)
for (M, I, per) in ((8192, 768, 3072), (8192, 3072, 768)):
    X = torch.randn(M, I, device="cuda").to(torch.bfloat16)
    dY = torch.randn(M, per, device="cuda").to(torch.bfloat16)
    G = torch.zeros(I * per + per, dtype=torch.float32, device="cuda")
    for _ in range(3):
        rtp.wgrad_step(X, dY, 0, G, G, per)
torch.cuda.synchronize()
