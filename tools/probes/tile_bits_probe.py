"""Dev probe (not a test): do the step GEMMs' results depend on the tile shape?
Runs each kind with every tile code (rtpb_debug_force_bn) and compares bits
with the default choice."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2311_01635_b200 import _lib, rtp  # noqa: E402

for (M, I, per) in [(8192, 768, 384), (8192, 3072, 96), (4096, 1024, 512)]:
    g = torch.Generator(device="cuda").manual_seed(0)
    X = (torch.rand(M, I, generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    sh = ((torch.rand(I * per + per, generator=g, device="cuda") * 2 - 1) * 0.1).to(torch.bfloat16)
    dY = (torch.rand(M, per, generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    outs = {}
    for code in [0, 1256, 1128, 256, 128, 64]:
        _lib.lib.rtpb_debug_force_bn(code)
        Y = torch.zeros(M, per, dtype=torch.bfloat16, device="cuda")
        rtp.fwd_step(X, sh, Y, 0, per)
        dX = torch.zeros(M, I, dtype=torch.bfloat16, device="cuda")
        acc = torch.zeros(M, I, dtype=torch.float32, device="cuda")
        rtp.dgrad_step(dY, 0, sh, acc, acc, M, I, per, True, False)  # fp32 partial
        torch.cuda.synchronize()
        outs[code] = (Y.clone(), acc.clone())
    _lib.lib.rtpb_debug_force_bn(0)
    for code, (y, a) in outs.items():
        print(M, I, per, "code", code, "fwd same bits:", torch.equal(y, outs[0][0]), "dgrad same bits:",
              torch.equal(a, outs[0][1]), flush=True)
