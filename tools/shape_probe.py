"""Dev probe (not a test): step-GEMM throughput vs cuBLAS (torch.matmul) at
the config (b) / (d) step shapes and one large square shape, warm L2.

python tools/shape_probe.py
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2311_01635_b200 import _lib, rtp  # noqa: E402

L = _lib.lib


def t_us(fn, iters=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters * 1e3


def probe(M, I, per, gelu=False, codes=(0,)):
    dev = "cuda"
    X = torch.randn(M, I, device=dev).to(torch.bfloat16)
    sh = (torch.randn(I * per + per, device=dev) * 0.01).to(torch.bfloat16)
    W = sh[:I * per].view(I, per)
    Y = torch.empty(M, per, dtype=torch.bfloat16, device=dev)
    H = torch.empty(M, per, dtype=torch.bfloat16, device=dev)
    dY = torch.randn(M, per, device=dev).to(torch.bfloat16)
    dX = torch.empty(M, I, dtype=torch.bfloat16, device=dev)
    pre = torch.randn(M, I, device=dev).to(torch.bfloat16)
    G = torch.zeros(I * per + per, dtype=torch.float32, device=dev)
    fl = 2.0 * M * I * per
    cub = {"fwd": t_us(lambda: torch.matmul(X, W, out=Y)),
           "dgrad": t_us(lambda: torch.matmul(dY, W.t(), out=dX)),
           "wgrad": t_us(lambda: torch.matmul(X.t(), dY))}
    print(f"M={M} I={I} per={per} cuBLAS: " + "  ".join(f"{k} {v:7.1f}us {fl / v / 1e6:5.0f}TF"
                                                      for k, v in cub.items()), flush=True)
    for code in codes:
        L.rtpb_debug_force_bn(code)
        r = {"fwd": t_us(lambda: rtp.fwd_step(X, sh, Y, 0, per, act=H if gelu else None)),
             "dgrad": t_us(lambda: rtp.dgrad_step(dY, 0, sh, None, dX, M, I, per, True, True,
                                                   pre=pre if gelu else None)),
             "wgrad": t_us(lambda: rtp.wgrad_step(X, dY, 0, G, G, per))}
        print(f"M={M} I={I} per={per} gelu={int(gelu)} tile={code:4d}: " +
              "  ".join(f"{k} {v:7.1f}us {fl / v / 1e6:5.0f}TF" for k, v in r.items()), flush=True)
    L.rtpb_debug_force_bn(0)


if __name__ == "__main__":
    probe(8192, 8192, 8192, codes=(0, 256))
    probe(8192, 768, 3072, gelu=True, codes=(0, 256, 1128))
    probe(8192, 768, 3072, gelu=False)
    probe(8192, 3072, 768, gelu=True, codes=(0, 256, 1128))
    probe(16384, 4096, 2048, codes=(0,))
    probe(16384, 4096, 2048, gelu=True)
    probe(16384, 16384, 512, gelu=True)   # config (d) ffn2 step at N=8
