"""Dev tool: time every tile config (forced) for the MLP step GEMM shapes."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2311_01635_b200 import _lib, rtp  # noqa: E402

L = _lib.lib


def t_us(fn, iters=30):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters * 1e3


def sweep(M, I, per, gelu=False):
    dev = "cuda"
    X = torch.randn(M, I, device=dev).to(torch.bfloat16)
    sh = (torch.randn(I * per + per, device=dev) * 0.01).to(torch.bfloat16)
    Y = torch.empty(M, per, dtype=torch.bfloat16, device=dev)
    H = torch.empty(M, per, dtype=torch.bfloat16, device=dev)
    dY = torch.randn(M, per, device=dev).to(torch.bfloat16)
    dX = torch.empty(M, I, dtype=torch.bfloat16, device=dev)
    pre = torch.randn(M, I, device=dev).to(torch.bfloat16)
    G = torch.zeros(I * per + per, dtype=torch.float32, device=dev)
    fl = 2.0 * M * I * per
    res = {}
    for code in (0, 64, 128, 256, 1128, 1256):
        L.rtpb_debug_force_bn(code)
        r = {}
        r["fwd"] = t_us(lambda: rtp.fwd_step(X, sh, Y, 0, per, act=H if gelu else None))
        r["dgrad"] = t_us(lambda: rtp.dgrad_step(dY, 0, sh, None, dX, M, I, per, True, True,
                                                  pre=pre if gelu else None))
        r["wgrad"] = t_us(lambda: rtp.wgrad_step(X, dY, 0, G, G, per))
        res[code] = r
        print(f"M={M} I={I} per={per} gelu={gelu} tile={code:5d}: " +
              "  ".join(f"{k} {v:6.1f}us {fl / v / 1e6:6.0f}TF" for k, v in r.items()), flush=True)
    L.rtpb_debug_force_bn(0)


if __name__ == "__main__":
    sweep(8192, 768, 3072, gelu=True)   # ffn1 (fwd+gelu), dgrad, wgrad
    sweep(8192, 3072, 768, gelu=True)   # ffn2 (dgrad+gelu')
    sweep(16384, 4096, 2048)
