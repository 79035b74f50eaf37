"""Dev probe: step kernels vs a torch fp32 reference on the GPU (not a test).

python tools/probe_steps.py  -> prints normwise errors and rough TFLOP/s.
"""
import ctypes as C
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
L = C.CDLL(os.path.join(ROOT, "paper_2311_01635_b200", "librtpb.so"))
L.rtpb_last_error.restype = C.c_char_p
L.rtpb_step_workspace_bytes.restype = C.c_size_t
L.rtpb_step_workspace_bytes.argtypes = [C.c_int] * 2 + [C.c_size_t] * 3
vp, sz = C.c_void_p, C.c_size_t
L.rtpb_fwd_step.argtypes = [C.c_int, vp, sz, vp, vp, sz, sz, vp, sz, sz, sz, sz, C.c_int, vp, sz, vp]
L.rtpb_dgrad_step.argtypes = [C.c_int, vp, sz, sz, vp, vp, sz, vp, sz, vp, sz, sz, sz, sz, C.c_int, vp, sz, vp]
L.rtpb_wgrad_step.argtypes = [C.c_int, vp, sz, vp, sz, sz, vp, vp, sz, sz, sz, vp, sz, vp]
L.rtpb_debug_force_bn.argtypes = [C.c_int]


def chk(rc):
    if rc:
        raise RuntimeError(L.rtpb_last_error().decode())


def nerr(got, ref):
    return ((got.float() - ref.float()).abs().max() / ref.float().abs().max().clamp_min(1e-30)).item()


def run(M, I, O, n, dt, bn=0):
    L.rtpb_debug_force_bn(bn)
    f32 = dt == 1
    tdt = torch.float32 if f32 else torch.bfloat16
    dev = "cuda"
    per = O // n
    g = torch.Generator(device=dev).manual_seed(0)
    X = (torch.rand(M, I, device=dev, generator=g) * 2 - 1).to(tdt)
    dY = (torch.rand(M, O, device=dev, generator=g) * 2 - 1).to(tdt)
    W = ((torch.rand(I, O, device=dev, generator=g) * 2 - 1) * 0.1).to(tdt)
    b = ((torch.rand(O, device=dev, generator=g) * 2 - 1) * 0.1).to(tdt)
    shards = [torch.cat([W[:, j * per:(j + 1) * per].reshape(-1), b[j * per:(j + 1) * per]]).contiguous()
              for j in range(n)]
    s = torch.cuda.current_stream().cuda_stream
    ws_bytes = max(L.rtpb_step_workspace_bytes(w, dt, M, I, per) for w in range(3))
    ws = torch.zeros(max(ws_bytes, 16), dtype=torch.uint8, device=dev)
    # forward: every shard into its column block, plain + GELU variants
    Y = torch.zeros(M, O, dtype=tdt, device=dev)
    H = torch.zeros(M, O, dtype=tdt, device=dev)
    for j in range(n):
        chk(L.rtpb_fwd_step(dt, X.data_ptr(), I, shards[j].data_ptr(), Y.data_ptr(), O, j * per, H.data_ptr(), O,
                            M, I, per, 1 | 16, ws.data_ptr(), ws.numel(), s))
    ref = X.float() @ W.float() + b.float()
    e_fwd = nerr(Y, ref)
    e_gelu = nerr(H, torch.nn.functional.gelu(ref))
    # dgrad accumulated over the n shards, last step emits dX and dX*gelu'(pre)
    acc = torch.zeros(M, I, dtype=torch.float32, device=dev)
    dX = torch.zeros(M, I, dtype=tdt, device=dev)
    for j in range(n):
        fl = (2 if j == 0 else 0) | (4 if j == n - 1 else 0)
        chk(L.rtpb_dgrad_step(dt, dY.data_ptr(), O, j * per, shards[j].data_ptr(), acc.data_ptr(), I, dX.data_ptr(),
                              I, None, 0, M, I, per, fl, ws.data_ptr(), ws.numel(), s))
    refdx = dY.float() @ W.float().t()
    e_dx = nerr(dX, refdx)
    # wgrad into a travelling shard for each j (G_in = G_out = zeros then twice)
    e_dw = 0.0
    for j in range(n):
        G = torch.zeros(I * per + per, dtype=torch.float32, device=dev)
        chk(L.rtpb_wgrad_step(dt, X.data_ptr(), I, dY.data_ptr(), O, j * per, G.data_ptr(), G.data_ptr(), M, I, per,
                              ws.data_ptr(), ws.numel(), s))
        chk(L.rtpb_wgrad_step(dt, X.data_ptr(), I, dY.data_ptr(), O, j * per, G.data_ptr(), G.data_ptr(), M, I, per,
                              ws.data_ptr(), ws.numel(), s))
        dyj = dY.float()[:, j * per:(j + 1) * per]
        refg = torch.cat([(X.float().t() @ dyj).reshape(-1), dyj.sum(0)]) * 2
        e_dw = max(e_dw, nerr(G, refg))
    torch.cuda.synchronize()
    print(f"M={M} I={I} O={O} n={n} dt={'f32' if f32 else 'bf16'} bn={bn}: fwd {e_fwd:.2e} gelu {e_gelu:.2e} "
          f"dx {e_dx:.2e} dw {e_dw:.2e}", flush=True)
    return max(e_fwd, e_gelu, e_dx, e_dw)


def bench(M, I, per, dt=0, iters=20):
    L.rtpb_debug_force_bn(0)
    dev = "cuda"
    tdt = torch.bfloat16 if dt == 0 else torch.float32
    X = torch.randn(M, I, device=dev).to(tdt)
    sh = torch.randn(I * per + per, device=dev).to(tdt) * 0.01
    Y = torch.empty(M, per, dtype=tdt, device=dev)
    dY = torch.randn(M, per, device=dev).to(tdt)
    acc = torch.empty(M, I, dtype=torch.float32, device=dev)
    dX = torch.empty(M, I, dtype=tdt, device=dev)
    G = torch.zeros(I * per + per, dtype=torch.float32, device=dev)
    ws = torch.zeros(max(16, max(L.rtpb_step_workspace_bytes(w, dt, M, I, per) for w in range(3))),
                     dtype=torch.uint8, device=dev)
    s = torch.cuda.current_stream().cuda_stream
    fns = {
        "fwd": lambda: chk(L.rtpb_fwd_step(dt, X.data_ptr(), I, sh.data_ptr(), Y.data_ptr(), per, 0, None, 0, M, I, per,
                                           16, ws.data_ptr(), ws.numel(), s)),
        "fwd_gelu": lambda: chk(L.rtpb_fwd_step(dt, X.data_ptr(), I, sh.data_ptr(), Y.data_ptr(), per, 0, Y.data_ptr(),
                                                per, M, I, per, 17, ws.data_ptr(), ws.numel(), s)),
        "dgrad_mid": lambda: chk(L.rtpb_dgrad_step(dt, dY.data_ptr(), per, 0, sh.data_ptr(), acc.data_ptr(), I, None, I,
                                                   None, 0, M, I, per, 0, ws.data_ptr(), ws.numel(), s)),
        "dgrad_1": lambda: chk(L.rtpb_dgrad_step(dt, dY.data_ptr(), per, 0, sh.data_ptr(), acc.data_ptr(), I,
                                                 dX.data_ptr(), I, None, 0, M, I, per, 6, ws.data_ptr(), ws.numel(), s)),
        "wgrad": lambda: chk(L.rtpb_wgrad_step(dt, X.data_ptr(), I, dY.data_ptr(), per, 0, G.data_ptr(), G.data_ptr(),
                                               M, I, per, ws.data_ptr(), ws.numel(), s)),
    }
    flops = 2.0 * M * I * per
    for name, fn in fns.items():
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / iters
        print(f"  {name:10s} M={M} I={I} per={per}: {ms*1e3:8.1f} us  {flops/ms/1e9:7.1f} TFLOP/s", flush=True)
    # torch reference matmul for scale
    Wt = torch.randn(I, per, device=dev).to(tdt)
    for _ in range(3):
        torch.matmul(X, Wt)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(iters):
        torch.matmul(X, Wt)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    print(f"  torch.matmul same shape: {ms*1e3:8.1f} us  {flops/ms/1e9:7.1f} TFLOP/s", flush=True)


if __name__ == "__main__":
    worst = 0.0
    cases = [(256, 128, 256, 2, 0, 64), (256, 128, 256, 2, 0, 128), (256, 128, 512, 2, 0, 256),
             (200, 64, 192, 3, 0, 0), (1000, 768, 3072, 4, 0, 0), (512, 256, 512, 4, 1, 0),
             (1024, 1024, 4096, 4, 1, 0), (130, 64, 64, 1, 1, 64)]
    for c in cases:
        try:
            worst = max(worst, run(*c))
        except Exception as e:  # noqa
            print("FAIL", c, e, flush=True)
            worst = 1e9
    print("WORST", worst)
    if "--bench" in sys.argv:
        bench(8192, 768, 3072)
        bench(8192, 3072, 768)
        bench(16384, 4096, 2048)
        bench(1024, 1024, 1024, dt=1)
