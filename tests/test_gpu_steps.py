"""GPU: the per-rotation-step tcgen05 kernels (include/rtpb.h layer 1) against
an fp32 torch reference of the same op on the same (already-rounded) inputs.
Tolerance (normwise max|d| / max|ref|): bf16 2e-2, fp32 (3xTF32) 1e-5."""
import pytest
import torch

pytestmark = pytest.mark.gpu

TOL = {"bf16": 2e-2, "f32": 1e-5}


def nerr(got, ref):
    return ((got.double() - ref.double()).abs().max() / ref.double().abs().max().clamp_min(1e-30)).item()


def make(M, I, O, n, dt, seed=0):
    from paper_2311_01635_b200 import rtp  # noqa: F401
    tdt = torch.float32 if dt == "f32" else torch.bfloat16
    g = torch.Generator(device="cuda").manual_seed(seed)
    X = (torch.rand(M, I, device="cuda", generator=g) * 2 - 1).to(tdt)
    dY = (torch.rand(M, O, device="cuda", generator=g) * 2 - 1).to(tdt)
    W = ((torch.rand(I, O, device="cuda", generator=g) * 2 - 1) * 0.1).to(tdt)
    b = ((torch.rand(O, device="cuda", generator=g) * 2 - 1) * 0.1).to(tdt)
    per = O // n
    shards = [torch.cat([W[:, j * per:(j + 1) * per].reshape(-1), b[j * per:(j + 1) * per]]).contiguous()
              for j in range(n)]
    return X, dY, W, b, shards


CASES = [
    # M, I, O, n, dtype, forced tile (0 = heuristic; BN for one CTA, 1000+BN for a CTA pair)
    (256, 128, 256, 2, "bf16", 64),
    (256, 128, 256, 2, "bf16", 128),
    (256, 128, 512, 2, "bf16", 256),
    (512, 128, 512, 2, "bf16", 1256),  # cta_group::2, 256 x 256 tiles
    (512, 128, 512, 2, "bf16", 1128),  # cta_group::2, 256 x 128 tiles
    (1000, 768, 3072, 4, "bf16", 1256),  # pair tiles with a ragged last 256-row tile
    (300, 64, 256, 1, "bf16", 1128),
    (200, 64, 192, 3, "bf16", 0),     # ragged M, per = 64
    (1000, 768, 3072, 4, "bf16", 0),  # GPT-2 width, tail rows
    (8192, 768, 3072, 4, "bf16", 0),  # config (b) dW: 8-way ordered split-K + fused bias sums
    (8192, 3072, 768, 8, "bf16", 0),  # ffn2 at N = 8 (per 96): split-K on 256 x 128 pair tiles
    (8192, 768, 3072, 8, "bf16", 0),  # ffn1 at N = 8 (per 384)
    (4000, 768, 3000, 3, "bf16", 1128),  # pair 256 x 128, ragged K and N
    (8, 8, 16, 2, "bf16", 0),         # minimal aligned shape
    (512, 256, 512, 4, "f32", 0),
    (1024, 1024, 4096, 4, "f32", 0),  # config (a) shapes, one worker's rows
    (130, 64, 64, 1, "f32", 64),
]


@pytest.mark.parametrize("M,I,O,n,dt,bn", CASES)
def test_step_kernels_vs_torch(M, I, O, n, dt, bn):
    from paper_2311_01635_b200 import _lib, rtp
    _lib.lib.rtpb_debug_force_bn(bn)
    try:
        X, dY, W, b, shards = make(M, I, O, n, dt)
        per = O // n
        Y = torch.zeros(M, O, dtype=X.dtype, device="cuda")
        H = torch.zeros(M, O, dtype=X.dtype, device="cuda")
        for j in range(n):
            rtp.fwd_step(X, shards[j], Y, j * per, per, act=H)
        ref = X.double() @ W.double() + b.double()
        assert nerr(Y, ref) < TOL[dt]
        assert nerr(H, torch.nn.functional.gelu(ref)) < TOL[dt]
        # dX accumulated across n steps in the fp32 accumulator
        acc = torch.zeros(M, I, dtype=torch.float32, device="cuda")
        dX = torch.zeros(M, I, dtype=X.dtype, device="cuda")
        for j in range(n):
            rtp.dgrad_step(dY, j * per, shards[j], acc, dX, M, I, per, first=j == 0, last=j == n - 1)
        assert nerr(dX, dY.double() @ W.double().t()) < TOL[dt]
        # dX with gelu' fused into the last step (model.cpp:101-104)
        pre = Y
        dpre = torch.zeros_like(dX)
        # use a square-compatible pre for the fused test: pre must be M x I
        pre_i = (torch.rand(M, I, device="cuda") * 4 - 2).to(X.dtype)
        for j in range(n):
            rtp.dgrad_step(dY, j * per, shards[j], acc, dpre, M, I, per, first=j == 0, last=j == n - 1, pre=pre_i)
        p = pre_i.double()
        gprime = 0.5 * (1 + torch.erf(p / 2 ** 0.5)) + p * torch.exp(-0.5 * p * p) / (2 * torch.pi) ** 0.5
        assert nerr(dpre, (dY.double() @ W.double().t()) * gprime) < TOL[dt]
        del pre
        # dW + db into a travelling shard, accumulated twice (G_in + P epilogue)
        for j in range(n):
            G = torch.zeros(I * per + per, dtype=torch.float32, device="cuda")
            rtp.wgrad_step(X, dY, j * per, G, G, per)
            rtp.wgrad_step(X, dY, j * per, G, G, per)
            dyj = dY.double()[:, j * per:(j + 1) * per]
            refg = torch.cat([(X.double().t() @ dyj).reshape(-1), dyj.sum(0)]) * 2
            assert nerr(G, refg) < TOL[dt]
            # bias gradient on its own scale (fused column sums on CTA-pair tiles)
            assert nerr(G[I * per:], refg[I * per:]) < TOL[dt]
            # out-of-place accumulation: G_out = G_in + P leaves G_in intact
            G2 = torch.empty_like(G)
            rtp.wgrad_step(X, dY, j * per, G, G2, per)
            assert nerr(G2, refg * 1.5) < TOL[dt]
            assert nerr(G, refg) < TOL[dt]
            # known-zero gradient (g_in = NULL): G_out = P, nothing read
            G3 = torch.full_like(G, float("nan"))
            rtp.wgrad_step(X, dY, j * per, None, G3, per)
            assert nerr(G3, refg * 0.5) < TOL[dt]
            assert nerr(G3[I * per:], refg[I * per:] * 0.5) < TOL[dt]
        torch.cuda.synchronize()
    finally:
        _lib.lib.rtpb_debug_force_bn(0)


def test_misaligned_geometry_raises_config_error():
    from paper_2311_01635_b200 import rtp
    X = torch.zeros(16, 12, dtype=torch.bfloat16, device="cuda")
    sh = torch.zeros(12 * 4 + 4, dtype=torch.bfloat16, device="cuda")
    Y = torch.zeros(16, 4, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(rtp.ConfigError):
        rtp.fwd_step(X, sh, Y, 0, 4)


def test_gpt2_width_bench_shapes_all_tile_widths():
    """Config (b) shapes (T=8192, 768<->3072) at every tile width."""
    from paper_2311_01635_b200 import _lib, rtp
    M, I, O = 2048, 768, 3072
    X, dY, W, b, shards = make(M, I, O, 1, "bf16", seed=3)
    ref = X.double() @ W.double() + b.double()
    for bn in (64, 128, 256, 1128, 1256):
        _lib.lib.rtpb_debug_force_bn(bn)
        try:
            Y = torch.zeros(M, O, dtype=torch.bfloat16, device="cuda")
            rtp.fwd_step(X, shards[0], Y, 0, O)
            assert nerr(Y, ref) < 2e-2
        finally:
            _lib.lib.rtpb_debug_force_bn(0)
