"""Full-size GPU parity: every BASELINE config at its real shapes, every
output and EVERY gradient shard (dW_j | db_j) compared whole.

The fp64 CPU oracle cannot run these sizes (config (c) is ~90 TFLOP per
step), so the reference here is the same arithmetic in fp64 on the device
(torch, cuBLAS DGEMM): Y = gelu(X W1 + b1) W2 + b2 and its exact-erf
backward (model.cpp:77-105, tensor.cpp:323-351), computed from the bf16
inputs the device path saw and the bf16 weights it holds (read back from
the home shards), chunked over rows. That fp64 reference is pinned to the C
oracle (oracle/rtp_oracle.c, itself pinned bit-for-bit to the reference's
goldens) on sampled entries in test_fp64_reference_pinned_to_oracle.
Tolerance: the north_star bf16 bound, normwise max|d|/max|ref| <= 2e-2 per
output tensor and per gradient shard.

Several workers share the one GPU (Lockstep transport): each worker's
shapes, schedule and kernels are those of one GPU of the N-GPU ring."""
import numpy as np
import pytest

from helpers import TOL

pytestmark = pytest.mark.gpu


def _nerr(got, ref) -> float:
    import torch
    d = (got.double() - ref.double()).abs().max()
    return float(d / ref.double().abs().max().clamp_min(1e-300))


def home_weights(lin, n, I, O):
    """Full (I x O) weight and (O) bias in fp64 from the home shards."""
    import torch
    per = O // n
    W = torch.empty(I, O, dtype=torch.float64, device="cuda")
    b = torch.empty(O, dtype=torch.float64, device="cuda")
    for r in range(n):
        assert lin.slot(r)["logical_id"] == r
        sh = lin.weight_shard(r).double()
        W[:, r * per:(r + 1) * per] = sh[:I * per].view(I, per)
        b[r * per:(r + 1) * per] = sh[I * per:]
    return W, b


def mlp_ref_fp64(xs, dys, W1, b1, W2, b2, chunk=4096):
    """fp64 MLP forward + backward over the row shards xs / dys (device
    bf16). Returns per-shard Y and dX, and dW1, db1, dW2, db2 summed over all
    rows (what the gradient shards hold after one step from zero)."""
    import torch
    s2 = 2.0 ** -0.5
    inv_sqrt_2pi = (2.0 * np.pi) ** -0.5
    dW1 = torch.zeros_like(W1)
    dW2 = torch.zeros_like(W2)
    db1 = torch.zeros_like(b1)
    db2 = torch.zeros_like(b2)
    ys, dxs = [], []
    for x, dy in zip(xs, dys):
        yparts, dxparts = [], []
        for a in range(0, x.shape[0], chunk):
            xc = x[a:a + chunk].double()
            dyc = dy[a:a + chunk].double()
            pre = xc @ W1 + b1
            cdf = 0.5 * (1.0 + torch.erf(pre * s2))
            act = pre * cdf
            yparts.append(act @ W2 + b2)
            dpre = (dyc @ W2.T) * (cdf + pre * torch.exp(-0.5 * pre * pre) * inv_sqrt_2pi)
            del cdf
            dxparts.append(dpre @ W1.T)
            dW2 += act.T @ dyc
            dW1 += xc.T @ dpre
            db1 += dpre.sum(0)
            db2 += dyc.sum(0)
            del pre, act, dpre
        ys.append(torch.cat(yparts))
        dxs.append(torch.cat(dxparts))
    return ys, dxs, dW1, db1, dW2, db2


def run_and_check(n, h, f, M, mode, seed=0, dtype="bf16", stream_base=0):
    """One Flyweight MLP block, n simulated workers of M rows, one step from
    zeroed gradients; checks Y, dX and every gradient shard whole."""
    import torch
    from paper_2311_01635_b200 import rtp
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    g = rtp.WorkerGroup(n, "lockstep")
    m = rtp.RtpMlp(g, "blk", h, f, dtype, seed=42, stream_base=stream_base)
    m.set_rotation_mode(mode)
    m.begin_step()
    m.zero_grads()
    gen = torch.Generator(device="cuda").manual_seed(seed)
    xs = [(torch.rand(M, h, device="cuda", generator=gen) * 2 - 1).to(tdt) for _ in range(n)]
    dys = [(torch.rand(M, h, device="cuda", generator=gen) * 2 - 1).to(tdt) for _ in range(n)]
    ys = m.forward(xs)
    dxs = m.backward(dys)
    g.synchronize()
    W1, b1 = home_weights(m.ffn1, n, h, f)
    W2, b2 = home_weights(m.ffn2, n, f, h)
    rys, rdxs, dW1, db1, dW2, db2 = mlp_ref_fp64(xs, dys, W1, b1, W2, b2)
    tol = TOL[dtype]
    errs = {"y": max(_nerr(a, b) for a, b in zip(ys, rys)), "dx": max(_nerr(a, b) for a, b in zip(dxs, rdxs))}
    for name, lin, dW, db, O in (("g1", m.ffn1, dW1, db1, f), ("g2", m.ffn2, dW2, db2, h)):
        per = O // n
        worst = 0.0
        for r in range(n):
            ref = torch.cat([dW[:, r * per:(r + 1) * per].reshape(-1), db[r * per:(r + 1) * per]])
            worst = max(worst, _nerr(lin.grad_shard(r), ref))
        errs[name] = worst
    # ownership after the step: every shard home (layers_test.cpp:100-112)
    for r in range(n):
        assert m.ffn1.slot(r)["logical_id"] == r and m.ffn2.slot(r)["logical_id"] == r
    m.close()
    g.close()
    del xs, dys, ys, dxs, rys, rdxs
    torch.cuda.empty_cache()
    for k, v in errs.items():
        assert v < tol, (k, v, errs)
    return errs


# ---------------------------------------------------------------- config (c)
@pytest.mark.parametrize("mode", ["outofplace", "inplace"])
def test_config_c_full_size_n8(mode):
    """Config (c): MLP 8192 -> 28672 -> 8192, T = 32768 over 8 workers
    (M = 4096, per = 3584 / 1024), both rotation modes."""
    run_and_check(8, 8192, 28672, 4096, mode, seed=11)


def test_config_c_full_size_n1():
    """Config (c) on one GPU (bench.py --config c): M = 32768, fused N = 1 schedule."""
    run_and_check(1, 8192, 28672, 32768, "outofplace", seed=12)


# ---------------------------------------------------------------- config (b)
@pytest.mark.parametrize("n", [1, 2, 4, 8])
def test_config_b_full_size(n):
    """Config (b): MLP 768 -> 3072 -> 768, 8192 rows per worker (the bench's
    per-GPU shape; N = 1 is the benched fused launch at M = 8192; N = 8 the
    thin split-K dW slices and paired dX)."""
    run_and_check(n, 768, 3072, 8192, "outofplace", seed=20 + n)


def test_config_b_inplace_n8():
    run_and_check(8, 768, 3072, 8192, "inplace", seed=30)


# ---------------------------------------------------------------- config (d)
def test_config_d_block_full_size_n8():
    """Config (d) block 4096 -> 16384 -> 4096 at its N = 8 shapes: 16384
    rows per worker (per = 2048 / 512, the 8-step fp32 dX accumulator),
    block 5 of the stack (stream base past 5 blocks' parameters)."""
    h, f = 4096, 16384
    run_and_check(8, h, f, 16384, "outofplace", seed=40, stream_base=5 * (2 * h * f + f + h))


def test_config_d_block_full_size_n1():
    """Config (d) block at the benched N = 1 shape (M = 16384, fused launches)."""
    run_and_check(1, 4096, 16384, 16384, "outofplace", seed=41)


# ---------------------------------------------------------------- fp32 at N = 8
@pytest.mark.parametrize("mode", ["outofplace", "inplace"])
def test_fp32_mlp_eight_workers_matches_reference(golden, mode):
    """fp32 (3xTF32) mode at N = 8 against the reference's own RtpMlp
    (tests/golden/mlp_ring.npz), tolerance 1e-5."""
    from helpers import run_mlp, nerr
    g = golden("mlp_ring")
    out = run_mlp(8, g["w1"], g["b1"], g["w2"], g["b2"], g["x"], g["dy"], "f32", mode)
    assert nerr(out["y"], g["n8_y"]) < TOL["f32"]
    assert nerr(out["dx"], g["n8_dx"]) < TOL["f32"]
    for r in range(8):
        assert nerr(out["grads1"][r], g["n8_grads1"][r]) < TOL["f32"]
        assert nerr(out["grads2"][r], g["n8_grads2"][r]) < TOL["f32"]


@pytest.mark.parametrize("n", [1, 2, 4, 8])
def test_bf16_mlp_ring_fixture(golden, n):
    """The bench's self-check fixture (reference RtpMlp, h=64, f=256) in the
    in-process transport, both modes."""
    from helpers import run_mlp, nerr
    g = golden("mlp_ring")
    for mode in ("outofplace", "inplace"):
        out = run_mlp(n, g["w1"], g["b1"], g["w2"], g["b2"], g["x"], g["dy"], "bf16", mode)
        assert nerr(out["y"], g[f"n{n}_y"]) < TOL["bf16"]
        assert nerr(out["dx"], g[f"n{n}_dx"]) < TOL["bf16"]
        for r in range(n):
            assert nerr(out["grads1"][r], g[f"n{n}_grads1"][r]) < TOL["bf16"]
            assert nerr(out["grads2"][r], g[f"n{n}_grads2"][r]) < TOL["bf16"]


# ---------------------------------------------------------------- the fp64 reference itself
def test_fp64_reference_pinned_to_oracle(oracle, golden):
    """mlp_ref_fp64 reproduces the C oracle's RTP MLP (fp64, the reference's
    summation order) to fp64 rounding on the golden fixture, so the
    full-size tests above compare against the oracle's arithmetic."""
    import torch
    g = golden("mlp_ring")
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    ref = oracle.rtp_mlp(4, g["w1"], g["b1"], g["w2"], g["b2"], g["x"], g["dy"])
    M = g["x"].shape[0] // 4
    xs = [dev(g["x"][r * M:(r + 1) * M]) for r in range(4)]
    dys = [dev(g["dy"][r * M:(r + 1) * M]) for r in range(4)]
    ys, dxs, dW1, db1, dW2, db2 = mlp_ref_fp64(xs, dys, dev(g["w1"]), dev(g["b1"]), dev(g["w2"]), dev(g["b2"]),
                                               chunk=16)
    assert np.max(np.abs(torch.cat(ys).cpu().numpy() - ref["y"])) < 1e-12
    assert np.max(np.abs(torch.cat(dxs).cpu().numpy() - ref["dx"])) < 1e-12
    h, f = g["w1"].shape
    for r in range(4):
        per1, per2 = f // 4, h // 4
        s1 = np.concatenate([dW1[:, r * per1:(r + 1) * per1].cpu().numpy().ravel(),
                             db1[r * per1:(r + 1) * per1].cpu().numpy()])
        s2 = np.concatenate([dW2[:, r * per2:(r + 1) * per2].cpu().numpy().ravel(),
                             db2[r * per2:(r + 1) * per2].cpu().numpy()])
        assert np.max(np.abs(s1 - ref["grads1"][r])) < 1e-12
        assert np.max(np.abs(s2 - ref["grads2"][r])) < 1e-12


# ---------------------------------------------------------------- chained stack
@pytest.mark.parametrize("mode", ["outofplace", "inplace"])
def test_chained_stack_vs_fp64(mode):
    """A 3-block Flyweight stack, blocks chained (each block posts its
    neighbour's first shift under its own last step), 4 workers, two training
    steps: the second step's outputs, dX and every block's gradient shards
    against the fp64 composition y = mlp3(mlp2(mlp1(x))) and its backward."""
    import torch
    from paper_2311_01635_b200 import rtp
    n, h, f, M, blocks = 4, 256, 1024, 512, 3
    g = rtp.WorkerGroup(n, "lockstep")
    per_block = 2 * h * f + f + h
    mlps = []
    for b in range(blocks):
        m = rtp.RtpMlp(g, f"block{b}", h, f, "bf16", seed=42, stream_base=b * per_block)
        m.set_rotation_mode(mode)
        m.begin_step()
        mlps.append(m)
    for a, b in zip(mlps, mlps[1:]):
        a.chain(b)
    gen = torch.Generator(device="cuda").manual_seed(3)
    for step in range(2):
        xs = [(torch.rand(M, h, device="cuda", generator=gen) * 2 - 1).to(torch.bfloat16) for _ in range(n)]
        dys = [(torch.rand(M, h, device="cuda", generator=gen) * 2 - 1).to(torch.bfloat16) for _ in range(n)]
        for m in mlps:
            m.zero_grads()
        acts = [xs]
        for m in mlps:
            acts.append(m.forward(acts[-1]))
        ups = [dys]  # ups[i]: upstream gradient of block blocks-1-i (device bf16)
        for m in reversed(mlps):
            ups.append(m.backward(ups[-1]))
        g.synchronize()
    # fp64 reference per block from the bf16 input and upstream the device saw:
    # Y, dX and both layers' gradient shards of every block of the chain
    for b in range(blocks):
        (W1, b1), (W2, b2) = home_weights(mlps[b].ffn1, n, h, f), home_weights(mlps[b].ffn2, n, f, h)
        up = ups[blocks - 1 - b]
        ys_ref, dx_ref, dW1, db1, dW2, db2 = mlp_ref_fp64(acts[b], up, W1, b1, W2, b2)
        assert max(_nerr(a, r) for a, r in zip(acts[b + 1], ys_ref)) < TOL["bf16"], b
        assert max(_nerr(a, r) for a, r in zip(ups[blocks - b], dx_ref)) < TOL["bf16"], b
        for lin, dW, db, O in ((mlps[b].ffn1, dW1, db1, f), (mlps[b].ffn2, dW2, db2, h)):
            pr = O // n
            for r in range(n):
                ref = torch.cat([dW[:, r * pr:(r + 1) * pr].reshape(-1), db[r * pr:(r + 1) * pr]])
                assert _nerr(lin.grad_shard(r), ref) < TOL["bf16"], (b, r)
    for m in mlps:
        for r in range(n):
            assert m.ffn1.slot(r)["logical_id"] == r and m.ffn2.slot(r)["logical_id"] == r
        m.close()
    g.close()
