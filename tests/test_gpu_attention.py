"""RtpAttention on the device (layers_attention.cpp:43-198)
against the reference's own RtpAttention (tests/golden/attention.npz, made
by oracle/_ref) and the C oracle (oracle/rtp_oracle.c orc_rtp_attention,
pinned bit-for-bit to those goldens by tests/test_oracle.py):
  * bit-exact: shard ownership per (phase, step, rank), shards home after a
    step, resident weights equal to the reference's shards;
  * normwise max|d|/max|ref| per output and per gradient shard: bf16 <= 2e-2,
    fp32 (3xTF32 projections, fp32 attention core) <= 1e-5."""
import numpy as np
import pytest

from helpers import TOL, dtype_round, nerr, to_dev, to_np

pytestmark = pytest.mark.gpu


def run_attention(n, heads, seq, wq, wk, wv, wo, x, dy, dtype="bf16", mode="inplace", transport="lockstep"):
    from paper_2311_01635_b200 import rtp
    rows, H = x.shape
    M = rows // n
    g = rtp.WorkerGroup(n, transport)
    a = rtp.RtpAttention(g, "attn", H, heads, seq, wq, wk, wv, wo, dtype)
    a.set_rotation_mode(mode)
    if mode == "outofplace":
        a.allocate_comm_spares()
    a.zero_grads()
    ys = a.forward([to_dev(x[r * M:(r + 1) * M], dtype) for r in range(n)])
    fwd_ids = [a.slot(r)["logical_id"] for r in range(n)]
    dxs = a.backward([to_dev(dy[r * M:(r + 1) * M], dtype) for r in range(n)])
    g.synchronize()
    out = {"y": np.concatenate([to_np(t) for t in ys]), "dx": np.concatenate([to_np(t) for t in dxs]),
           "grads": np.stack([a.shard(r, grad=True) for r in range(n)]),
           "weights": np.stack([a.shard(r) for r in range(n)]),
           "fwd_ids": fwd_ids, "bwd_ids": [a.slot(r)["logical_id"] for r in range(n)], "trace": a.trace(),
           "traffic": g.traffic(), "ledger": [g.ledger(r) for r in range(n)]}
    a.close()
    g.close()
    return out


def ref_shard(wq, wk, wv, wo, n, j):
    """attention_shard_groups + flatten (layers_common.cpp:54-74)."""
    H = wq.shape[0]
    gw = H // n
    return np.concatenate([wq[:, j * gw:(j + 1) * gw].ravel(), wk[:, j * gw:(j + 1) * gw].ravel(),
                           wv[:, j * gw:(j + 1) * gw].ravel(), wo[j * gw:(j + 1) * gw, :].ravel()])


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
@pytest.mark.parametrize("mode", ["inplace", "outofplace"])
@pytest.mark.parametrize("n", [1, 2, 4])
def test_attention_matches_reference(golden, n, mode, dtype):
    g = golden("attention")
    heads, seq = int(g["heads"]), int(g["seq"])
    W = [g[k] for k in ("wq", "wk", "wv", "wo")]
    out = run_attention(n, heads, seq, *W, g[f"n{n}_x"], g[f"n{n}_dy"], dtype, mode)
    assert nerr(out["y"], g[f"n{n}_y"]) < TOL[dtype]
    assert nerr(out["dx"], g[f"n{n}_dx"]) < TOL[dtype]
    for r in range(n):
        assert nerr(out["grads"][r], g[f"n{n}_grads"][r]) < TOL[dtype], r
    # ownership: train forward ends with rank r holding shard r+1, backward re-homes
    assert out["fwd_ids"] == [(r + 1) % n for r in range(n)]
    assert out["bwd_ids"] == list(range(n))
    fwd, bwd = out["trace"]
    for s in range(n):
        assert fwd[s] == [(r - s) % n for r in range(n)]
        assert bwd[s] == [(r + 1 + s) % n for r in range(n)]
    # N-1 weight hops forward, N-1 weight+gradient hops backward
    assert [k for k, _, _ in out["traffic"]] == ["rotation_cw"] * (n - 1) + ["rotation_ccw"] * (n - 1)
    for r in range(n):
        assert np.array_equal(out["weights"][r], dtype_round(ref_shard(*W, n, r), dtype))


def test_attention_lockstep_equals_concurrent(golden):
    g = golden("attention")
    W = [g[k] for k in ("wq", "wk", "wv", "wo")]
    a = run_attention(4, 4, 8, *W, g["n4_x"], g["n4_dy"], "bf16", "outofplace", "lockstep")
    b = run_attention(4, 4, 8, *W, g["n4_x"], g["n4_dy"], "bf16", "outofplace", "concurrent")
    for k in ("y", "dx", "grads"):
        assert np.array_equal(a[k], b[k]), k


@pytest.mark.parametrize("n", [2, 4, 8])
def test_attention_vs_oracle_eight_heads(oracle, n):
    """hidden 64, 8 heads (head_dim 8), seq 16, two sequences per worker."""
    rng = np.random.default_rng(31 + n)
    H, heads, seq = 64, 8, 16
    W = [rng.uniform(-0.1, 0.1, (H, H)) for _ in range(4)]
    rows = n * 2 * seq
    x, dy = rng.uniform(-1, 1, (rows, H)), rng.uniform(-1, 1, (rows, H))
    ref = oracle.rtp_attention(n, heads, seq, *W, x, dy)
    for dtype in ("bf16", "f32"):
        out = run_attention(n, heads, seq, *W, x, dy, dtype, "outofplace")
        assert nerr(out["y"], ref["y"]) < TOL[dtype], dtype
        assert nerr(out["dx"], ref["dx"]) < TOL[dtype], dtype
        for r in range(n):
            assert nerr(out["grads"][r], ref["grads"][r]) < TOL[dtype], (dtype, r)


def _attention_fp64(W, x, dy, heads, seq):
    """Serial multi-head attention fp64 forward + backward (the math of
    layers_attention.cpp with one shard), torch on the device."""
    import torch
    wq, wk, wv, wo = (torch.from_numpy(w).cuda() for w in W)
    X = torch.from_numpy(x).cuda().requires_grad_(True)
    params = [p.requires_grad_(True) for p in (wq, wk, wv, wo)]
    rows, H = X.shape
    hd = H // heads
    B = rows // seq

    def split(t):
        return t.view(B, seq, heads, hd).transpose(1, 2)
    q, k, v = split(X @ params[0]), split(X @ params[1]), split(X @ params[2])
    p = torch.softmax(q @ k.transpose(-1, -2) / hd ** 0.5, dim=-1)
    a = (p @ v).transpose(1, 2).reshape(rows, H)
    y = a @ params[3]
    y.backward(torch.from_numpy(dy).cuda())
    return y.detach().cpu().numpy(), X.grad.cpu().numpy(), [p.grad.cpu().numpy() for p in params]


def test_attention_long_sequences_vs_fp64():
    """hidden 256, 4 heads (head_dim 64), seq 256 (8 key tiles), 2 workers x
    2 sequences, bf16 and fp32, against an fp64 serial computation; gradient
    shards assembled in the reference layout."""
    rng = np.random.default_rng(7)
    H, heads, seq, n = 256, 4, 256, 2
    W = [rng.uniform(-0.1, 0.1, (H, H)) for _ in range(4)]
    rows = n * 2 * seq
    x, dy = rng.uniform(-1, 1, (rows, H)), rng.uniform(-1, 1, (rows, H))
    for dtype in ("bf16", "f32"):
        Wd = [dtype_round(w, dtype) for w in W]
        y_ref, dx_ref, gw_ref = _attention_fp64(Wd, dtype_round(x, dtype), dtype_round(dy, dtype), heads, seq)
        out = run_attention(n, heads, seq, *W, x, dy, dtype, "outofplace")
        tol = TOL[dtype] if dtype == "bf16" else 2e-5  # fp32 core: 256-term softmax sums in fp32
        assert nerr(out["y"], y_ref) < tol, dtype
        assert nerr(out["dx"], dx_ref) < tol, dtype
        for r in range(n):
            assert nerr(out["grads"][r], ref_shard(*gw_ref, n, r)) < tol, (dtype, r)


def test_attention_eval_rehomes_and_records_nothing(golden):
    import torch
    from paper_2311_01635_b200 import rtp
    g = golden("attention")
    W = [g[k] for k in ("wq", "wk", "wv", "wo")]
    n = 4
    grp = rtp.WorkerGroup(n)
    a = rtp.RtpAttention(grp, "attn", 32, 4, 8, *W, "bf16")
    x = g["n4_x"]
    M = x.shape[0] // n
    ys = a.forward([to_dev(x[r * M:(r + 1) * M], "bf16") for r in range(n)], mode="eval")
    assert nerr(np.concatenate([to_np(t) for t in ys]), g["n4_y"]) < 2e-2
    assert [a.slot(r)["logical_id"] for r in range(n)] == list(range(n))
    with pytest.raises(rtp.StateError):
        a.backward([torch.zeros(M, 32, dtype=torch.bfloat16, device="cuda") for _ in range(n)])
    a.close()
    grp.close()


def test_attention_errors():
    import torch
    from paper_2311_01635_b200 import rtp
    W = [np.zeros((32, 32))] * 4
    grp = rtp.WorkerGroup(8)
    with pytest.raises(rtp.ConfigError, match="multiple"):
        rtp.RtpAttention(grp, "bad", 32, 4, 8, *W)  # 4 heads over 8 shards (partition.cpp:76-79)
    grp.close()
    grp = rtp.WorkerGroup(2)
    with pytest.raises(rtp.ConfigError):
        rtp.RtpAttention(grp, "bad", 30, 4, 8, *[np.zeros((30, 30))] * 4)  # hidden % heads
    a = rtp.RtpAttention(grp, "attn", 32, 4, 8, *W)
    with pytest.raises(rtp.DimensionError):
        a.forward([torch.zeros(12, 32, dtype=torch.bfloat16, device="cuda") for _ in range(2)])  # 12 % seq 8
    with pytest.raises(rtp.StateError):
        a.backward([torch.zeros(16, 32, dtype=torch.bfloat16, device="cuda") for _ in range(2)])
    a.close()
    grp.close()
