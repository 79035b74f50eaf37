"""Test helpers: exact fp64 -> bf16 / fp32 rounding, normwise errors, and
running the device RTP layers on host fp64 fixtures."""
import numpy as np

TOL = {"bf16": 2e-2, "f32": 1e-5}


def bf16_rne_bits(x: np.ndarray) -> np.ndarray:
    """Exact round-to-nearest-even of float64 values to bf16 bit patterns
    (round-to-odd into fp32, then RNE to bf16: no double rounding)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    f = x.astype(np.float32)
    inexact = f.astype(np.float64) != x
    u = f.view(np.uint32).copy()
    away = np.abs(f.astype(np.float64)) > np.abs(x)
    u = np.where(inexact & away, u - 1, u)
    u = np.where(inexact, u | 1, u).astype(np.uint32)
    rounding = (np.uint32(0x7FFF) + ((u >> 16) & 1)).astype(np.uint32)
    return ((u + rounding) >> 16).astype(np.uint16)


def bf16_round(x: np.ndarray) -> np.ndarray:
    """fp64 -> nearest bf16 value, returned as fp64."""
    bits = bf16_rne_bits(x).astype(np.uint32) << 16
    return bits.view(np.float32).astype(np.float64)


def dtype_round(x, dtype):
    return bf16_round(x) if dtype == "bf16" else np.asarray(x, np.float32).astype(np.float64)


def nerr(got, ref) -> float:
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    den = max(np.max(np.abs(ref)), 1e-300)
    return float(np.max(np.abs(got - ref)) / den)


def to_dev(a, dtype):
    import torch
    t = torch.from_numpy(np.ascontiguousarray(a, np.float64))
    return t.to(torch.float32 if dtype == "f32" else torch.bfloat16).cuda().contiguous()


def to_np(t):
    return t.detach().double().cpu().numpy()


def run_linear(n, w, b, x, dy, dtype="bf16", mode="inplace", transport="lockstep", flyweight=None):
    """RtpLinear Train fwd + bwd on n simulated workers (one device)."""
    from paper_2311_01635_b200 import rtp
    rows, i_dim = x.shape
    o_dim = w.shape[1] if w is not None else flyweight[1]
    M = rows // n
    g = rtp.WorkerGroup(n, transport)
    if flyweight is None:
        lin = rtp.RtpLinear(g, "lin", i_dim, o_dim, dtype, weight=w, bias=b)
    else:
        seed, _, base = flyweight
        lin = rtp.RtpLinear(g, "lin", i_dim, o_dim, dtype, seed=seed, stream_base=base)
    lin.set_rotation_mode(mode)
    if mode == "outofplace":
        lin.allocate_comm_spares()
    lin.zero_grads()
    xs = [to_dev(x[r * M:(r + 1) * M], dtype) for r in range(n)]
    dys = [to_dev(dy[r * M:(r + 1) * M], dtype) for r in range(n)]
    ys = lin.forward(xs)
    fwd_ids = [lin.slot(r)["logical_id"] for r in range(n)]
    fwd_offsets = [lin.slot(r)["rotation_offset"] for r in range(n)]
    dxs = lin.backward(dys)
    g.synchronize()
    out = {
        "y": np.concatenate([to_np(t) for t in ys]),
        "dx": np.concatenate([to_np(t) for t in dxs]),
        "grads": np.stack([to_np(lin.grad_shard(r)) for r in range(n)]),
        "weights": np.stack([to_np(lin.weight_shard(r)) for r in range(n)]),
        "fwd_ids": fwd_ids,
        "fwd_offsets": fwd_offsets,
        "bwd_ids": [lin.slot(r)["logical_id"] for r in range(n)],
        "trace": lin.trace(),
        "traffic": g.traffic(),
        "ledger": [g.ledger(r) for r in range(n)],
        "shard_len": lin.shard_len(),
    }
    lin.close()
    g.close()
    return out


def run_mlp(n, w1, b1, w2, b2, x, dy, dtype="bf16", mode="inplace", transport="lockstep"):
    from paper_2311_01635_b200 import rtp
    rows, h = x.shape
    f = w1.shape[1]
    M = rows // n
    g = rtp.WorkerGroup(n, transport)
    m = rtp.RtpMlp(g, "mlp", h, f, dtype, w1=w1, b1=b1, w2=w2, b2=b2)
    m.set_rotation_mode(mode)
    m.begin_step()
    m.zero_grads()
    xs = [to_dev(x[r * M:(r + 1) * M], dtype) for r in range(n)]
    dys = [to_dev(dy[r * M:(r + 1) * M], dtype) for r in range(n)]
    ys = m.forward(xs)
    dxs = m.backward(dys)
    g.synchronize()
    out = {
        "y": np.concatenate([to_np(t) for t in ys]),
        "dx": np.concatenate([to_np(t) for t in dxs]),
        "grads1": np.stack([to_np(m.ffn1.grad_shard(r)) for r in range(n)]),
        "grads2": np.stack([to_np(m.ffn2.grad_shard(r)) for r in range(n)]),
        "ledger": [g.ledger(r) for r in range(n)],
    }
    m.close()
    g.close()
    return out


STACK = dict(blocks=3, h=256, f=1024, rows_per_worker=256, steps=2)


def run_stack_local(g, ranks, n, chain=True, **kw):
    """A stack of Flyweight MLP blocks (out-of-place), `steps` training steps
    (zero_grads, forward through the blocks, backward in reverse), optionally
    chained so each block prefetches its neighbour's first shift. Runs the
    group's local ranks `ranks`; returns their outputs of the last step, dX
    and every block's gradient shards (keys per rank)."""
    import torch
    from paper_2311_01635_b200 import rtp
    p = {**STACK, **kw}
    h, f, M = p["h"], p["f"], p["rows_per_worker"]
    per_block = 2 * h * f + f + h
    mlps = []
    for b in range(p["blocks"]):
        m = rtp.RtpMlp(g, f"block{b}", h, f, "bf16", seed=42, stream_base=b * per_block)
        m.set_rotation_mode("outofplace")
        m.begin_step()
        mlps.append(m)
    if chain:
        for a, b in zip(mlps, mlps[1:]):
            a.chain(b)
    out = {}
    for step in range(p["steps"]):
        xs, dys = [], []
        for r in ranks:
            gen = torch.Generator().manual_seed(1000 * step + r)
            xs.append(((torch.rand(M, h, generator=gen) * 2 - 1).to(torch.bfloat16)).cuda())
            dys.append(((torch.rand(M, h, generator=gen) * 2 - 1).to(torch.bfloat16)).cuda())
        for m in mlps:
            m.zero_grads()
        inp = xs
        for m in mlps:
            inp = m.forward(inp)
        up = dys
        for m in reversed(mlps):
            up = m.backward(up)
        g.synchronize()
    for k, r in enumerate(ranks):
        out[f"y{r}"] = to_np(inp[k])
        out[f"dx{r}"] = to_np(up[k])
        for b, m in enumerate(mlps):
            out[f"g{b}_1_{r}"] = to_np(m.ffn1.grad_shard(r))
            out[f"g{b}_2_{r}"] = to_np(m.ffn2.grad_shard(r))
            out[f"home{b}_{r}"] = np.array([m.ffn1.slot(r)["logical_id"], m.ffn2.slot(r)["logical_id"]])
    for m in mlps:
        m.close()
    return out
