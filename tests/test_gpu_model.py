"""The whole rotated model on the device (RtpModel, model.cpp:7-121:
embedding -> blocks of attention + FFN-or-MoE with residual connections ->
head; SURVEY §8f.2 block wiring and §8f.4 embedding + head) against the
reference's own RtpModel(SerialModel(dims, 42)) run (tests/golden/model.npz):
same parameters (SplitMix64 in SerialModel order), same ids, the reference's
dlogits as upstream; logits, every layer's gradient shard on every rank and
the MoE gate gradients within the north_star tolerance; shards home."""
import numpy as np
import pytest

from helpers import TOL, nerr, to_dev, to_np

pytestmark = pytest.mark.gpu


def run_model(g, n, moe, mode, dtype, transport="lockstep"):
    from paper_2311_01635_b200 import rtp
    kind = "moe" if moe else "dense"
    p = f"{kind}_n{n}_"
    dims = {k: int(g[k]) for k in ("heads", "hidden", "layers", "seq", "vocab", "ffn")}
    grp = rtp.WorkerGroup(n, transport)
    m = rtp.RtpModel(grp, moe=moe, seed=42, mode=mode, dtype=dtype, **dims)
    m.zero_grads()
    m.begin_step()
    ids = g[p + "ids"]
    rows = ids.size // n
    logits = m.forward([ids[r * rows:(r + 1) * rows] for r in range(n)])
    dl = g[p + "dlogits"]
    m.backward([to_dev(dl[r * rows:(r + 1) * rows], dtype) for r in range(n)])
    grp.synchronize()
    out = {"logits": np.concatenate([to_np(t) for t in logits]),
           "grads": [np.stack([m.layer_shard(li, r, grad=True) for r in range(n)]) for li in range(m.layer_count())]}
    if moe:
        out["gate_grads"] = np.stack([np.stack([m.gate_grad(b, r) for r in range(n)]) for b in range(dims["layers"])])
    m.close()
    grp.close()
    return out


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
@pytest.mark.parametrize("mode", ["inplace", "outofplace"])
@pytest.mark.parametrize("n", [1, 2, 4])
def test_dense_model_matches_reference(golden, n, mode, dtype):
    g = golden("model")
    out = run_model(g, n, False, mode, dtype)
    p = f"dense_n{n}_"
    assert nerr(out["logits"], g[p + "logits"]) < TOL[dtype]
    for li, gr in enumerate(out["grads"]):
        for r in range(n):
            assert nerr(gr[r], g[p + f"grads{li}"][r]) < TOL[dtype], (li, r)


@pytest.mark.parametrize("n", [2, 4])
def test_moe_model_matches_reference(golden, n):
    """fp32 mode: the gate sees the model's residual stream, so routing is
    compared at the precision closest to the reference's fp64."""
    g = golden("model")
    out = run_model(g, n, True, "outofplace", "f32")
    p = f"moe_n{n}_"
    assert nerr(out["logits"], g[p + "logits"]) < TOL["f32"]
    for li, gr in enumerate(out["grads"]):
        for r in range(n):
            assert nerr(gr[r], g[p + f"grads{li}"][r]) < TOL["f32"], (li, r)
    for b in range(int(g["layers"])):
        for r in range(n):
            assert nerr(out["gate_grads"][b][r], g[p + "gate_grads"][b][r]) < TOL["f32"], (b, r)
