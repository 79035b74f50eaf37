"""RtpEmbedding and RtpMoe on the device (layers_linear.cpp:74-136,
layers_moe.cpp:18-198) against the reference's own layers
(tests/golden/embedding.npz, tests/golden/moe.npz, made by oracle/_ref):
bit-exact ownership / rotation order and routing-dependent outputs within the
north_star tolerances (normwise: bf16 2e-2, fp32 1e-5)."""
import numpy as np
import pytest

from helpers import TOL, dtype_round, nerr, to_dev, to_np

pytestmark = pytest.mark.gpu


def run_embedding(n, table, ids, dy, dtype="bf16", mode="inplace", transport="lockstep"):
    from paper_2311_01635_b200 import rtp
    g = rtp.WorkerGroup(n, transport)
    e = rtp.RtpEmbedding(g, "emb", table, dtype)
    e.set_rotation_mode(mode)
    if mode == "outofplace":
        e.allocate_comm_spares()
    e.zero_grads()
    ys = e.forward([ids[r] for r in range(n)])
    fwd_ids = [e.slot(r)["logical_id"] for r in range(n)]
    M = ids.shape[1]
    e.backward([to_dev(dy[r * M:(r + 1) * M], dtype) for r in range(n)])
    g.synchronize()
    out = {"y": np.concatenate([to_np(t) for t in ys]), "grads": np.stack([e.shard(r, True) for r in range(n)]),
           "weights": np.stack([e.shard(r) for r in range(n)]), "fwd_ids": fwd_ids,
           "bwd_ids": [e.slot(r)["logical_id"] for r in range(n)], "traffic": g.traffic()}
    e.close()
    g.close()
    return out


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
@pytest.mark.parametrize("mode", ["inplace", "outofplace"])
@pytest.mark.parametrize("n", [1, 2, 4])
def test_embedding_matches_reference(golden, n, mode, dtype):
    g = golden("embedding")
    table = g["table"]
    out = run_embedding(n, table, g[f"n{n}_ids"], g[f"n{n}_dy"], dtype, mode)
    # forward is a pure gather: exactly the reference's values in the layer dtype
    assert np.array_equal(out["y"], dtype_round(g[f"n{n}_y"], dtype))
    for r in range(n):
        assert nerr(out["grads"][r], g[f"n{n}_grads"][r]) < TOL[dtype], r
    assert out["fwd_ids"] == [(r + 1) % n for r in range(n)]
    assert out["bwd_ids"] == list(range(n))
    vocab, emb = table.shape
    per = emb // n
    for r in range(n):
        assert np.array_equal(out["weights"][r], dtype_round(table[:, r * per:(r + 1) * per].ravel(), dtype))
    assert [k for k, _, _ in out["traffic"]] == ["rotation_cw"] * (n - 1) + ["rotation_ccw"] * (n - 1)


def test_embedding_rejects_ids_outside_the_vocabulary(golden):
    from paper_2311_01635_b200 import rtp
    g = golden("embedding")
    grp = rtp.WorkerGroup(2)
    e = rtp.RtpEmbedding(grp, "emb", g["table"])
    with pytest.raises(rtp.IndexError_):
        e.forward([np.array([1, 2, 64]), np.array([0, 1, 2])])  # vocab 64
    with pytest.raises(rtp.IndexError_):
        e.forward([np.array([1, -1, 3]), np.array([0, 1, 2])])
    e.close()
    grp.close()


def run_moe(n, gate, experts, x, dy, dtype="bf16", mode="inplace", transport="lockstep"):
    from paper_2311_01635_b200 import rtp
    g = rtp.WorkerGroup(n, transport)
    m = rtp.RtpMoe(g, "moe", gate, experts, dtype)
    m.set_rotation_mode(mode)
    if mode == "outofplace":
        m.allocate_comm_spares()
    m.zero_grads()
    M = x.shape[0] // n
    ys = m.forward([to_dev(x[r * M:(r + 1) * M], dtype) for r in range(n)])
    fwd_ids = [m.slot(r)["logical_id"] for r in range(n)]
    dxs = m.backward([to_dev(dy[r * M:(r + 1) * M], dtype) for r in range(n)])
    g.synchronize()
    out = {"y": np.concatenate([to_np(t) for t in ys]), "dx": np.concatenate([to_np(t) for t in dxs]),
           "grads": np.stack([m.shard(r, True) for r in range(n)]),
           "gate_grads": np.stack([m.gate_grad(r) for r in range(n)]), "fwd_ids": fwd_ids,
           "bwd_ids": [m.slot(r)["logical_id"] for r in range(n)]}
    m.close()
    g.close()
    return out


def _experts(g, n):
    H, F = int(g["hidden"]), int(g["ffn"])
    out = []
    for e in g[f"n{n}_experts"]:
        w1 = e[:H * F].reshape(H, F)
        b1 = e[H * F:H * F + F]
        w2 = e[H * F + F:H * F + F + F * H].reshape(F, H)
        b2 = e[H * F + F + F * H:]
        out.append((w1, b1, w2, b2))
    return out


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
@pytest.mark.parametrize("mode", ["inplace", "outofplace"])
@pytest.mark.parametrize("n", [1, 2, 4])
def test_moe_matches_reference(golden, n, mode, dtype):
    g = golden("moe")
    out = run_moe(n, g[f"n{n}_gate"], _experts(g, n), g[f"n{n}_x"], g[f"n{n}_dy"], dtype, mode)
    assert nerr(out["y"], g[f"n{n}_y"]) < TOL[dtype]
    assert nerr(out["dx"], g[f"n{n}_dx"]) < TOL[dtype]
    for r in range(n):
        assert nerr(out["grads"][r], g[f"n{n}_grads"][r]) < TOL[dtype], r
        assert nerr(out["gate_grads"][r], g[f"n{n}_gate_grads"][r]) < TOL[dtype], r
    assert out["fwd_ids"] == [(r + 1) % n for r in range(n)]
    assert out["bwd_ids"] == list(range(n))


def test_moe_lockstep_equals_concurrent(golden):
    g = golden("moe")
    args = (4, g["n4_gate"], _experts(g, 4), g["n4_x"], g["n4_dy"], "bf16", "outofplace")
    a = run_moe(*args, transport="lockstep")
    b = run_moe(*args, transport="concurrent")
    for k in ("y", "dx", "grads", "gate_grads"):
        assert np.array_equal(a[k], b[k]), k


def test_moe_expert_count_must_equal_workers():
    from paper_2311_01635_b200 import rtp
    grp = rtp.WorkerGroup(2)
    H, F = 16, 32
    e = (np.zeros((H, F)), np.zeros(F), np.zeros((F, H)), np.zeros(H))
    with pytest.raises(rtp.ConfigError):
        rtp.RtpMoe(grp, "moe", np.zeros((H, 3)), [e, e, e])
    grp.close()
