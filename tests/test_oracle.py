"""CPU: pin the C restatement (oracle/rtp_oracle.c) to the reference's own
outputs (tests/golden/*.npz, produced from the reference sources by
tests/golden/make_golden.py). Everything here must be bit-exact."""
import numpy as np
import pytest


def test_uniform_stream_matches_reference(golden, oracle):
    g = golden("uniform")
    assert np.array_equal(oracle.uniform(42, 0, 4096, -0.1, 0.1), g["seed42"])
    assert np.array_equal(oracle.uniform(7, 1000, 512, -1.0, 1.0), g["seed7_skip1000"])


def test_splitmix_counter_form_matches_sequential_stream(oracle):
    # rng.hpp:16-22: state += gamma before mixing, so draw k uses seed + (k+1)*gamma
    seed = 12345
    state = seed
    mask = (1 << 64) - 1
    for k in range(64):
        state = (state + 0x9E3779B97F4A7C15) & mask
        z = state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & mask
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & mask
        z = z ^ (z >> 31)
        assert oracle.splitmix_at(seed, k) == z


def test_flyweight_closed_form_matches_shard_view(golden, oracle):
    g = golden("flyweight")
    h, f, blocks, n, seed = (int(g[k]) for k in ("h", "f", "blocks", "n", "seed"))
    for b in range(blocks):
        for name, (i_dim, o_dim) in (("ffn1", (h, f)), ("ffn2", (f, h))):
            base = int(g[f"b{b}_{name}_base"])
            for j in range(n):
                got = oracle.linear_shard(seed, base, i_dim, o_dim, n, j)
                assert np.array_equal(got, g[f"b{b}_{name}_s{j}"]), (b, name, j)


@pytest.mark.parametrize("n", [1, 2, 4, 8])
def test_rtp_linear_matches_reference_bitwise(golden, oracle, n):
    g = golden("linear")
    r = oracle.rtp_linear(n, g["w"], g["b"], g["x"], g["dy"], trace=True)
    for oop in (0, 1):  # the reference's out-of-place mode is bitwise the in-place one
        p = f"n{n}_oop{oop}_"
        assert np.array_equal(r["y"], g[p + "y"])
        assert np.array_equal(r["dx"], g[p + "dx"])
        assert np.array_equal(r["grads"], g[p + "grads"])
        # forward ends with rank r holding shard r+1; backward re-homes
        assert list(r["fwd_ids"][-1]) == list(g[p + "fwd_ids"])
        assert list(r["bwd_ids"][-1]) == [(rk + 1 + n - 1) % n for rk in range(n)]
        assert list(g[p + "bwd_ids"]) == list(range(n))


@pytest.mark.parametrize("n", [1, 2, 4, 8])
def test_position_laws(oracle, golden, n):
    g = golden("linear")
    r = oracle.rtp_linear(n, g["w"], g["b"], g["x"], g["dy"], trace=True)
    for s in range(n):
        for rk in range(n):
            assert r["fwd_ids"][s, rk] == (rk - s) % n  # layers_common.cpp:135-142
            assert r["bwd_ids"][s, rk] == (rk + 1 + s) % n  # layers_common.cpp:144-151


def test_rtp_linear_n1_equals_serial(golden):
    g = golden("linear")
    assert np.array_equal(g["n1_oop0_y"], g["serial_y"])  # layers_test.cpp:27-40
    assert np.array_equal(g["n1_oop0_dx"], g["serial_dx"])


def test_traffic_records(golden):
    g = golden("linear")
    i_dim, o_dim = g["w"].shape
    for n in (2, 4, 8):
        per = o_dim // n
        L = i_dim * per + per
        t = g[f"n{n}_oop0_traffic"]
        assert [tuple(x) for x in t] == [(0, L, 0)] * (n - 1) + [(1, L, L)] * (n - 1)
    assert len(g["n1_oop0_traffic"]) == 0


@pytest.mark.parametrize("n", [1, 2, 4, 8])
def test_rtp_mlp_matches_reference_bitwise(golden, oracle, n):
    g = golden("mlp")
    r = oracle.rtp_mlp(n, g["w1"], g["b1"], g["w2"], g["b2"], g["x"], g["dy"])
    for k in ("y", "dx", "grads1", "grads2"):
        assert np.array_equal(r[k], g[f"n{n}_{k}"]), k


@pytest.mark.parametrize("n", [1, 2, 4])
def test_rtp_attention_matches_reference_bitwise(golden, oracle, n):
    """SURVEY §8f.2 groundwork: the C restatement of RtpAttention (head
    partition, per-(sequence, head) softmax attention, output projection
    accumulated over the rotation, the tape, W+G backward rotation) reproduces
    the reference's outputs and gradient shards bit for bit."""
    g = golden("attention")
    r = oracle.rtp_attention(n, int(g["heads"]), int(g["seq"]), g["wq"], g["wk"], g["wv"], g["wo"],
                             g[f"n{n}_x"], g[f"n{n}_dy"])
    for k in ("y", "dx", "grads"):
        assert np.array_equal(r[k], g[f"n{n}_{k}"]), k


def test_gelu_matches_reference_values(oracle):
    # tensor_test.cpp:371-393 style: exact erf form and derivative by central differences
    x = np.linspace(-4, 4, 101)
    y = oracle.gelu(x)
    from math import erf, sqrt
    ref = np.array([v * 0.5 * (1 + erf(v / sqrt(2))) for v in x])
    assert np.max(np.abs(y - ref)) < 1e-15
    d = oracle.gelu_backward(x, np.ones_like(x))
    h = 1e-6
    fd = (oracle.gelu(x + h) - oracle.gelu(x - h)) / (2 * h)
    assert np.max(np.abs(d - fd)) < 1e-8


def _ring_model(n, ops):
    """Pure-python model of WorkerGroup rotations (ring.cpp:265-293) on
    id-encoded slots (ring_test.cpp:16-28)."""
    ids = list(range(n))
    offs = [0] * n
    w0 = [r * 100.0 for r in range(n)]
    g0 = [float(r) for r in range(n)]
    if n == 1:
        return ids, offs, w0, g0
    for op in ops:
        cw = op in (0, 2)
        grad = op in (1, 2)
        src = [(r - 1) % n if cw else (r + 1) % n for r in range(n)]
        ids = [ids[src[r]] for r in range(n)]
        offs = [offs[src[r]] + (1 if cw else -1) for r in range(n)]
        w0 = [w0[src[r]] for r in range(n)]
        if grad:
            g0 = [g0[src[r]] for r in range(n)]
    return ids, offs, w0, g0


@pytest.mark.parametrize("n", [1, 2, 3, 4, 8])
def test_ring_model_matches_reference(golden, n):
    g = golden("ring")
    ids, offs, w0, g0 = _ring_model(n, g[f"n{n}_ops"].tolist())
    assert ids == g[f"n{n}_ids"].tolist()
    assert offs == g[f"n{n}_offsets"].tolist()
    assert w0 == g[f"n{n}_w0"].tolist()
    assert g0 == g[f"n{n}_g0"].tolist()


def test_memory_model_rows(golden, oracle):
    g = golden("ledger")
    # table1_memory RTP rows (analysis.cpp:45-46): param_mem column
    for N in (1, 2, 4, 8):
        W, G = 1000, 2000
        oop = g[f"table1_s5_N{N}"]
        inp = g[f"table1_s6_N{N}"]
        assert int(inp[1]) == W + G
        assert int(oop[1]) == (W + G + (max(W, G) if N > 1 else 0))
        assert oracle.rtp_memory(W, G, N, False) * N == (W + G) * (1 if N > 1 else N)
    # instrumented ledger peaks of one MLP step (analysis_test.cpp:151-194 pattern)
    for n in (2, 4, 8):
        fpb = int(g[f"n{n}_oop0_flat_param_bytes"])
        assert int(g[f"n{n}_oop0_param"]) == fpb // n
        assert int(g[f"n{n}_oop0_grad"]) == fpb // n
        assert int(g[f"n{n}_oop0_comm"]) == 0
        assert int(g[f"n{n}_oop1_comm"]) == fpb // n  # one spare per layer, model-wide
