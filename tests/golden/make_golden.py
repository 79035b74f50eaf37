"""Generate tests/golden/*.npz from the REFERENCE ITSELF.

Runs oracle/_ref/librtpref.so — the unmodified reference sources under
/root/reference/proj/src compiled by path (oracle/Makefile) behind the
extern "C" shim oracle/ref_shim.cpp — and stores small inputs and outputs.
tests/test_oracle.py pins our C restatement (oracle/rtp_oracle.c) to these
bit-for-bit; the GPU parity tests then compare the CUDA path to the oracle.

Inputs follow the reference's conventions: weights from
SplitMix64(seed) in SerialModel FFN order (serial.cpp:349-350) with
U[-0.1, 0.1]; activations X then dY from SplitMix64(seed ^ 0xA5A5A5A5A5A5A5A5)
(model.cpp:143) with U[-1, 1] (layers_test.cpp:90-91).

Usage: python tests/golden/make_golden.py   (needs /root/reference)
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from oracle import Reference, build_oracle  # noqa: E402

FIX = 0xA5A5A5A5A5A5A5A5


def acts(R, seed, rows, i_dim, o_dim):
    x = R.uniform(seed ^ FIX, 0, rows * i_dim, -1.0, 1.0).reshape(rows, i_dim)
    dy = R.uniform(seed ^ FIX, rows * i_dim, rows * o_dim, -1.0, 1.0).reshape(rows, o_dim)
    return x, dy


def main():
    build_oracle(with_ref=True)
    R = Reference()
    out = {}

    # 1. SplitMix64 uniform stream (rng.hpp:10-32, tensor.cpp:99-103)
    out["uniform"] = dict(seed42=R.uniform(42, 0, 4096, -0.1, 0.1),
                          seed7_skip1000=R.uniform(7, 1000, 512, -1.0, 1.0))

    # 2. Flyweight shards: shard_view(flatten_shards(linear_shard_groups)) for
    #    both FFN linears of a 2-block stack (block 1 tests the stream base).
    h, f, blocks, n = 32, 64, 2, 4
    p = R.mlp_params(42, h, f, blocks)
    fly = {"h": h, "f": f, "blocks": blocks, "n": n, "seed": 42}
    off = 0
    for blk in range(blocks):
        for name, (i_dim, o_dim) in (("ffn1", (h, f)), ("ffn2", (f, h))):
            w = p[off: off + i_dim * o_dim].reshape(i_dim, o_dim)
            b = p[off + i_dim * o_dim: off + i_dim * o_dim + o_dim]
            fly[f"b{blk}_{name}_base"] = off
            for j in range(n):
                fly[f"b{blk}_{name}_s{j}"] = R.linear_shard(w, b, n, j)
            off += i_dim * o_dim + o_dim
    out["flyweight"] = fly

    # 3. RtpLinear fwd+bwd (layers_linear.cpp:18-72), N in {1,2,4,8}, both
    #    rotation modes; plus SerialLinear (serial.cpp:59-77).
    rows, i_dim, o_dim = 64, 32, 64
    p = R.mlp_params(3, i_dim, o_dim, 1)
    w = p[: i_dim * o_dim].reshape(i_dim, o_dim)
    b = p[i_dim * o_dim: i_dim * o_dim + o_dim]
    x, dy = acts(R, 3, rows, i_dim, o_dim)
    lin = {"w": w, "b": b, "x": x, "dy": dy}
    s = R.serial_linear(w, b, x, dy)
    for k, v in s.items():
        lin[f"serial_{k}"] = v
    for nn in (1, 2, 4, 8):
        for oop in (0, 1):
            r = R.rtp_linear(nn, w, b, x, dy, outofplace=bool(oop))
            for k, v in r.items():
                lin[f"n{nn}_oop{oop}_{k}"] = v
    out["linear"] = lin

    # 4. MLP block (model.cpp:77-83, 99-105), N in {1,2,4,8}
    rows, h, f = 64, 32, 128
    p = R.mlp_params(42, h, f, 1)
    w1 = p[: h * f].reshape(h, f)
    b1 = p[h * f: h * f + f]
    w2 = p[h * f + f: h * f + f + f * h].reshape(f, h)
    b2 = p[h * f + f + f * h:]
    x, dy = acts(R, 42, rows, h, h)
    mlp = {"w1": w1, "b1": b1, "w2": w2, "b2": b2, "x": x, "dy": dy, "seed": 42}
    for nn in (1, 2, 4, 8):
        r = R.rtp_mlp(nn, w1, b1, w2, b2, x, dy)
        for k, v in r.items():
            mlp[f"n{nn}_{k}"] = v
    out["mlp"] = mlp

    # 4a. Ring self-check fixture for bench.py --gpus N (every N in {1,2,4,8}
    #     meets the device's 8-column shard constraint: per = 64/8 at N=8).
    #     The reference's in-place and out-of-place results are bitwise equal
    #     (layers_test.cpp:343-365; asserted here), so one set serves both.
    rows, h, f = 128, 64, 256
    p = R.mlp_params(42, h, f, 1)
    w1 = p[: h * f].reshape(h, f)
    b1 = p[h * f: h * f + f]
    w2 = p[h * f + f: h * f + f + f * h].reshape(f, h)
    b2 = p[h * f + f + f * h:]
    x, dy = acts(R, 42, rows, h, h)
    ring_mlp = {"w1": w1, "b1": b1, "w2": w2, "b2": b2, "x": x, "dy": dy, "seed": 42}
    for nn in (1, 2, 4, 8):
        r = R.rtp_mlp(nn, w1, b1, w2, b2, x, dy, outofplace=True)
        ri = R.rtp_mlp(nn, w1, b1, w2, b2, x, dy, outofplace=False)
        assert all(np.array_equal(r[k], ri[k]) for k in r), "out-of-place != in-place"
        for k, v in r.items():
            ring_mlp[f"n{nn}_{k}"] = v
    out["mlp_ring"] = ring_mlp

    # 4b. RtpAttention (layers_attention.cpp:43-198), heads split
    #     over N in {1,2,4}, sequences of 8, two per worker, both transports.
    #     Weights: one SplitMix64(42) stream, U[-0.1, 0.1], wq wk wv wo in order.
    H, heads, seq = 32, 4, 8
    wall = R.uniform(42, 0, 4 * H * H, -0.1, 0.1)
    att = {"heads": heads, "seq": seq, "seed": 42}
    for i, name in enumerate(("wq", "wk", "wv", "wo")):
        att[name] = wall[i * H * H:(i + 1) * H * H].reshape(H, H)
    for nn in (1, 2, 4):
        rows_a = nn * 2 * seq
        xa, dya = acts(R, 43 + nn, rows_a, H, H)
        att[f"n{nn}_x"], att[f"n{nn}_dy"] = xa, dya
        r = R.rtp_attention(nn, heads, seq, att["wq"], att["wk"], att["wv"], att["wo"], xa, dya)
        rc = R.rtp_attention(nn, heads, seq, att["wq"], att["wk"], att["wv"], att["wo"], xa, dya, concurrent=True)
        assert all(np.array_equal(r[k], rc[k]) for k in r), "lockstep != concurrent"
        for k, v in r.items():
            att[f"n{nn}_{k}"] = v
    out["attention"] = att

    # 4c. RtpMoe (layers_moe.cpp:18-198): top-1 gating over N
    #     experts that rotate past the batch. X (and dY) are bf16-representable
    #     values so a bf16 device run sees the reference's exact routing inputs.
    H, F = 32, 64
    moe = {"hidden": H, "ffn": F}
    import sys as _s
    _s.path.insert(0, os.path.join(ROOT, "tests"))
    from helpers import bf16_round
    for nn in (1, 2, 4):
        p = R.uniform(4242 + nn, 0, H * nn + nn * (2 * H * F + F + H), -0.1, 0.1)
        gate = p[:H * nn].reshape(H, nn)
        experts, off = [], H * nn
        for e in range(nn):
            w1 = p[off:off + H * F].reshape(H, F); off += H * F
            b1 = p[off:off + F]; off += F
            w2 = p[off:off + F * H].reshape(F, H); off += F * H
            b2 = p[off:off + H]; off += H
            experts.append((w1, b1, w2, b2))
        rows_m = nn * 16
        xm, dym = acts(R, 77 + nn, rows_m, H, H)
        xm, dym = bf16_round(xm), bf16_round(dym)
        r = R.rtp_moe(nn, gate, experts, xm, dym)
        rc = R.rtp_moe(nn, gate, experts, xm, dym, concurrent=True)
        assert all(np.array_equal(r[k], rc[k]) for k in r), "lockstep != concurrent"
        moe[f"n{nn}_gate"] = gate
        moe[f"n{nn}_experts"] = np.stack([np.concatenate([a.ravel() for a in e]) for e in experts])
        moe[f"n{nn}_x"], moe[f"n{nn}_dy"] = xm, dym
        for k, v in r.items():
            moe[f"n{nn}_{k}"] = v
    out["moe"] = moe

    # 4d. RtpEmbedding (layers_linear.cpp:74-136): table sharded on the
    #     embedding dimension, repeated ids (scatter-add order), N in {1,2,4}.
    vocab, emb, rpw = 64, 32, 16
    table = R.uniform(99, 0, vocab * emb, -0.1, 0.1).reshape(vocab, emb)
    embd = {"table": table}
    rng_ids = np.random.default_rng(5)
    for nn in (1, 2, 4):
        ids = rng_ids.integers(0, vocab, size=(nn, rpw)).astype(np.int64)
        ids[:, 1] = ids[:, 0]  # a repeated id on every worker
        dye = R.uniform(100 + nn, 0, nn * rpw * emb, -1, 1).reshape(nn * rpw, emb)
        r = R.rtp_embedding(nn, table, ids, dye)
        embd[f"n{nn}_ids"], embd[f"n{nn}_dy"] = ids, dye
        for k, v in r.items():
            embd[f"n{nn}_{k}"] = v
    out["embedding"] = embd

    # 4e. The whole RtpModel (model.cpp:7-121; SURVEY §8f.2 block wiring,
    #     §8f.4 embedding + head): SerialModel(dims, 42) parameters,
    #     make_batch_fixture ids, mse_grad upstream; dense N in {1,2,4} and
    #     MoE N in {2,4} (one expert per worker).
    model = {}
    dims = dict(heads=4, hidden=32, layers=2, seq=8, vocab=64, ffn=128)
    for moe_on, ns in ((False, (1, 2, 4)), (True, (2, 4))):
        for nn in ns:
            r = R.rtp_model(nn, dims["heads"], dims["hidden"], dims["layers"], dims["seq"], dims["vocab"],
                            dims["ffn"], moe=moe_on, seed=42, batch=4)
            ro = R.rtp_model(nn, dims["heads"], dims["hidden"], dims["layers"], dims["seq"], dims["vocab"],
                             dims["ffn"], moe=moe_on, seed=42, batch=4, outofplace=True)
            assert np.array_equal(r["logits"], ro["logits"]), "out-of-place != in-place"
            p = f"{'moe' if moe_on else 'dense'}_n{nn}_"
            model[p + "ids"], model[p + "logits"], model[p + "dlogits"] = r["ids"], r["logits"], r["dlogits"]
            for li, gr in enumerate(r["grads"]):
                model[p + f"grads{li}"] = gr
            if moe_on:
                model[p + "gate_grads"] = r["gate_grads"]
    model.update({k: np.int64(v) for k, v in dims.items()})
    out["model"] = model

    # 5. Ring primitive (ring.cpp:265-293) on id-encoded slots (ring_test.cpp:16-28)
    rng = np.random.default_rng(77)
    ring = {}
    for nn in (1, 2, 3, 4, 8):
        ops = rng.integers(0, 4, size=40).astype(np.int32)
        r = R.ring_ops(nn, ops.tolist(), length=6)
        ring[f"n{nn}_ops"] = ops
        for k, v in r.items():
            ring[f"n{nn}_{k}"] = v
    out["ring"] = ring

    # 6. Ledger peaks for one MLP step (analysis.cpp:236-333 style binding)
    led = {}
    for nn in (1, 2, 4, 8):
        for oop in (0, 1):
            r = R.mlp_ledger(nn, oop, 64, 32, 128)
            for k, v in r.items():
                led[f"n{nn}_oop{oop}_{k}"] = np.int64(v)
    # table1_memory RTP rows (analysis.cpp:45-46): strategy ids 5=Rtp, 6=RtpInplace
    for st in (5, 6):
        for N in (1, 2, 4, 8):
            led[f"table1_s{st}_N{N}"] = np.array(R.table1(st, 1000, 2000, 300, 40, N), np.int64)
    out["ledger"] = led

    # 7. The reference's report commands (commands.cpp:87-181) as CSV text:
    #    the schemas the device reports (paper_2311_01635_b200/reports.py) keep.
    import json
    reports = {}
    for which in ("memtable", "ledger", "sweep"):
        for nn in (2, 4):
            for strat in ("rtp-inplace", "rtp-outofplace"):
                reports[f"{which}_n{nn}_{strat}"] = R.cmd_csv(which, nn, strat, 8)
    with open(os.path.join(HERE, "reports.json"), "w") as fh:
        json.dump(reports, fh, indent=1, sort_keys=True)

    only = sys.argv[1:]  # e.g. `make_golden.py attention`: rewrite only those fixtures
    for name, d in out.items():
        if only and name not in only:
            continue
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **{k: np.asarray(v) for k, v in d.items()})
        print("wrote", name, len(d), "arrays")


if __name__ == "__main__":
    main()
