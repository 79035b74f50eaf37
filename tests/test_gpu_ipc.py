"""GPU: the distributed path for real — one PROCESS per worker on the IPC
transport (copy-engine ring shifts through CUDA IPC mappings, stream-memory-op
ordering; tests/ipc_worker.py), all processes sharing the box's GPU. Results
must equal the in-process Lockstep run bit for bit (same kernels, same order)
and the reference's golden outputs within the bf16 tolerance; ownership,
rotation order and the traffic log must be the reference's exactly."""
import os
import subprocess
import sys

import numpy as np
import pytest

from helpers import TOL, nerr, run_linear, run_mlp

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def spawn(case, n, mode, tmp_path, env=None):
    from paper_2311_01635_b200 import rtp
    uid = rtp.WorkerGroup.ipc_unique_id().hex()
    outs = [str(tmp_path / f"{case}_{mode}_{n}_{r}.npz") for r in range(n)]
    procs = [subprocess.Popen([sys.executable, os.path.join(ROOT, "tests", "ipc_worker.py"), case, str(n), str(r),
                               uid, mode, outs[r]], stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True,
                              env={**os.environ, **(env or {})})
             for r in range(n)]
    logs = []
    for p in procs:
        try:
            logs.append(p.communicate(timeout=240)[0])
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise
    for p, log in zip(procs, logs):
        assert p.returncode == 0, log[-3000:]
    return [dict(np.load(o)) for o in outs]


@pytest.mark.parametrize("mode", ["inplace", "outofplace"])
@pytest.mark.parametrize("n", [2, 4])
def test_linear_multiprocess_ipc(golden, tmp_path, n, mode):
    g = golden("linear")
    res = spawn("linear", n, mode, tmp_path)
    ref = run_linear(n, g["w"], g["b"], g["x"], g["dy"], "bf16", mode)  # in-process lockstep, same kernels
    y = np.concatenate([r["y"] for r in res])
    dx = np.concatenate([r["dx"] for r in res])
    assert np.array_equal(y, ref["y"]) and np.array_equal(dx, ref["dx"])
    for r in range(n):
        assert np.array_equal(res[r]["grad"], ref["grads"][r]), r
        assert np.array_equal(res[r]["weight"], ref["weights"][r]), r
    p = f"n{n}_oop{int(mode == 'outofplace')}_"
    assert nerr(y, g[p + "y"]) < TOL["bf16"] and nerr(dx, g[p + "dx"]) < TOL["bf16"]
    assert [int(r["fwd_id"]) for r in res] == list(g[p + "fwd_ids"])
    assert [int(r["bwd_id"]) for r in res] == list(g[p + "bwd_ids"])
    for r in range(n):
        fwd, bwd = res[r]["trace"]
        for s in range(n):  # each process records its own rank's column
            assert fwd[s][r] == (r - s) % n and bwd[s][r] == (r + 1 + s) % n
    # per-rank device memory measured in each process, exact bytes: W/N bf16,
    # G/N fp32, CommBuffer = out-of-place spare (W/N) + the staging chunk of
    # the in-place shifts (test_memory_ledger_exact_bytes' model)
    i_dim, o_dim = g["w"].shape
    L = i_dim * (o_dim // n) + o_dim // n
    chunk = min(max(1 << 20, (L * 4) // 32) + 255 & ~255, L * 4)
    for r in range(n):
        param, grad, comm = (int(v) for v in res[r]["ledger"])
        assert (param, grad) == (2 * L, 4 * L), r
        assert comm == (2 * L if mode == "outofplace" else 0) + chunk, (r, comm)
        assert [tuple(int(v) for v in t) for t in res[r]["traffic"]] == [tuple(int(v) for v in t)
                                                                          for t in g[p + "traffic"]]


@pytest.mark.parametrize("flags", ["0", "1"])
@pytest.mark.parametrize("n", [2, 4])
def test_mlp_multiprocess_ipc(golden, tmp_path, n, flags):
    """flags=1: the step GEMMs wait in-kernel on shard-arrival flags
    (RTPB_FLAGS) instead of stream events; same bits either way."""
    g = golden("mlp")
    res = spawn("mlp", n, "outofplace", tmp_path, env={"RTPB_FLAGS": flags})
    ref = run_mlp(n, g["w1"], g["b1"], g["w2"], g["b2"], g["x"], g["dy"], "bf16", "outofplace")
    y = np.concatenate([r["y"] for r in res])
    dx = np.concatenate([r["dx"] for r in res])
    assert np.array_equal(y, ref["y"]) and np.array_equal(dx, ref["dx"])
    for r in range(n):
        assert np.array_equal(res[r]["grad1"], ref["grads1"][r]) and np.array_equal(res[r]["grad2"], ref["grads2"][r])
    assert nerr(y, g[f"n{n}_y"]) < TOL["bf16"] and nerr(dx, g[f"n{n}_dx"]) < TOL["bf16"]


def test_mlp_multiprocess_ipc_dx_dw_side_by_side(golden, tmp_path):
    """One worker per GPU with dW on the aux stream beside dX (forced split of
    the SMs): the gradient shard's ordering moves from compute to aux."""
    g = golden("mlp")
    n = 2
    res = spawn("mlp", n, "outofplace", tmp_path, env={"RTPB_NWAY_DX_SMS": "74"})
    y = np.concatenate([r["y"] for r in res])
    dx = np.concatenate([r["dx"] for r in res])
    assert nerr(y, g[f"n{n}_y"]) < TOL["bf16"] and nerr(dx, g[f"n{n}_dx"]) < TOL["bf16"]
    for r in range(n):
        assert nerr(res[r]["grad1"], g[f"n{n}_grads1"][r]) < TOL["bf16"]
        assert nerr(res[r]["grad2"], g[f"n{n}_grads2"][r]) < TOL["bf16"]


@pytest.mark.parametrize("flags", ["0", "1"])
@pytest.mark.parametrize("chain", ["1", "0"])
def test_chained_stack_multiprocess_ipc(tmp_path, chain, flags):
    """A 3-block stack, two training steps, blocks chained (each block posts
    its neighbour's first shift under its own last step) or not: one process
    per worker equals the in-process run bit for bit, and chaining changes no
    bit (it only moves when shifts are posted). Two steps: flags=1 catches a
    stale arrival flag from the previous step."""
    from helpers import run_stack_local
    from paper_2311_01635_b200 import rtp
    n = 4
    res = spawn("stack", n, "outofplace", tmp_path, env={"RTPB_TEST_CHAIN": chain, "RTPB_FLAGS": flags})
    g = rtp.WorkerGroup(n, "lockstep")
    ref = run_stack_local(g, list(range(n)), n, chain=False)
    g.close()
    for r in range(n):
        for k, v in res[r].items():
            assert np.array_equal(v, ref[k]), (r, k)
        for b in range(3):
            assert list(res[r][f"home{b}_{r}"]) == [r, r]
