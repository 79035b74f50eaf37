"""GPU: pass launches (rtpb_fwd_pass / rtpb_dgrad_pass) — every rotation step
of one layer pass in one persistent launch — against the per-step launches
they replace (rtpb_fwd_step / rtpb_dgrad_step / rtpb_dgrad_step2), bit for
bit: same tiles, same K order, the fp32 dX accumulator summed in step order.
Also the count-in protocol the comm stream relies on (done[s] reaches the
announced target; the launch re-zeroes its counters and arrival flags)."""
import pytest
import torch

pytestmark = pytest.mark.gpu


def _setup(M, I, per, n, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    dev = "cuda"

    def u(*shape, scale=1.0):
        return ((torch.rand(*shape, generator=g, device=dev) * 2 - 1) * scale).to(torch.bfloat16)

    x = u(M, I)
    bufs = [u(I * per + per, scale=0.1), u(I * per + per, scale=0.1)]
    dy = u(M, n * per)
    r = 1 % n
    cols = [((r - s) % n) * per for s in range(n)]
    return x, bufs, dy, cols


def _counters(k=16):
    return torch.zeros(k, dtype=torch.int32, device="cuda")


@pytest.mark.parametrize("M,I,per,n", [(512, 256, 96, 4), (1000, 384, 128, 8), (2048, 768, 384, 2)])
@pytest.mark.parametrize("gelu", [False, True])
def test_fwd_pass_equals_per_step(M, I, per, n, gelu):
    from paper_2311_01635_b200 import rtp
    x, bufs, _, cols = _setup(M, I, per, n)
    y_ref = torch.zeros(M, n * per, dtype=torch.bfloat16, device="cuda")
    a_ref = torch.zeros_like(y_ref) if gelu else None
    for s in range(n):
        rtp.fwd_step(x, bufs[s & 1], y_ref, cols[s], per, act=a_ref)
    y = torch.zeros_like(y_ref)
    a = torch.zeros_like(y_ref) if gelu else None
    ready, done, ctr = _counters(), _counters(), _counters(1)
    ready[:n] = 1  # every shard already landed
    tgt = rtp.fwd_pass(x, bufs[0], bufs[1], y, cols, per, act=a, ready=ready, done=done, reset_ctr=ctr)
    torch.cuda.synchronize()
    assert torch.equal(y, y_ref)
    if gelu:
        assert torch.equal(a, a_ref)
    assert tgt == rtp.pass_done_target(0, M, I, per, n) and tgt > 0
    # the launch re-zeroed its count-ins, the pass's arrival flags and its CTA counter
    assert int(done.abs().sum()) == 0 and int(ready[:n].abs().sum()) == 0 and int(ctr.item()) == 0


def test_fwd_pass_counts_in_per_step():
    """Without a reset counter the count-ins stay: every step reaches the target."""
    from paper_2311_01635_b200 import rtp
    M, I, per, n = 640, 256, 64, 4
    x, bufs, _, cols = _setup(M, I, per, n)
    y = torch.zeros(M, n * per, dtype=torch.bfloat16, device="cuda")
    done = _counters()
    tgt = rtp.fwd_pass(x, bufs[0], bufs[1], y, cols, per, done=done)
    torch.cuda.synchronize()
    assert done[:n].tolist() == [tgt] * n and int(done[n:].abs().sum()) == 0


@pytest.mark.parametrize("M,I,per,n", [(512, 256, 96, 4), (1000, 384, 128, 8), (2048, 768, 384, 2),
                                       (768, 512, 64, 3)])
@pytest.mark.parametrize("gelu", [False, True])
def test_dgrad_pass_equals_per_step(M, I, per, n, gelu):
    from paper_2311_01635_b200 import rtp
    _, bufs, dy, cols = _setup(M, I, per, n, seed=1)
    pre = ((torch.rand(M, I, device="cuda") * 4 - 2).to(torch.bfloat16)) if gelu else None
    acc = torch.zeros(M, I, dtype=torch.float32, device="cuda")
    dx_ref = torch.zeros(M, I, dtype=torch.bfloat16, device="cuda")
    for s in range(n):
        rtp.dgrad_step(dy, cols[s], bufs[s & 1], acc, dx_ref, M, I, per, s == 0, s == n - 1,
                       pre=pre if s == n - 1 else None)
    dx = torch.zeros_like(dx_ref)
    acc2 = torch.zeros_like(acc)
    ready, done, ctr = _counters(), _counters(), _counters(1)
    ready[:n] = 1
    rtp.dgrad_pass(dy, bufs[0], bufs[1], cols, acc2, dx, I, per, pre=pre, ready=ready, done=done, reset_ctr=ctr)
    torch.cuda.synchronize()
    assert torch.equal(dx, dx_ref)
    assert int(done.abs().sum()) == 0 and int(ready[:n].abs().sum()) == 0


@pytest.mark.parametrize("M,I,per,n", [(512, 256, 96, 4), (1000, 384, 128, 8), (768, 512, 64, 3)])
@pytest.mark.parametrize("gelu", [False, True])
def test_dgrad_pass_paired_equals_step2(M, I, per, n, gelu):
    """Paired units (2g, 2g+1) = rtpb_dgrad_step2 over the same two shards; an
    odd last step runs alone."""
    from paper_2311_01635_b200 import _lib, rtp
    _, bufs, dy, cols = _setup(M, I, per, n, seed=2)
    pre = ((torch.rand(M, I, device="cuda") * 4 - 2).to(torch.bfloat16)) if gelu else None
    acc = torch.zeros(M, I, dtype=torch.float32, device="cuda")
    dx_ref = torch.zeros(M, I, dtype=torch.bfloat16, device="cuda")
    ws = torch.zeros(int(_lib.lib.rtpb_step_workspace_bytes(1, 0, M, I, per)), dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    groups = (n + 1) // 2
    for g_ in range(groups):
        first, last = g_ == 0, g_ == groups - 1
        flags = (_lib.EPI_FIRST if first else 0) | (_lib.EPI_LAST if last else 0) | \
            (_lib.EPI_GELU_BWD if (gelu and last) else 0)
        p = pre if (gelu and last) else None
        s0 = 2 * g_
        if s0 + 1 < n:
            rtp.check(_lib.lib.rtpb_dgrad_step2(0, dy.data_ptr(), dy.stride(0), cols[s0], bufs[0].data_ptr(),
                                                cols[s0 + 1], bufs[1].data_ptr(), acc.data_ptr(), I,
                                                dx_ref.data_ptr(), I, None if p is None else p.data_ptr(), I, M, I,
                                                per, flags, ws.data_ptr(), ws.numel(), st))
        else:
            rtp.dgrad_step(dy, cols[s0], bufs[0], acc, dx_ref, M, I, per, first, last, pre=p)
    dx = torch.zeros_like(dx_ref)
    acc2 = torch.zeros_like(acc)
    done = _counters()
    tgt = rtp.dgrad_pass(dy, bufs[0], bufs[1], cols, acc2, dx, I, per, pre=pre, pair=True, done=done)
    torch.cuda.synchronize()
    assert torch.equal(dx, dx_ref)
    assert done[:groups].tolist() == [tgt] * groups  # one count-in total per pair
    assert tgt == rtp.pass_done_target(1, M, I, per, n, (_lib.EPI_GELU_BWD if gelu else 0) | 128)


def _relay(done, ready, steps, target):
    """The comm stream's part of the dW pass protocol on a side stream: G(s+1)
    'lands' (ready[s+1] := 1) once step s has counted in (done[s] >= target).
    Queued before the launch, as the layers do (kernels preloaded)."""
    from cuda.bindings import driver as cu
    side = torch.cuda.Stream()
    h = side.cuda_stream
    for s in range(steps - 1):
        cu.cuStreamWaitValue32(h, done.data_ptr() + 4 * s, target, cu.CUstreamWaitValue_flags.CU_STREAM_WAIT_VALUE_GEQ)
        cu.cuStreamWriteValue32(h, ready.data_ptr() + 4 * (s + 1), 1, 0)
    return side


@pytest.mark.parametrize("M,I,per,n", [(1024, 256, 96, 4), (2048, 768, 384, 8), (512, 512, 64, 3)])
@pytest.mark.parametrize("zero", [True, False])
def test_wgrad_pass_matches_per_step(M, I, per, n, zero):
    """rtpb_wgrad_pass (every step's dW into one travelling shard, bias parts
    from rtpb_colsum) against n rtpb_wgrad_step calls, with the arrival
    protocol driven by a side stream as the comm stream drives it in a ring:
    the weight part bit for bit (same tiles and split-K at the same SM budget,
    steps in order), the bias part within fp32 rounding (dY's column sums are
    grouped differently from the fused per-step sums); count-ins reach the
    announced target and are re-zeroed with the flags."""
    from paper_2311_01635_b200 import _lib, rtp
    import ctypes as C
    x, _, dy, cols = _setup(M, I, per, n, seed=3)
    g_ref = torch.zeros(I * per + per, dtype=torch.float32, device="cuda")
    if not zero:
        g_ref.uniform_(-1, 1)
    g0 = g_ref.clone()
    for s in range(n):
        rtp.wgrad_step(x, dy, cols[s], None if (zero and s == 0) else g_ref, g_ref, per)
    g = g0.clone()
    ws = torch.zeros(int(_lib.lib.rtpb_step_workspace_bytes(2, 0, M, I, per)), dtype=torch.uint8, device="cuda")
    cws = torch.zeros(int(_lib.lib.rtpb_colsum_workspace_bytes(M, n * per)), dtype=torch.uint8, device="cuda")
    db = torch.zeros(n * per, dtype=torch.float32, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    rtp.check(_lib.lib.rtpb_colsum(dy.data_ptr(), dy.stride(0), M, n * per, db.data_ptr(), cws.data_ptr(), cws.numel(),
                                   st))
    ready, done, ctr = _counters(), _counters(), _counters(1)
    target = rtp.pass_done_target(2, M, I, per, n)
    _lib.lib.rtpb_preload_kernels()  # the relay's waits are queued before the launch
    torch.cuda.synchronize()
    side = _relay(done, ready, n, target)
    tgt = C.c_uint(0)
    rtp.check(_lib.lib.rtpb_wgrad_pass(x.data_ptr(), x.stride(0), dy.data_ptr(), dy.stride(0), n * per, g.data_ptr(),
                                       rtp._pass_cols(cols), n, M, I, per, _lib.EPI_FIRST if zero else 0,
                                       db.data_ptr(), ready.data_ptr(), done.data_ptr(), C.byref(tgt),
                                       ctr.data_ptr(), ws.data_ptr(), ws.numel(), st))
    side.synchronize()
    torch.cuda.synchronize()
    assert tgt.value == target
    assert torch.equal(g[:I * per], g_ref[:I * per])
    b_ref, b = g_ref[I * per:], g[I * per:]
    assert float((b - b_ref).abs().max()) / float(b_ref.abs().max()) < 1e-5
    assert int(done.abs().sum()) == 0 and int(ready[:n].abs().sum()) == 0


def test_pass_launch_refuses_a_different_announced_target():
    """A caller that queued its comm-stream waits for an announced count-in
    target gets an error, not a launch that would count to another value."""
    from paper_2311_01635_b200 import rtp
    M, I, per, n = 512, 256, 96, 4
    x, bufs, _, cols = _setup(M, I, per, n)
    y = torch.zeros(M, n * per, dtype=torch.bfloat16, device="cuda")
    right = rtp.pass_done_target(0, M, I, per, n)
    before = rtp.launch_count()
    with pytest.raises(rtp.StateError):
        rtp.fwd_pass(x, bufs[0], bufs[1], y, cols, per, announced_target=right + 1)
    assert rtp.launch_count() == before
    assert rtp.fwd_pass(x, bufs[0], bufs[1], y, cols, per, announced_target=right) == right
    torch.cuda.synchronize()


def test_pass_rejects_bad_geometry():
    from paper_2311_01635_b200 import rtp
    x, bufs, _, cols = _setup(256, 128, 48, 2)  # per not a multiple of 32
    y = torch.zeros(256, 96, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(rtp.ConfigError):
        rtp.fwd_pass(x, bufs[0], bufs[1], y, cols, 48)
    x, bufs, _, cols = _setup(256, 128, 64, 2)
    y = torch.zeros(256, 96, dtype=torch.bfloat16, device="cuda")  # narrower than the column blocks
    with pytest.raises(rtp.DimensionError):
        rtp.fwd_pass(x, bufs[0], bufs[1], y, cols, 64)


def _sim_run(n, tmp_path, tag, env):
    import os
    import subprocess
    import sys
    import numpy as np
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = str(tmp_path / f"sim_{tag}_{n}.npz")
    p = subprocess.run([sys.executable, os.path.join(root, "tests", "sim_worker.py"), str(n), out],
                       capture_output=True, text=True, timeout=300, env={**os.environ, **env})
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-3000:]
    return dict(np.load(out))


@pytest.mark.parametrize("n", [2, 4, 8])
def test_pass_protocol_simulated_ring_equals_per_step(n, tmp_path):
    """The whole protocol with real shard movement: n workers in one process
    (Lockstep, device copies), RTPB_SIM_FLAGS=1 sizing each worker's grids to
    its share of the SMs, so every pass launch, count-in wait, arrival flag,
    buffer alternation and the dW chain run as they would on n GPUs. A chained
    3-block stack (h=256, f=1024: every layer takes the pass launches), two
    training steps: every output, dX and gradient shard equals the per-step
    event-ordered run bit for bit."""
    import numpy as np
    ref = _sim_run(n, tmp_path, "ref", {"RTPB_FLAGS": "0"})
    got = _sim_run(n, tmp_path, "pass", {"RTPB_FLAGS": "1", "RTPB_SIM_FLAGS": "1"})
    assert ref.keys() == got.keys()
    for k in ref:
        if "grad" in k:
            # the dW pass launch runs on its SM share: its split-K (and the
            # bias sums' grouping) differ from the full-machine per-step dW,
            # so gradient shards agree to fp32 rounding, not bit for bit
            den = max(float(np.max(np.abs(ref[k]))), 1e-30)
            assert float(np.max(np.abs(ref[k] - got[k]))) / den < 1e-5, k
        else:
            assert np.array_equal(ref[k], got[k]), k
