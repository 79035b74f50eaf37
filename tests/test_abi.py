"""CPU: the C-ABI library loads, exports every symbol include/rtpb.h declares,
and its pure host logic (ring schedule, error mapping) behaves; the
multi-process ring protocol is checked with world_size-2 gloo."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "rtpb.h")


def declared_functions():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(rtpb_[a-z0-9_]+)\s*\(", txt)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("rtpb_fwd_step", "rtpb_dgrad_step", "rtpb_wgrad_step", "rtpb_flyweight_init",
                 "rtpb_group_create", "rtpb_group_create_nccl", "rtpb_linear_forward", "rtpb_linear_backward",
                 "rtpb_mlp_forward", "rtpb_mlp_backward", "rtpb_group_rotate", "rtpb_ring_plan"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2311_01635_b200 import _lib
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (rtpb_[a-z0-9_]+)", out))
    missing = [n for n in declared_functions() if n not in exported]
    assert not missing, missing
    # and the Python binding declares a signature for each of them
    assert not [n for n in declared_functions() if n not in _lib._SIGS]


def test_library_is_sm100a_and_uses_tcgen05_and_tma():
    from paper_2311_01635_b200 import _lib
    out = subprocess.run(["cuobjdump", "-lelf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass or "UTCQMMA" in sass  # tcgen05.mma kind::f16 / tf32
    assert "UTMALDG" in sass  # TMA tensor loads
    assert "LDTM" in sass  # tcgen05.ld (TMEM -> registers)


def test_ring_plan_position_laws():
    from paper_2311_01635_b200 import _lib
    L = _lib.lib
    for n in (1, 2, 3, 4, 8):
        for r in range(n):
            for s in range(n):
                lid, snd, rcv = C.c_int64(), C.c_int64(), C.c_int64()
                _lib.check(L.rtpb_ring_plan(n, r, 0, s, C.byref(lid), C.byref(snd), C.byref(rcv)))
                assert lid.value == (r - s) % n
                assert (snd.value, rcv.value) == (((r + 1) % n, (r - 1) % n) if s + 1 < n else (-1, -1))
                _lib.check(L.rtpb_ring_plan(n, r, 1, s, C.byref(lid), C.byref(snd), C.byref(rcv)))
                assert lid.value == (r + 1 + s) % n
                assert (snd.value, rcv.value) == (((r - 1) % n, (r + 1) % n) if s + 1 < n else (-1, -1))
    with pytest.raises(_lib.ConfigError):
        _lib.check(L.rtpb_ring_plan(4, 4, 0, 0, None, None, None))


def test_step_workspace_sizes():
    from paper_2311_01635_b200 import _lib
    L = _lib.lib
    # one layout for all step kinds: [bias-grad tickets + partials][fp32 splits]
    sizes = [L.rtpb_step_workspace_bytes(w, _lib.BF16, 1024, 768, 3072) for w in range(3)]
    assert sizes[0] == sizes[1] == sizes[2] > 0
    assert L.rtpb_step_workspace_bytes(0, _lib.F32, 1024, 768, 3072) >= 2 * 4 * (1024 * 768 + 768 * 3072)


def test_step_entry_validates_before_touching_the_device():
    from paper_2311_01635_b200 import _lib
    L = _lib.lib
    rc = L.rtpb_fwd_step(_lib.BF16, None, 12, None, None, 4, 0, None, 0, 16, 12, 4, _lib.EPI_STORE_PRE, None, 0,
                         None)
    assert rc == _lib.ConfigError.code
    assert "multiple" in L.rtpb_last_error().decode()


def test_group_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2311_01635_b200 import rtp
    with pytest.raises(rtp.RtpError):
        rtp.WorkerGroup(2)


def _gloo_worker(rank, world, port, q):
    import torch.distributed as dist
    try:
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        import torch
        from paper_2311_01635_b200 import _lib, rtp
        # 1. NCCL bootstrap id: rank 0 creates it, the group broadcasts it
        uid = torch.zeros(128, dtype=torch.uint8)
        if rank == 0:
            uid = torch.frombuffer(bytearray(rtp.WorkerGroup.nccl_unique_id()), dtype=torch.uint8).clone()
        dist.broadcast(uid, src=0)
        ids = [torch.zeros(128, dtype=torch.uint8) for _ in range(world)]
        dist.all_gather(ids, uid)
        assert all(torch.equal(ids[0], t) for t in ids)
        # 2. SPMD ring protocol: every process derives its own schedule from
        # rtpb_ring_plan; the shard id it sends must be the one its receiver
        # expects at the next step (what NcclTransport's bookkeeping assumes).
        L = _lib.lib
        for phase in (0, 1):
            for s in range(world):
                lid, snd, rcv = C.c_int64(), C.c_int64(), C.c_int64()
                _lib.check(L.rtpb_ring_plan(world, rank, phase, s, C.byref(lid), C.byref(snd), C.byref(rcv)))
                if snd.value < 0:
                    continue
                out = torch.tensor([lid.value], dtype=torch.int64)
                inc = torch.zeros(1, dtype=torch.int64)
                reqs = [dist.isend(out, snd.value), dist.irecv(inc, rcv.value)]
                for r_ in reqs:
                    r_.wait()
                nxt = C.c_int64()
                _lib.check(L.rtpb_ring_plan(world, rank, phase, s + 1, C.byref(nxt), None, None))
                assert inc.item() == nxt.value, (phase, s, inc.item(), nxt.value)
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # noqa
        q.put((rank, repr(e)))


def test_two_process_gloo_ring_protocol():
    import random

    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = random.randint(20000, 40000)
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(res) == [(0, "ok"), (1, "ok")], res


def test_fused_n1_schedules_cover_the_config_shapes():
    """Host-side list scheduling of the fused N = 1 MLP launches (no GPU):
    every BASELINE config shape gets a plan with a finite cost-model makespan."""
    import math
    from paper_2311_01635_b200 import _lib
    for M, h, f in ((8192, 768, 3072), (16384, 4096, 16384), (4096, 8192, 28672), (1000, 768, 3072), (8, 8, 16)):
        for which in (0, 1):
            t = _lib.lib.rtpb_debug_fused_plan(M, h, f, which)
            assert t > 0 and math.isfinite(t), (M, h, f, which)


def test_every_gemm_instantiation_is_preloaded():
    """preload_device_kernels sets every step-GEMM instantiation's shared-memory
    opt-in up front (a lazy attribute set may wait for running instances of the
    kernel, which deadlocks against grids spinning on later launches): the
    list in gemm_launch.cu must cover every instantiation the library holds."""
    import os
    from paper_2311_01635_b200 import _lib
    out = subprocess.run(["nm", "-C", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    out += subprocess.run(["nm", "-C", _lib.LIB_PATH], capture_output=True, text=True).stdout
    inst = set(re.findall(r"rtp_gemm_kernel<rtpb::GemmCfg<([^>]*)>", out))
    src = open(os.path.join(os.path.dirname(HEADER), "..", "paper_2311_01635_b200", "csrc", "kernels",
                            "gemm_launch.cu")).read()
    listed = set(re.findall(r"set_smem_attr<GemmCfg<([^>]*)>>\(\);", src))
    norm = lambda s: ",".join(p.strip() for p in s.replace("(int)", "").replace("(bool)", "").split(","))  # noqa: E731
    assert inst, "no instantiations found"
    missing = {norm(i) for i in inst} - {norm(i) for i in listed}
    assert not missing, missing
