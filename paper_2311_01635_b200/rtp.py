"""Python mirror of the reference's RTP layer API over librtpb.so.

Same names and argument meaning as proj/include/rtp (WorkerGroup ring.hpp:65,
RtpLinear layers.hpp:129, the ffn1->gelu->ffn2 block of model.cpp:77-105),
with activations as CUDA torch tensors (one per local worker). torch is only
plumbing here: device memory and stream interop. All compute and all ring
transfers run in the native library; there is no fallback.

Errors raise the reference's exception classes (ConfigError, DimensionError,
ProtocolError, StateError, IndexError_) mapped from the C status codes.
"""
from __future__ import annotations

import ctypes as C

import torch

from . import _lib
from ._lib import (BF16, F32, ConfigError, DimensionError, IndexError_, ProtocolError, RtpError,  # noqa: F401
                   StateError, check, lib, ptr_array)

_DT = {"bf16": BF16, "f32": F32, BF16: BF16, F32: F32}
_TORCH_DT = {BF16: torch.bfloat16, F32: torch.float32}
_TRANSPORT = {"lockstep": _lib.TRANSPORT_LOCKSTEP, "concurrent": _lib.TRANSPORT_CONCURRENT}
MEM_CATEGORIES = ("param", "grad", "activation", "comm", "other")
_OPTIONS = {"exact_gelu": 1, "paired_dx": 2}


class WorkerGroup:
    """WorkerGroup(n, transport) (ring.hpp:65-125) with device workers.

    transport: "lockstep" | "concurrent" (all n workers in this process,
    ``devices[r]`` hosting worker r; default all on the current device), or use
    ``WorkerGroup.nccl(n, rank, device, unique_id)`` for one process per GPU.
    """

    def __init__(self, n: int, transport: str = "lockstep", devices=None, _handle=None):
        self.n = n
        if _handle is not None:
            self._h = _handle
        else:
            h = C.c_void_p()
            devs = None
            if devices is not None:
                if len(devices) != n:
                    raise ConfigError(f"device list size {len(devices)} does not match {n} workers")
                devs = (C.c_int * n)(*devices)
            check(lib.rtpb_group_create(n, _TRANSPORT[transport], devs, C.byref(h)))
            self._h = h
        cnt = lib.rtpb_group_local_ranks(self._h, None)
        arr = (C.c_size_t * max(1, cnt))()
        lib.rtpb_group_local_ranks(self._h, arr)
        self.local_ranks = [int(arr[i]) for i in range(cnt)]
        self._streams = {}

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        check(lib.rtpb_nccl_unique_id(buf))
        return buf.raw

    @classmethod
    def nccl(cls, n: int, rank: int, device: int, unique_id: bytes) -> "WorkerGroup":
        h = C.c_void_p()
        buf = C.create_string_buffer(bytes(unique_id), 128)
        check(lib.rtpb_group_create_nccl(n, rank, device, buf, C.byref(h)))
        return cls(n, _handle=h)

    @staticmethod
    def ipc_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        check(lib.rtpb_ipc_unique_id(buf))
        return buf.raw

    @classmethod
    def ipc(cls, n: int, rank: int, device: int, unique_id: bytes) -> "WorkerGroup":
        """One process per worker, copy-engine ring shifts through CUDA IPC
        (processes on one node; workers may share a GPU)."""
        h = C.c_void_p()
        buf = C.create_string_buffer(bytes(unique_id), 128)
        check(lib.rtpb_group_create_ipc(n, rank, device, buf, C.byref(h)))
        return cls(n, _handle=h)

    @classmethod
    def solo(cls, n: int, rank: int = 0, device: int = 0) -> "WorkerGroup":
        """Measurement: rank `rank` of an n-worker ring, no peers, shifts skipped."""
        h = C.c_void_p()
        check(lib.rtpb_group_create_solo(n, rank, device, C.byref(h)))
        return cls(n, _handle=h)

    def size(self) -> int:
        return self.n

    def device_of(self, rank: int) -> torch.device:
        s = self.stream(rank)
        return s.device

    def stream(self, rank: int, comm: bool = False) -> torch.cuda.ExternalStream:
        key = (rank, comm)
        if key not in self._streams:
            p = lib.rtpb_group_stream(self._h, rank, int(comm))
            if not p:
                raise _lib.IndexError_(f"worker {rank} is not hosted by this process")
            # The stream was created on the worker's device; torch needs the device.
            self._streams[key] = torch.cuda.ExternalStream(p, device=self._dev_guess(rank))
        return self._streams[key]

    def _dev_guess(self, rank):
        return torch.device("cuda", int(lib.rtpb_group_device(self._h, rank)))

    def synchronize(self):
        check(lib.rtpb_group_synchronize(self._h))

    def traffic(self):
        cnt = lib.rtpb_group_traffic(self._h, None, None, None, 0)
        k = (C.c_int64 * max(1, cnt))()
        w = (C.c_int64 * max(1, cnt))()
        g = (C.c_int64 * max(1, cnt))()
        lib.rtpb_group_traffic(self._h, k, w, g, cnt)
        names = {0: "rotation_cw", 1: "rotation_ccw", 2: "allgather"}
        return [(names[k[i]], int(w[i]), int(g[i])) for i in range(cnt)]

    def clear_traffic(self):
        lib.rtpb_group_clear_traffic(self._h)

    def corrupt_next_exchange(self, rank: int, what: str):
        check(lib.rtpb_group_corrupt_next_exchange(self._h, rank, {"tag": 1, "shard_id": 2}[what]))

    def ledger(self, rank: int) -> dict:
        cur = (C.c_size_t * 5)()
        peak = (C.c_size_t * 5)()
        tot = C.c_size_t()
        check(lib.rtpb_group_ledger(self._h, rank, cur, peak, C.byref(tot)))
        out = {f"current_{c}": int(cur[i]) for i, c in enumerate(MEM_CATEGORIES)}
        out.update({f"peak_{c}": int(peak[i]) for i, c in enumerate(MEM_CATEGORIES)})
        out["peak_total"] = int(tot.value)
        return out

    def reset_ledger_peaks(self):
        check(lib.rtpb_group_reset_ledger_peaks(self._h))

    # ---- stream interop: our streams <-> torch's current stream ----
    # Every call makes the worker streams wait for torch's current stream on
    # entry and torch's current stream wait for them on exit, so torch's
    # caching allocator can only reuse a caller tensor's memory after the
    # library is done with it (no record_stream on library-owned streams,
    # which may be destroyed before the tensors are freed).
    def _enter(self, tensors_per_rank):
        for r in self.local_ranks:
            s = self.stream(r)
            s.wait_stream(torch.cuda.current_stream(s.device))

    def _leave(self):
        for r in self.local_ranks:
            s = self.stream(r)
            torch.cuda.current_stream(s.device).wait_stream(s)

    def rotate(self, op: str, weights, grads=None, spares=None, w_bytes=None, g_bytes=None, keep_spare=False):
        """Ring primitive on raw per-rank device buffers (ring.cpp:265-333).
        op: "cw" (W), "ccw" (W+G), "cw_wg", "ccw_w". With spares (out of
        place) and keep_spare=True the received shard stays in spares[k]."""
        code = {"cw": 0, "ccw": 1, "cw_wg": 2, "ccw_w": 3}[op] | (8 if keep_spare else 0)
        self._enter([[w] + ([grads[k]] if grads else []) + ([spares[k]] if spares else [])
                     for k, w in enumerate(weights)])
        wb = w_bytes if w_bytes is not None else weights[0].numel() * weights[0].element_size()
        gb = g_bytes if g_bytes is not None else (grads[0].numel() * grads[0].element_size() if grads else 0)
        check(lib.rtpb_group_rotate(self._h, code, ptr_array(weights), ptr_array(grads) if grads else None,
                                    ptr_array(spares) if spares else None, wb, gb))
        self._leave()

    def allgather(self, shards, out):
        self._enter([[a, b] for a, b in zip(shards, out)])
        check(lib.rtpb_group_allgather(self._h, ptr_array(shards), ptr_array(out),
                                       shards[0].numel() * shards[0].element_size()))
        self._leave()

    def close(self):
        if getattr(self, "_h", None):
            lib.rtpb_group_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _as_host_f64(a):
    import numpy as np
    if a is None:
        return None
    if isinstance(a, torch.Tensor):
        a = a.detach().cpu().double().numpy()
    return np.ascontiguousarray(a, dtype=np.float64)


class _Layer:
    dtype_code: int
    group: WorkerGroup

    def _acts(self, rows, cols, like=None):
        out = []
        for r in self.group.local_ranks:
            dev = self.group.stream(r).device
            out.append(torch.empty(rows, cols, dtype=_TORCH_DT[self.dtype_code], device=dev))
        return out

    def _check_inputs(self, xs, cols):
        if len(xs) != len(self.group.local_ranks):
            raise DimensionError(f"expected {len(self.group.local_ranks)} activations (one per local worker)")
        rows = xs[0].shape[0]
        for x in xs:
            if x.dim() != 2 or x.shape[0] != rows or x.shape[1] != cols:
                raise DimensionError(f"activation of shape {tuple(x.shape)} does not match ({rows}, {cols})")
            if x.dtype != _TORCH_DT[self.dtype_code] or not x.is_cuda or not x.is_contiguous():
                raise DimensionError("activations must be contiguous CUDA tensors of the layer dtype")
        return rows


class RtpLinear(_Layer):
    """RtpLinear(group, label, weight, bias, n) (layers_linear.cpp:6-16).

    weight (in x out) / bias (out): host fp64 (numpy or torch) as in the
    reference, or None for Flyweight initialisation from (seed, stream_base).
    """

    def __init__(self, group: WorkerGroup, label: str, in_dim: int, out_dim: int, dtype="bf16", weight=None,
                 bias=None, seed: int = 42, stream_base: int = 0, _handle=None):
        self.group, self.label = group, label
        self.in_dim, self.out_dim = in_dim, out_dim
        self.dtype_code = _DT[dtype]
        self._owned = _handle is None
        if _handle is not None:
            self._h = _handle
            return
        w, b = _as_host_f64(weight), _as_host_f64(bias)
        if w is not None and w.shape != (in_dim, out_dim):
            raise DimensionError(f"weight shape {w.shape} does not match ({in_dim}, {out_dim})")
        h = C.c_void_p()
        check(lib.rtpb_linear_create(group._h, label.encode(), in_dim, out_dim, self.dtype_code,
                                     None if w is None else w.ctypes.data, None if b is None else b.ctypes.data,
                                     seed, stream_base, C.byref(h)))
        self._h = h

    def n(self):
        return self.group.n

    def shard_len(self) -> int:
        return int(lib.rtpb_linear_shard_len(self._h))

    def set_rotation_mode(self, mode: str):
        check(lib.rtpb_linear_set_rotation_mode(self._h, {"inplace": 0, "outofplace": 1}[mode]))

    def allocate_comm_spares(self):
        check(lib.rtpb_linear_allocate_comm_spares(self._h))

    def set_option(self, name: str, value: bool):
        """"exact_gelu" (bf16 epilogues: exact-erf GELU instead of tanh.approx)
        or "paired_dx" (out-of-place: two steps' dX in one GEMM; off restores
        the reference's per-step sums, out-of-place == in-place bitwise)."""
        check(lib.rtpb_linear_set_option(self._h, _OPTIONS[name], int(bool(value))))

    def release_comm_spares(self):
        check(lib.rtpb_linear_release_comm_spares(self._h))

    def zero_grads(self):
        check(lib.rtpb_linear_zero_grads(self._h))

    def forward(self, xs, mode: str = "train", out=None):
        rows = self._check_inputs(xs, self.in_dim)
        ys = out if out is not None else self._acts(rows, self.out_dim)
        self.group._enter([[x, y] for x, y in zip(xs, ys)])
        check(lib.rtpb_linear_forward(self._h, ptr_array(xs), rows, ptr_array(ys),
                                      _lib.MODE_EVAL if mode == "eval" else _lib.MODE_TRAIN))
        self.group._leave()
        if mode != "eval":
            self._x_keep = list(xs)  # the layer reads X again in backward (x_cache_)
        return ys

    def backward(self, dys, out=None):
        rows = self._check_inputs(dys, self.out_dim)
        dxs = out if out is not None else self._acts(rows, self.in_dim)
        self.group._enter([[a, b] for a, b in zip(dys, dxs)])
        check(lib.rtpb_linear_backward(self._h, ptr_array(dys), rows, ptr_array(dxs)))
        self.group._leave()
        self._x_keep = None
        return dxs

    def slot(self, rank: int) -> dict:
        lid, off = C.c_int64(), C.c_int64()
        w, g = C.c_void_p(), C.c_void_p()
        check(lib.rtpb_linear_slot(self._h, rank, C.byref(lid), C.byref(off), C.byref(w), C.byref(g)))
        return {"logical_id": lid.value, "rotation_offset": off.value, "weight_ptr": w.value, "grad_ptr": g.value}

    def _read(self, rank: int, which: int, dtype) -> torch.Tensor:
        t = torch.empty(self.shard_len(), dtype=dtype, device=self.group.stream(rank).device)
        torch.cuda.synchronize(t.device)
        check(lib.rtpb_linear_read_shard(self._h, rank, which, t.data_ptr()))
        return t

    def weight_shard(self, rank: int) -> torch.Tensor:
        """Copy of the weight shard resident at `rank` ([W_j | b_j], layer dtype)."""
        return self._read(rank, 0, _TORCH_DT[self.dtype_code])

    def grad_shard(self, rank: int) -> torch.Tensor:
        """Copy of the gradient accumulator resident at `rank` (fp32)."""
        return self._read(rank, 1, torch.float32)

    def trace(self):
        n = self.group.n
        arr = (C.c_int64 * (2 * n * n))()
        check(lib.rtpb_linear_trace(self._h, arr))
        vals = list(arr)
        return ([vals[s * n:(s + 1) * n] for s in range(n)],
                [vals[n * n + s * n: n * n + (s + 1) * n] for s in range(n)])

    def close(self):
        if self._owned and getattr(self, "_h", None):
            lib.rtpb_linear_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class RtpMlp(_Layer):
    """ffn1 (h->f) -> gelu -> ffn2 (f->h) as RtpModel composes it
    (model.cpp:77-83 forward, 99-105 backward), GELU fused into the step
    epilogues. Parameters: host fp64 (w1 h x f, b1 f, w2 f x h, b2 h) or all
    None for Flyweight init (ffn1 from stream_base, ffn2 after it)."""

    def __init__(self, group: WorkerGroup, label: str, h: int, f: int, dtype="bf16", w1=None, b1=None, w2=None,
                 b2=None, seed: int = 42, stream_base: int = 0):
        self.group, self.label, self.h, self.f = group, label, h, f
        self.dtype_code = _DT[dtype]
        ps = [_as_host_f64(p) for p in (w1, b1, w2, b2)]
        hdl = C.c_void_p()
        check(lib.rtpb_mlp_create(group._h, label.encode(), h, f, self.dtype_code,
                                  *[None if p is None else p.ctypes.data for p in ps], seed, stream_base,
                                  C.byref(hdl)))
        self._h = hdl
        self.ffn1 = RtpLinear(group, label + "/ffn1", h, f, dtype, _handle=lib.rtpb_mlp_layer(hdl, 0))
        self.ffn2 = RtpLinear(group, label + "/ffn2", f, h, dtype, _handle=lib.rtpb_mlp_layer(hdl, 1))

    def set_rotation_mode(self, mode: str):
        check(lib.rtpb_mlp_set_rotation_mode(self._h, {"inplace": 0, "outofplace": 1}[mode]))

    def begin_step(self):
        check(lib.rtpb_mlp_begin_step(self._h))

    def set_option(self, name: str, value: bool):
        """RtpLinear.set_option on both layers (and the fused N = 1 launches)."""
        check(lib.rtpb_mlp_set_option(self._h, _OPTIONS[name], int(bool(value))))

    def chain(self, nxt: "RtpMlp | None"):
        """Stack order: `nxt` follows this block in forward. Linked blocks post
        the neighbour's first weight shift under their own last step."""
        check(lib.rtpb_mlp_chain(self._h, nxt._h if nxt is not None else None))
        self._next = nxt  # keep the neighbour alive while linked

    def zero_grads(self):
        check(lib.rtpb_mlp_zero_grads(self._h))

    def forward(self, xs, mode: str = "train", out=None):
        rows = self._check_inputs(xs, self.h)
        ys = out if out is not None else self._acts(rows, self.h)
        self.group._enter([[x, y] for x, y in zip(xs, ys)])
        check(lib.rtpb_mlp_forward(self._h, ptr_array(xs), rows, ptr_array(ys),
                                   _lib.MODE_EVAL if mode == "eval" else _lib.MODE_TRAIN))
        self.group._leave()
        if mode != "eval":
            self._x_keep = list(xs)  # ffn1 reads X again in backward
        return ys

    def backward(self, dys, out=None):
        rows = self._check_inputs(dys, self.h)
        dxs = out if out is not None else self._acts(rows, self.h)
        self.group._enter([[a, b] for a, b in zip(dys, dxs)])
        check(lib.rtpb_mlp_backward(self._h, ptr_array(dys), rows, ptr_array(dxs)))
        self.group._leave()
        self._x_keep = None
        return dxs

    def close(self):
        if getattr(self, "_h", None):
            self.ffn1._h = self.ffn2._h = None
            lib.rtpb_mlp_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class RtpAttention(_Layer):
    """RtpAttention(group, label, wq, wk, wv, wo, heads, seq, n)
    (layers.hpp:170-191, layers_attention.cpp:43-198): heads split into N
    groups, projections without bias. wq..wo: host fp64 hidden x hidden.
    Activations: (batch * seq) x hidden CUDA tensors, one per local worker."""

    def __init__(self, group: WorkerGroup, label: str, hidden: int, heads: int, seq: int, wq, wk, wv, wo,
                 dtype="bf16"):
        self.group, self.label, self.hidden, self.heads, self.seq = group, label, hidden, heads, seq
        self.dtype_code = _DT[dtype]
        ws = [_as_host_f64(w) for w in (wq, wk, wv, wo)]
        for w in ws:
            if w.shape != (hidden, hidden):
                raise DimensionError(f"projection weight shape {w.shape} does not match ({hidden}, {hidden})")
        h = C.c_void_p()
        check(lib.rtpb_attention_create(group._h, label.encode(), hidden, heads, seq, self.dtype_code,
                                        *[w.ctypes.data for w in ws], C.byref(h)))
        self._h = h

    def shard_len(self) -> int:
        return int(lib.rtpb_attention_shard_len(self._h))

    def set_rotation_mode(self, mode: str):
        check(lib.rtpb_attention_set_rotation_mode(self._h, {"inplace": 0, "outofplace": 1}[mode]))

    def allocate_comm_spares(self):
        check(lib.rtpb_attention_allocate_comm_spares(self._h))

    def release_comm_spares(self):
        check(lib.rtpb_attention_release_comm_spares(self._h))

    def zero_grads(self):
        check(lib.rtpb_attention_zero_grads(self._h))

    def forward(self, xs, mode: str = "train", out=None):
        rows = self._check_inputs(xs, self.hidden)
        ys = out if out is not None else self._acts(rows, self.hidden)
        self.group._enter([[x, y] for x, y in zip(xs, ys)])
        check(lib.rtpb_attention_forward(self._h, ptr_array(xs), rows, ptr_array(ys),
                                         _lib.MODE_EVAL if mode == "eval" else _lib.MODE_TRAIN))
        self.group._leave()
        if mode != "eval":
            self._x_keep = list(xs)
        return ys

    def backward(self, dys, out=None):
        rows = self._check_inputs(dys, self.hidden)
        dxs = out if out is not None else self._acts(rows, self.hidden)
        self.group._enter([[a, b] for a, b in zip(dys, dxs)])
        check(lib.rtpb_attention_backward(self._h, ptr_array(dys), rows, ptr_array(dxs)))
        self.group._leave()
        self._x_keep = None
        return dxs

    def slot(self, rank: int) -> dict:
        lid, off = C.c_int64(), C.c_int64()
        check(lib.rtpb_attention_slot(self._h, rank, C.byref(lid), C.byref(off)))
        return {"logical_id": lid.value, "rotation_offset": off.value}

    def shard(self, rank: int, grad: bool = False):
        """Resident weight / gradient shard in the reference's flat layout
        [Wq_j | Wk_j | Wv_j | Wo_j] (fp64 numpy)."""
        import numpy as np
        out = np.empty(self.shard_len(), dtype=np.float64)
        check(lib.rtpb_attention_read_shard(self._h, rank, int(grad), out.ctypes.data_as(C.POINTER(C.c_double))))
        return out

    def trace(self):
        n = self.group.n
        arr = (C.c_int64 * (2 * n * n))()
        check(lib.rtpb_attention_trace(self._h, arr))
        vals = list(arr)
        return ([vals[s * n:(s + 1) * n] for s in range(n)],
                [vals[n * n + s * n: n * n + (s + 1) * n] for s in range(n)])

    def close(self):
        if getattr(self, "_h", None):
            lib.rtpb_attention_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _read_host(fn, h, rank, which, count):
    import numpy as np
    out = np.empty(count, dtype=np.float64)
    check(fn(h, rank, which, out.ctypes.data_as(C.POINTER(C.c_double))))
    return out


class RtpEmbedding(_Layer):
    """RtpEmbedding(group, label, table, n) (layers.hpp:150-168,
    layers_linear.cpp:74-136): table (vocab x emb, host fp64) sharded on the
    embedding dimension. forward(ids) takes host int64 id lists, one per
    local worker; backward(dy) has no input gradient."""

    def __init__(self, group: WorkerGroup, label: str, table, dtype="bf16"):
        t = _as_host_f64(table)
        self.group, self.label = group, label
        self.vocab, self.emb = t.shape
        self.dtype_code = _DT[dtype]
        h = C.c_void_p()
        check(lib.rtpb_embedding_create(group._h, label.encode(), self.vocab, self.emb, self.dtype_code,
                                        t.ctypes.data, C.byref(h)))
        self._h = h

    def shard_len(self) -> int:
        return int(lib.rtpb_embedding_shard_len(self._h))

    def set_rotation_mode(self, mode: str):
        check(lib.rtpb_embedding_set_rotation_mode(self._h, {"inplace": 0, "outofplace": 1}[mode]))

    def allocate_comm_spares(self):
        check(lib.rtpb_embedding_allocate_comm_spares(self._h))

    def zero_grads(self):
        check(lib.rtpb_embedding_zero_grads(self._h))

    def forward(self, ids, mode: str = "train"):
        import numpy as np
        arrs = [np.ascontiguousarray(np.asarray(v, dtype=np.int64)) for v in ids]
        if len(arrs) != len(self.group.local_ranks):
            raise DimensionError("expected one id list per local worker")
        ys = [torch.empty(len(a), self.emb, dtype=_TORCH_DT[self.dtype_code], device=self.group.device_of(r))
              for a, r in zip(arrs, self.group.local_ranks)]
        self.group._enter(None)
        ptrs = (C.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])
        counts = (C.c_size_t * len(arrs))(*[len(a) for a in arrs])
        check(lib.rtpb_embedding_forward(self._h, ptrs, counts, ptr_array(ys),
                                         _lib.MODE_EVAL if mode == "eval" else _lib.MODE_TRAIN))
        self.group._leave()
        return ys

    def backward(self, dys):
        rows = self._check_inputs(dys, self.emb)
        self.group._enter(None)
        check(lib.rtpb_embedding_backward(self._h, ptr_array(dys), rows))
        self.group._leave()

    def slot(self, rank: int) -> dict:
        lid, off = C.c_int64(), C.c_int64()
        check(lib.rtpb_embedding_slot(self._h, rank, C.byref(lid), C.byref(off)))
        return {"logical_id": lid.value, "rotation_offset": off.value}

    def shard(self, rank: int, grad: bool = False):
        return _read_host(lib.rtpb_embedding_read_shard, self._h, rank, int(grad), self.shard_len())

    def close(self):
        if getattr(self, "_h", None):
            lib.rtpb_embedding_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class RtpMoe(_Layer):
    """RtpMoe(group, label, gate, experts, n) (layers.hpp:193-229,
    layers_moe.cpp:18-198): top-1 gating (gate hidden x n, replicated),
    one expert (w1, b1, w2, b2) per worker; experts rotate past the batch."""

    def __init__(self, group: WorkerGroup, label: str, gate, experts, dtype="bf16"):
        import numpy as np
        g = _as_host_f64(gate)
        if len(experts) != group.n:
            raise ConfigError(f"moe_shard_groups: {len(experts)} experts for {group.n} shards")
        if g.ndim != 2 or g.shape[1] != group.n:
            raise ConfigError(f"gate weight {g.shape} must have one column per expert ({group.n})")
        self.group, self.label = group, label
        self.hidden = g.shape[0]
        self.ffn = np.asarray(experts[0][0]).shape[1]
        self.dtype_code = _DT[dtype]
        self._packed = [np.ascontiguousarray(np.concatenate([_as_host_f64(a).ravel() for a in e])) for e in experts]
        ptrs = (C.c_void_p * len(self._packed))(*[p.ctypes.data for p in self._packed])
        h = C.c_void_p()
        check(lib.rtpb_moe_create(group._h, label.encode(), self.hidden, self.ffn, self.dtype_code, g.ctypes.data,
                                  ptrs, C.byref(h)))
        self._h = h

    def shard_len(self) -> int:
        return int(lib.rtpb_moe_shard_len(self._h))

    def set_rotation_mode(self, mode: str):
        check(lib.rtpb_moe_set_rotation_mode(self._h, {"inplace": 0, "outofplace": 1}[mode]))

    def allocate_comm_spares(self):
        check(lib.rtpb_moe_allocate_comm_spares(self._h))

    def zero_grads(self):
        check(lib.rtpb_moe_zero_grads(self._h))

    def forward(self, xs, mode: str = "train", out=None):
        rows = self._check_inputs(xs, self.hidden)
        ys = out if out is not None else self._acts(rows, self.hidden)
        self.group._enter(None)
        check(lib.rtpb_moe_forward(self._h, ptr_array(xs), rows, ptr_array(ys),
                                   _lib.MODE_EVAL if mode == "eval" else _lib.MODE_TRAIN))
        self.group._leave()
        if mode != "eval":
            self._x_keep = list(xs)
        return ys

    def backward(self, dys, out=None):
        rows = self._check_inputs(dys, self.hidden)
        dxs = out if out is not None else self._acts(rows, self.hidden)
        self.group._enter(None)
        check(lib.rtpb_moe_backward(self._h, ptr_array(dys), rows, ptr_array(dxs)))
        self.group._leave()
        self._x_keep = None
        return dxs

    def slot(self, rank: int) -> dict:
        lid, off = C.c_int64(), C.c_int64()
        check(lib.rtpb_moe_slot(self._h, rank, C.byref(lid), C.byref(off)))
        return {"logical_id": lid.value, "rotation_offset": off.value}

    def shard(self, rank: int, grad: bool = False):
        return _read_host(lib.rtpb_moe_read_shard, self._h, rank, int(grad), self.shard_len())

    def gate_grad(self, rank: int):
        import numpy as np
        out = np.empty((self.hidden, self.group.n), dtype=np.float64)
        check(lib.rtpb_moe_gate_grad(self._h, rank, out.ctypes.data_as(C.POINTER(C.c_double))))
        return out

    def close(self):
        if getattr(self, "_h", None):
            lib.rtpb_moe_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class RtpModel:
    """RtpModel (model.cpp:7-121) with SerialModel(dims, seed)'s parameters:
    embedding -> layers x (attention + FFN or MoE, residuals) -> head."""

    def __init__(self, group: WorkerGroup, heads=4, hidden=32, layers=2, seq=16, vocab=64, ffn=128, moe=False,
                 seed=42, mode="inplace", dtype="bf16"):
        self.group, self.vocab, self.hidden, self.layers = group, vocab, hidden, layers
        self.dtype_code = _DT[dtype]
        h = C.c_void_p()
        check(lib.rtpb_model_create(group._h, heads, hidden, layers, seq, vocab, ffn, int(moe), seed,
                                    {"inplace": 0, "outofplace": 1}[mode], self.dtype_code, C.byref(h)))
        self._h = h

    def begin_step(self):
        check(lib.rtpb_model_begin_step(self._h))

    def zero_grads(self):
        check(lib.rtpb_model_zero_grads(self._h))

    def forward(self, ids, mode="train"):
        import numpy as np
        arrs = [np.ascontiguousarray(np.asarray(v, dtype=np.int64)) for v in ids]
        outs = [torch.empty(len(a), self.vocab, dtype=_TORCH_DT[self.dtype_code], device=self.group.device_of(r))
                for a, r in zip(arrs, self.group.local_ranks)]
        self.group._enter(None)
        ptrs = (C.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])
        counts = (C.c_size_t * len(arrs))(*[len(a) for a in arrs])
        check(lib.rtpb_model_forward(self._h, ptrs, counts, ptr_array(outs),
                                     _lib.MODE_EVAL if mode == "eval" else _lib.MODE_TRAIN))
        self.group._leave()
        return outs

    def backward(self, dlogits):
        self.group._enter(None)
        check(lib.rtpb_model_backward(self._h, ptr_array(dlogits), dlogits[0].shape[0]))
        self.group._leave()

    def layer_count(self) -> int:
        return int(lib.rtpb_model_layer_count(self._h))

    def layer_shard(self, layer: int, rank: int, grad: bool = False):
        import numpy as np
        out = np.empty(int(lib.rtpb_model_layer_shard_len(self._h, layer)), dtype=np.float64)
        check(lib.rtpb_model_read_layer_shard(self._h, layer, rank, int(grad),
                                              out.ctypes.data_as(C.POINTER(C.c_double))))
        return out

    def gate_grad(self, block: int, rank: int):
        import numpy as np
        out = np.empty((self.hidden, self.group.n), dtype=np.float64)
        check(lib.rtpb_model_gate_grad(self._h, block, rank, out.ctypes.data_as(C.POINTER(C.c_double))))
        return out

    def close(self):
        if getattr(self, "_h", None):
            lib.rtpb_model_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# --- step kernels (layer (1) of rtpb.h), on torch tensors ---

def _ws(which, dtype_code, M, I, per, device):
    n = lib.rtpb_step_workspace_bytes(which, dtype_code, M, I, per)
    return torch.zeros(max(16, n), dtype=torch.uint8, device=device)  # zero-filled before first use


def fwd_step(x, w_shard, y, col0, per, act=None, store_pre=True, stream=None, exact_gelu=False):
    dt = F32 if x.dtype == torch.float32 else BF16
    M, I = x.shape
    ws = _ws(0, dt, M, I, per, x.device)
    flags = (_lib.EPI_STORE_PRE if store_pre else 0) | (_lib.EPI_GELU if act is not None else 0) | \
        (64 if exact_gelu else 0)
    s = (stream or torch.cuda.current_stream(x.device)).cuda_stream
    check(lib.rtpb_fwd_step(dt, x.data_ptr(), x.stride(0), w_shard.data_ptr(),
                            y.data_ptr() if y is not None else None, y.stride(0) if y is not None else 0, col0,
                            act.data_ptr() if act is not None else None, act.stride(0) if act is not None else 0,
                            M, I, per, flags, ws.data_ptr(), ws.numel(), s))


def dgrad_step(dy, col0, w_shard, acc, dx, M, I, per, first, last, pre=None, stream=None):
    dt = F32 if dy.dtype == torch.float32 else BF16
    ws = _ws(1, dt, M, I, per, dy.device)
    flags = (_lib.EPI_FIRST if first else 0) | (_lib.EPI_LAST if last else 0) | \
        (_lib.EPI_GELU_BWD if pre is not None else 0)
    s = (stream or torch.cuda.current_stream(dy.device)).cuda_stream
    check(lib.rtpb_dgrad_step(dt, dy.data_ptr(), dy.stride(0), col0, w_shard.data_ptr(),
                              acc.data_ptr() if acc is not None else None, I,
                              dx.data_ptr() if dx is not None else None, I,
                              pre.data_ptr() if pre is not None else None, I, M, I, per, flags,
                              ws.data_ptr(), ws.numel(), s))


def wgrad_step(x, dy, col0, g_in, g_out, per, stream=None):
    dt = F32 if x.dtype == torch.float32 else BF16
    M, I = x.shape
    ws = _ws(2, dt, M, I, per, x.device)
    s = (stream or torch.cuda.current_stream(x.device)).cuda_stream
    check(lib.rtpb_wgrad_step(dt, x.data_ptr(), x.stride(0), dy.data_ptr(), dy.stride(0), col0,
                              None if g_in is None else g_in.data_ptr(), g_out.data_ptr(), M, I, per, ws.data_ptr(),
                              ws.numel(), s))


def _pass_cols(cols):
    arr = (C.c_size_t * len(cols))(*cols)
    return arr


def pass_done_target(which, M, I, per, steps, flags=0) -> int:
    return int(lib.rtpb_pass_done_target(which, M, I, per, steps, flags))


def fwd_pass(x, buf0, buf1, y, cols, per, act=None, store_pre=True, ready=None, done=None, reset_ctr=None,
             exact_gelu=False, stream=None, announced_target=0):
    """rtpb_fwd_pass: step s of a layer's forward pass (shard in buffer s & 1,
    output column block cols[s]) for every s, in one launch. Returns the
    per-step count-in target on `done`."""
    M, I = x.shape
    flags = (_lib.EPI_STORE_PRE if store_pre else 0) | (_lib.EPI_GELU if act is not None else 0) | \
        (64 if exact_gelu else 0)
    ycols = (y if y is not None else act).shape[1]
    mask = sum(1 << s for s in range(len(cols)) if s & 1)
    tgt = C.c_uint(announced_target)
    s = (stream or torch.cuda.current_stream(x.device)).cuda_stream
    check(lib.rtpb_fwd_pass(x.data_ptr(), x.stride(0), buf0.data_ptr(), buf1.data_ptr(),
                            y.data_ptr() if y is not None else None, y.stride(0) if y is not None else 0,
                            act.data_ptr() if act is not None else None, act.stride(0) if act is not None else 0,
                            ycols, _pass_cols(cols), mask, len(cols), M, I, per, flags,
                            None if ready is None else ready.data_ptr(), None if done is None else done.data_ptr(),
                            C.byref(tgt), None if reset_ctr is None else reset_ctr.data_ptr(), s))
    return tgt.value


def dgrad_pass(dy, buf0, buf1, cols, acc, dx, I, per, pre=None, pair=False, ready=None, done=None, reset_ctr=None,
               stream=None):
    """rtpb_dgrad_pass: dX = sum_s dY[:, cols[s]:+per] . W_s^T over the pass's
    steps (shard s in buffer s & 1) in one launch; pair: paired dX units."""
    M = dy.shape[0]
    flags = (_lib.EPI_GELU_BWD if pre is not None else 0) | (128 if pair else 0)
    mask = sum(1 << s for s in range(len(cols)) if s & 1)
    tgt = C.c_uint(0)
    s = (stream or torch.cuda.current_stream(dy.device)).cuda_stream
    check(lib.rtpb_dgrad_pass(dy.data_ptr(), dy.stride(0), dy.shape[1], buf0.data_ptr(), buf1.data_ptr(),
                              _pass_cols(cols), mask, len(cols), acc.data_ptr(), acc.stride(0), dx.data_ptr(),
                              dx.stride(0), None if pre is None else pre.data_ptr(), 0 if pre is None else pre.stride(0),
                              M, I, per, flags, None if ready is None else ready.data_ptr(),
                              None if done is None else done.data_ptr(), C.byref(tgt),
                              None if reset_ctr is None else reset_ctr.data_ptr(), s))
    return tgt.value


def flyweight_init(dst, seed, stream_base, I, O, n, j, lo=-0.1, hi=0.1, stream=None):
    dt = F32 if dst.dtype == torch.float32 else BF16
    s = (stream or torch.cuda.current_stream(dst.device)).cuda_stream
    check(lib.rtpb_flyweight_init(dst.data_ptr(), dt, seed, stream_base, I, O, n, j, lo, hi, s))


def launch_count() -> int:
    return int(lib.rtpb_launch_count())


