"""oracle/oracle.py — TEST INFRASTRUCTURE ONLY (the CPU checker).

ctypes front-ends for
  * ``Oracle``    — our plain-C fp64 restatement (oracle/_build/liboracle.so,
                    rtp_oracle.c), pinned bit-exactly to the reference by
                    tests/golden/*.npz;
  * ``Reference`` — the reference sources themselves compiled by path
                    (oracle/_ref/librtpref.so, oracle/Makefile + ref_shim.cpp),
                    used to make the golden fixtures and as bench.py's
                    reference arm. Absent on machines without /root/reference
                    unless prebuilt and shipped.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / reference
arm) import this module. The product path (paper_2311_01635_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "librtpref.so")

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_sz = C.c_size_t
_u64 = C.c_uint64


def build_oracle(with_ref: bool | None = None) -> None:
    """make -C oracle (the C restatement; the reference lib too when its
    sources are present). Building the checker is not using it."""
    subprocess.check_call(["make", "-s", "-C", HERE, "oracle"])
    if with_ref is None:
        with_ref = os.path.isdir("/root/reference/proj/src")
    if with_ref:
        subprocess.check_call(["make", "-s", "-j8", "-C", HERE, "ref"])


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


class Oracle:
    """fp64 C restatement of the reference path (rtp_oracle.h)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build_oracle(with_ref=False)
        L = C.CDLL(path)
        L.orc_splitmix_at.argtypes = [_u64, _u64]
        L.orc_splitmix_at.restype = _u64
        L.orc_uniform.argtypes = [_u64, _u64, _u64, C.c_double, C.c_double, _dp]
        L.orc_linear_shard.argtypes = [_u64, _u64, _sz, _sz, _sz, _sz, _dp]
        L.orc_gelu.argtypes = [_dp, _dp, _sz]
        L.orc_gelu_backward.argtypes = [_dp, _dp, _dp, _sz]
        L.orc_rtp_linear.argtypes = [_sz, _sz, _sz, _sz, _dp, _dp, _dp, _dp, _dp, _dp, _dp, C.c_void_p]
        L.orc_rtp_linear.restype = C.c_int
        L.orc_rtp_mlp.argtypes = [_sz, _sz, _sz, _sz, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp]
        L.orc_rtp_attention.argtypes = [_sz, _sz, _sz, _sz, _sz, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp]
        L.orc_rtp_mlp.restype = C.c_int
        L.orc_sampled_dots.argtypes = [_dp, _sz, _sz, _dp, _sz, _sz, _sz, _ip, _ip, _sz, _dp]
        L.orc_rtp_memory.argtypes = [_u64, _u64, _u64, C.c_int]
        L.orc_rtp_memory.restype = _u64
        self.L = L

    def splitmix_at(self, seed: int, k: int) -> int:
        return int(self.L.orc_splitmix_at(seed, k))

    def uniform(self, seed, skip, count, lo, hi) -> np.ndarray:
        out = np.empty(count, np.float64)
        self.L.orc_uniform(seed, skip, count, lo, hi, out)
        return out

    def linear_shard(self, seed, base, I, O, n, j) -> np.ndarray:
        out = np.empty(I * (O // n) + O // n, np.float64)
        self.L.orc_linear_shard(seed, base, I, O, n, j, out)
        return out

    def gelu(self, x):
        x = _f64(x)
        y = np.empty_like(x)
        self.L.orc_gelu(x.ravel(), y.ravel(), x.size)
        return y

    def gelu_backward(self, x, up):
        x, up = _f64(x), _f64(up)
        y = np.empty_like(x)
        self.L.orc_gelu_backward(x.ravel(), up.ravel(), y.ravel(), x.size)
        return y

    def rtp_linear(self, n, w, b, x, dy, trace=False):
        """RtpLinear Train fwd + bwd over n simulated workers (fp64)."""
        w, b, x, dy = _f64(w), _f64(b), _f64(x), _f64(dy)
        rows, I = x.shape
        O = w.shape[1]
        per = O // n
        y = np.empty((rows, O))
        dx = np.empty((rows, I))
        g = np.empty((n, I * per + per))
        tr = np.empty(2 * n * n, np.int64) if trace else None
        rc = self.L.orc_rtp_linear(n, rows, I, O, w, b, x, dy, y, dx, g,
                                   tr.ctypes.data if trace else None)
        if rc:
            raise ValueError(f"orc_rtp_linear: ConfigError (code {rc})")
        out = {"y": y, "dx": dx, "grads": g}
        if trace:
            out["fwd_ids"] = tr[: n * n].reshape(n, n)
            out["bwd_ids"] = tr[n * n:].reshape(n, n)
        return out

    def rtp_mlp(self, n, w1, b1, w2, b2, x, dy):
        w1, b1, w2, b2, x, dy = map(_f64, (w1, b1, w2, b2, x, dy))
        rows, h = x.shape
        f = w1.shape[1]
        y = np.empty((rows, h))
        dx = np.empty((rows, h))
        g1 = np.empty((n, h * (f // n) + f // n))
        g2 = np.empty((n, f * (h // n) + h // n))
        rc = self.L.orc_rtp_mlp(n, rows, h, f, w1, b1, w2, b2, x, dy, y, dx, g1, g2)
        if rc:
            raise ValueError(f"orc_rtp_mlp: ConfigError (code {rc})")
        return {"y": y, "dx": dx, "grads1": g1, "grads2": g2}

    def rtp_attention(self, n, heads, seq, wq, wk, wv, wo, x, dy):
        wq, wk, wv, wo, x, dy = map(_f64, (wq, wk, wv, wo, x, dy))
        rows, H = x.shape
        y, dx = np.empty((rows, H)), np.empty((rows, H))
        g = np.empty((n, 4 * H * (H // n)))
        rc = self.L.orc_rtp_attention(n, rows, H, heads, seq, wq, wk, wv, wo, x, dy, y, dx, g)
        if rc:
            raise ValueError(f"orc_rtp_attention: ConfigError (code {rc})")
        return {"y": y, "dx": dx, "grads": g}

    def sampled_dots(self, a, lda, sa, b, ldb, sb, k, ri, ci):
        ri = np.ascontiguousarray(ri, np.int64)
        ci = np.ascontiguousarray(ci, np.int64)
        out = np.empty(len(ri))
        self.L.orc_sampled_dots(_f64(a).ravel(), lda, sa, _f64(b).ravel(), ldb, sb, k, ri, ci, len(ri), out)
        return out

    def rtp_memory(self, W, G, N, outofplace) -> int:
        return int(self.L.orc_rtp_memory(W, G, N, int(outofplace)))


class Reference:
    """The reference itself (sources compiled by path; oracle/ref_shim.cpp)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where /root/reference exists")
        L = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_uniform.argtypes = [_u64, _u64, _u64, C.c_double, C.c_double, _dp]
        L.ref_linear_shard.argtypes = [_sz, _sz, _sz, _sz, _dp, _dp, _dp]
        L.ref_mlp_params.argtypes = [_u64, _sz, _sz, _sz, _dp]
        L.ref_serial_linear.argtypes = [_sz, _sz, _sz, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp]
        L.ref_rtp_linear.argtypes = [_sz, C.c_int, C.c_int, _sz, _sz, _sz, _dp, _dp, _dp, _dp, _dp,
                                     _dp, _dp, _ip, _ip, _ip, C.POINTER(_sz)]
        L.ref_rtp_attention.argtypes = [_sz, C.c_int, _sz, _sz, _sz, _sz, _dp, _dp, _dp, _dp, _dp, _dp, _dp,
                                        _dp, _dp]
        L.ref_rtp_mlp.argtypes = [_sz, C.c_int, C.c_int, _sz, _sz, _sz, _dp, _dp, _dp, _dp, _dp,
                                  _dp, _dp, _dp, _dp, _dp]
        L.ref_rtp_moe.argtypes = [_sz, C.c_int, _sz, _sz, _sz, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp]
        L.ref_rtp_embedding.argtypes = [_sz, C.c_int, _sz, _sz, _sz, _dp, C.POINTER(C.c_int64), _dp, _dp, _dp]
        L.ref_rtp_model.argtypes = [_sz, C.c_int, C.c_int, _sz, _sz, _sz, _sz, _sz, _sz, C.c_int, _u64, _sz,
                                    C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(_sz),
                                    C.POINTER(_sz)]
        L.ref_cmd_csv.argtypes = [C.c_int, _sz, C.c_char_p, _sz, C.c_char_p, _sz]
        L.ref_time_mlp.argtypes = [_sz, C.c_int, _sz, _sz, _sz, _u64, C.c_int, C.POINTER(C.c_double)]
        L.ref_mlp_ledger.argtypes = [_sz, C.c_int, _sz, _sz, _sz, _u64, C.POINTER(_sz), C.POINTER(_sz)]
        L.ref_ring_ops.argtypes = [_sz, C.c_int, C.POINTER(C.c_int), _sz, _sz, _ip, _ip, _dp, _dp]
        L.ref_table1.argtypes = [C.c_int, _u64, _u64, _u64, _u64, _u64, C.POINTER(_u64)]
        for name in ("ref_uniform", "ref_linear_shard", "ref_mlp_params", "ref_serial_linear",
                     "ref_rtp_linear", "ref_rtp_mlp", "ref_time_mlp", "ref_mlp_ledger",
                     "ref_ring_ops", "ref_table1", "ref_rtp_moe", "ref_rtp_embedding", "ref_cmd_csv", "ref_rtp_model"):
            getattr(L, name).restype = C.c_int
        self.L = L

    def _chk(self, rc):
        if rc:
            raise RuntimeError(f"reference error {rc}: {self.L.ref_last_error().decode()}")

    def uniform(self, seed, skip, count, lo, hi):
        out = np.empty(count)
        self._chk(self.L.ref_uniform(seed, skip, count, lo, hi, out))
        return out

    def linear_shard(self, w, b, n, r):
        w, b = _f64(w), _f64(b)
        I, O = w.shape
        out = np.empty(I * (O // n) + O // n)
        self._chk(self.L.ref_linear_shard(I, O, n, r, w, b, out))
        return out

    def mlp_params(self, seed, h, f, blocks=1):
        out = np.empty(blocks * (h * f + f + f * h + h))
        self._chk(self.L.ref_mlp_params(seed, h, f, blocks, out))
        return out

    def serial_linear(self, w, b, x, dy):
        w, b, x, dy = map(_f64, (w, b, x, dy))
        rows, I = x.shape
        O = w.shape[1]
        y, dx, gw, gb = np.empty((rows, O)), np.empty((rows, I)), np.empty((I, O)), np.empty(O)
        self._chk(self.L.ref_serial_linear(rows, I, O, w, b, x, dy, y, dx, gw, gb))
        return {"y": y, "dx": dx, "gw": gw, "gb": gb}

    def rtp_linear(self, n, w, b, x, dy, concurrent=False, outofplace=False):
        w, b, x, dy = map(_f64, (w, b, x, dy))
        rows, I = x.shape
        O = w.shape[1]
        per = O // n
        y, dx = np.empty((rows, O)), np.empty((rows, I))
        g = np.empty((n, I * per + per))
        fwd_ids, bwd_ids = np.empty(n, np.int64), np.empty(n, np.int64)
        traffic = np.zeros(3 * 4 * n + 3, np.int64)
        nt = _sz(0)
        self._chk(self.L.ref_rtp_linear(n, int(concurrent), int(outofplace), rows, I, O, w, b, x, dy,
                                        y, dx, g, fwd_ids, bwd_ids, traffic, C.byref(nt)))
        return {"y": y, "dx": dx, "grads": g, "fwd_ids": fwd_ids, "bwd_ids": bwd_ids,
                "traffic": traffic[: 3 * nt.value].reshape(-1, 3)}

    def rtp_mlp(self, n, w1, b1, w2, b2, x, dy, concurrent=False, outofplace=False):
        w1, b1, w2, b2, x, dy = map(_f64, (w1, b1, w2, b2, x, dy))
        rows, h = x.shape
        f = w1.shape[1]
        y, dx = np.empty((rows, h)), np.empty((rows, h))
        g1 = np.empty((n, h * (f // n) + f // n))
        g2 = np.empty((n, f * (h // n) + h // n))
        self._chk(self.L.ref_rtp_mlp(n, int(concurrent), int(outofplace), rows, h, f, w1, b1, w2, b2,
                                     x, dy, y, dx, g1, g2))
        return {"y": y, "dx": dx, "grads1": g1, "grads2": g2}

    def rtp_attention(self, n, heads, seq, wq, wk, wv, wo, x, dy, concurrent=False):
        wq, wk, wv, wo, x, dy = map(_f64, (wq, wk, wv, wo, x, dy))
        rows, H = x.shape
        y, dx = np.empty((rows, H)), np.empty((rows, H))
        g = np.empty((n, 4 * H * (H // n)))
        self._chk(self.L.ref_rtp_attention(n, int(concurrent), rows, H, heads, seq, wq, wk, wv, wo, x, dy,
                                           y, dx, g))
        return {"y": y, "dx": dx, "grads": g}

    def rtp_moe(self, n, gate, experts, x, dy, concurrent=False):
        """experts: list of n (w1, b1, w2, b2)."""
        gate, x, dy = map(_f64, (gate, x, dy))
        rows, H = x.shape
        f = experts[0][0].shape[1]
        packed = _f64(np.concatenate([np.concatenate([_f64(a).ravel() for a in e]) for e in experts]))
        L = 2 * H * f + f + H
        y, dx = np.empty((rows, H)), np.empty((rows, H))
        g, gg = np.empty((n, L)), np.empty((n, H, n))
        self._chk(self.L.ref_rtp_moe(n, int(concurrent), rows, H, f, gate, packed, x, dy, y, dx, g, gg))
        return {"y": y, "dx": dx, "grads": g, "gate_grads": gg}

    def rtp_embedding(self, n, table, ids, dy, concurrent=False):
        """ids: (n, rows_per_worker) int64."""
        table, dy = _f64(table), _f64(dy)
        vocab, emb = table.shape
        ids = np.ascontiguousarray(ids, np.int64)
        rpw = ids.shape[1]
        y = np.empty((n * rpw, emb))
        g = np.empty((n, vocab * (emb // n)))
        self._chk(self.L.ref_rtp_embedding(n, int(concurrent), vocab, emb, rpw, table,
                                           ids.ctypes.data_as(C.POINTER(C.c_int64)), dy, y, g))
        return {"y": y, "grads": g}

    def rtp_model(self, n, heads, hidden, layers, seq, vocab, ffn, moe=False, seed=42, batch=4, outofplace=False,
                  concurrent=False):
        """RtpModel(SerialModel(dims, seed)) one training step (verify.cpp:54-79)."""
        nl = _sz(0)
        lens = (_sz * 64)()
        args = [n, int(concurrent), int(outofplace), heads, hidden, layers, seq, vocab, ffn, int(moe), seed, batch]
        self._chk(self.L.ref_rtp_model(*args, None, None, None, None, None, C.byref(nl), lens))
        L = [int(lens[i]) for i in range(nl.value)]
        rows = batch * seq
        ids = np.empty(rows, np.int64)
        logits, dlogits = np.empty((rows, vocab)), np.empty((rows, vocab))
        grads = np.empty(n * sum(L))
        gg = np.empty(max(1, layers * n * hidden * n))
        ptr = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
        self._chk(self.L.ref_rtp_model(*args, ptr(ids), ptr(logits), ptr(dlogits), ptr(grads), ptr(gg),
                                       C.byref(nl), lens))
        out, off = [], 0
        for ln in L:
            out.append(grads[off:off + n * ln].reshape(n, ln))
            off += n * ln
        return {"ids": ids, "logits": logits, "dlogits": dlogits, "grads": out,
                "gate_grads": gg[:layers * n * hidden * n].reshape(layers, n, hidden, n) if moe else None}

    def cmd_csv(self, which: str, n: int, strategy: str, batch: int) -> str:
        """CSV text of the reference's `rtpsim memtable|ledger|sweep` commands."""
        buf = C.create_string_buffer(1 << 20)
        code = {"memtable": 0, "ledger": 1, "sweep": 2}[which]
        self._chk(self.L.ref_cmd_csv(code, n, strategy.encode(), batch, buf, len(buf)))
        return buf.value.decode()

    def time_mlp(self, n, rows, h, f, seed=42, iters=1, concurrent=True) -> float:
        s = C.c_double(0)
        self._chk(self.L.ref_time_mlp(n, int(concurrent), rows, h, f, seed, iters, C.byref(s)))
        return s.value

    def mlp_ledger(self, n, outofplace, rows, h, f, seed=42):
        peaks = (_sz * 5)()
        fpb = _sz(0)
        self._chk(self.L.ref_mlp_ledger(n, int(outofplace), rows, h, f, seed, peaks, C.byref(fpb)))
        return {"param": peaks[0], "grad": peaks[1], "activation": peaks[2], "comm": peaks[3],
                "other": peaks[4], "flat_param_bytes": fpb.value}

    def ring_ops(self, n, ops, length=2, concurrent=False):
        arr = (C.c_int * max(1, len(ops)))(*ops)
        ids, offs = np.empty(n, np.int64), np.empty(n, np.int64)
        w0, g0 = np.empty(n), np.empty(n)
        self._chk(self.L.ref_ring_ops(n, int(concurrent), arr, len(ops), length, ids, offs, w0, g0))
        return {"ids": ids, "offsets": offs, "w0": w0, "g0": g0}

    def table1(self, strategy, W, G, A, Ap, N):
        out = (_u64 * 3)()
        self._chk(self.L.ref_table1(strategy, W, G, A, Ap, N, out))
        return tuple(int(v) for v in out)
