"""ctypes binding of include/rtpb.h (librtpb.so, built in-tree by `make lib`).

The product path has no fallback: if the shared library is missing or fails
to load, importing this module raises. The library is the B200 (sm_100a)
implementation; nothing here computes.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# RTPB_LIB: load an A/B build of the same library (tools/build_variant.sh)
LIB_PATH = os.environ.get("RTPB_LIB") or os.path.join(HERE, "librtpb.so")

RTPB_OK = 0
ERR_NAMES = {1: "Generic", 2: "Config", 3: "Dimension", 4: "Protocol", 5: "State", 6: "Index", 7: "Cuda", 8: "Nccl"}

BF16, F32 = 0, 1
EPI_GELU, EPI_FIRST, EPI_LAST, EPI_GELU_BWD, EPI_STORE_PRE, EPI_NO_BIAS = 1, 2, 4, 8, 16, 32
TRANSPORT_LOCKSTEP, TRANSPORT_CONCURRENT, TRANSPORT_NCCL = 0, 1, 2
MODE_TRAIN, MODE_EVAL = 0, 1
ROT_INPLACE, ROT_OUTOFPLACE = 0, 1

_sz, _u64, _i64, _vp, _int, _dbl = C.c_size_t, C.c_uint64, C.c_int64, C.c_void_p, C.c_int, C.c_double
_vpp = C.POINTER(C.c_void_p)

# name: (restype, argtypes)
_SIGS = {
    "rtpb_last_error": (C.c_char_p, []),
    "rtpb_version": (C.c_char_p, []),
    "rtpb_launch_count": (_u64, []),
    "rtpb_preload_kernels": (None, []),
    "rtpb_debug_force_bn": (None, [_int]),
    "rtpb_debug_trace": (None, [_vp, _sz]),
    "rtpb_debug_skip_comm": (None, [_int]),
    "rtpb_debug_read_flags": (_int, [_vp, _sz, _sz, _sz, C.POINTER(C.c_uint), C.POINTER(_int)]),
    "rtpb_debug_flag_address": (_u64, [_vp, _sz, _sz]),
    "rtpb_profile_enable": (None, [_int]),
    "rtpb_profile_read": (_sz, [C.POINTER(_int), C.POINTER(_dbl), C.POINTER(C.c_float), C.POINTER(C.c_float),
                                C.POINTER(_int), _sz]),
    "rtpb_set_sm_budget": (None, [_int]),
    "rtpb_debug_fused_plan": (_dbl, [_sz, _sz, _sz, _int]),
    "rtpb_step_workspace_bytes": (_sz, [_int, _int, _sz, _sz, _sz]),
    "rtpb_flyweight_init": (_int, [_vp, _int, _u64, _u64, _sz, _sz, _sz, _sz, _dbl, _dbl, _vp]),
    "rtpb_fwd_step": (_int, [_int, _vp, _sz, _vp, _vp, _sz, _sz, _vp, _sz, _sz, _sz, _sz, _int, _vp, _sz, _vp]),
    "rtpb_dgrad_step": (_int, [_int, _vp, _sz, _sz, _vp, _vp, _sz, _vp, _sz, _vp, _sz, _sz, _sz, _sz, _int, _vp,
                               _sz, _vp]),
    "rtpb_dgrad_step2": (_int, [_int, _vp, _sz, _sz, _vp, _sz, _vp, _vp, _sz, _vp, _sz, _vp, _sz, _sz, _sz, _sz,
                                 _int, _vp, _sz, _vp]),
    "rtpb_pass_done_target": (C.c_uint, [_int, _sz, _sz, _sz, _sz, _int]),
    "rtpb_fwd_pass": (_int, [_vp, _sz, _vp, _vp, _vp, _sz, _vp, _sz, _sz, C.POINTER(_sz), C.c_uint, _sz, _sz, _sz,
                             _sz, _int, _vp, _vp, C.POINTER(C.c_uint), _vp, _vp]),
    "rtpb_dgrad_pass": (_int, [_vp, _sz, _sz, _vp, _vp, C.POINTER(_sz), C.c_uint, _sz, _vp, _sz, _vp, _sz, _vp, _sz,
                               _sz, _sz, _sz, _int, _vp, _vp, C.POINTER(C.c_uint), _vp, _vp]),
    "rtpb_wgrad_pass": (_int, [_vp, _sz, _vp, _sz, _sz, _vp, C.POINTER(_sz), _sz, _sz, _sz, _sz, _int, _vp, _vp, _vp,
                               C.POINTER(C.c_uint), _vp, _vp, _sz, _vp]),
    "rtpb_colsum_workspace_bytes": (_sz, [_sz, _sz]),
    "rtpb_colsum": (_int, [_vp, _sz, _sz, _sz, _vp, _vp, _sz, _vp]),
    "rtpb_wgrad_step": (_int, [_int, _vp, _sz, _vp, _sz, _sz, _vp, _vp, _sz, _sz, _sz, _vp, _sz, _vp]),
    "rtpb_gelu": (_int, [_int, _vp, _vp, _sz, _vp]),
    "rtpb_convert": (_int, [_vp, _int, _vp, _int, _sz, _vp]),
    "rtpb_fill": (_int, [_vp, _int, _sz, _dbl, _vp]),
    "rtpb_gelu_backward": (_int, [_int, _vp, _vp, _vp, _sz, _vp]),
    "rtpb_ring_plan": (_int, [_sz, _sz, _int, _sz, C.POINTER(_i64), C.POINTER(_i64), C.POINTER(_i64)]),
    # group / layer handles
    "rtpb_group_create": (_int, [_sz, _int, C.POINTER(_int), _vpp]),
    "rtpb_nccl_unique_id": (_int, [_vp]),
    "rtpb_group_create_nccl": (_int, [_sz, _sz, _int, _vp, _vpp]),
    "rtpb_ipc_unique_id": (_int, [_vp]),
    "rtpb_group_create_ipc": (_int, [_sz, _sz, _int, _vp, _vpp]),
    "rtpb_group_create_solo": (_int, [_sz, _sz, _int, _vpp]),
    "rtpb_group_destroy": (_int, [_vp]),
    "rtpb_group_size": (_sz, [_vp]),
    "rtpb_group_local_ranks": (_sz, [_vp, C.POINTER(_sz)]),
    "rtpb_group_stream": (_vp, [_vp, _sz, _int]),
    "rtpb_group_device": (_int, [_vp, _sz]),
    "rtpb_group_synchronize": (_int, [_vp]),
    "rtpb_group_traffic": (_sz, [_vp, C.POINTER(_i64), C.POINTER(_i64), C.POINTER(_i64), _sz]),
    "rtpb_group_clear_traffic": (None, [_vp]),
    "rtpb_group_corrupt_next_exchange": (_int, [_vp, _sz, _int]),
    "rtpb_group_ledger": (_int, [_vp, _sz, C.POINTER(_sz), C.POINTER(_sz), C.POINTER(_sz)]),
    "rtpb_group_reset_ledger_peaks": (_int, [_vp]),
    "rtpb_group_rotate": (_int, [_vp, _int, _vpp, _vpp, _vpp, _sz, _sz]),
    "rtpb_group_allgather": (_int, [_vp, _vpp, _vpp, _sz]),
    "rtpb_linear_create": (_int, [_vp, C.c_char_p, _sz, _sz, _int, _vp, _vp, _u64, _u64, _vpp]),
    "rtpb_linear_destroy": (_int, [_vp]),
    "rtpb_linear_set_rotation_mode": (_int, [_vp, _int]),
    "rtpb_linear_allocate_comm_spares": (_int, [_vp]),
    "rtpb_linear_release_comm_spares": (_int, [_vp]),
    "rtpb_linear_zero_grads": (_int, [_vp]),
    "rtpb_linear_shard_len": (_sz, [_vp]),
    "rtpb_linear_forward": (_int, [_vp, _vpp, _sz, _vpp, _int]),
    "rtpb_linear_backward": (_int, [_vp, _vpp, _sz, _vpp]),
    "rtpb_linear_slot": (_int, [_vp, _sz, C.POINTER(_i64), C.POINTER(_i64), _vpp, _vpp]),
    "rtpb_linear_trace": (_int, [_vp, C.POINTER(_i64)]),
    "rtpb_linear_read_shard": (_int, [_vp, _sz, _int, _vp]),
    "rtpb_mlp_create": (_int, [_vp, C.c_char_p, _sz, _sz, _int, _vp, _vp, _vp, _vp, _u64, _u64, _vpp]),
    "rtpb_mlp_destroy": (_int, [_vp]),
    "rtpb_mlp_set_rotation_mode": (_int, [_vp, _int]),
    "rtpb_mlp_begin_step": (_int, [_vp]),
    "rtpb_mlp_zero_grads": (_int, [_vp]),
    "rtpb_mlp_forward": (_int, [_vp, _vpp, _sz, _vpp, _int]),
    "rtpb_mlp_backward": (_int, [_vp, _vpp, _sz, _vpp]),
    "rtpb_mlp_chain": (_int, [_vp, _vp]),
    "rtpb_mlp_layer": (_vp, [_vp, _int]),
    "rtpb_attention_create": (_int, [_vp, C.c_char_p, _sz, _sz, _sz, _int, _vp, _vp, _vp, _vp, _vpp]),
    "rtpb_attention_destroy": (_int, [_vp]),
    "rtpb_attention_set_rotation_mode": (_int, [_vp, _int]),
    "rtpb_attention_allocate_comm_spares": (_int, [_vp]),
    "rtpb_attention_release_comm_spares": (_int, [_vp]),
    "rtpb_attention_zero_grads": (_int, [_vp]),
    "rtpb_attention_shard_len": (_sz, [_vp]),
    "rtpb_attention_forward": (_int, [_vp, _vpp, _sz, _vpp, _int]),
    "rtpb_attention_backward": (_int, [_vp, _vpp, _sz, _vpp]),
    "rtpb_attention_slot": (_int, [_vp, _sz, C.POINTER(_i64), C.POINTER(_i64)]),
    "rtpb_attention_trace": (_int, [_vp, C.POINTER(_i64)]),
    "rtpb_attention_read_shard": (_int, [_vp, _sz, _int, C.POINTER(_dbl)]),
    "rtpb_embedding_create": (_int, [_vp, C.c_char_p, _sz, _sz, _int, _vp, _vpp]),
    "rtpb_embedding_destroy": (_int, [_vp]),
    "rtpb_embedding_set_rotation_mode": (_int, [_vp, _int]),
    "rtpb_embedding_allocate_comm_spares": (_int, [_vp]),
    "rtpb_embedding_release_comm_spares": (_int, [_vp]),
    "rtpb_embedding_zero_grads": (_int, [_vp]),
    "rtpb_embedding_shard_len": (_sz, [_vp]),
    "rtpb_embedding_forward": (_int, [_vp, _vpp, C.POINTER(_sz), _vpp, _int]),
    "rtpb_embedding_backward": (_int, [_vp, _vpp, _sz]),
    "rtpb_embedding_slot": (_int, [_vp, _sz, C.POINTER(_i64), C.POINTER(_i64)]),
    "rtpb_embedding_read_shard": (_int, [_vp, _sz, _int, C.POINTER(_dbl)]),
    "rtpb_moe_create": (_int, [_vp, C.c_char_p, _sz, _sz, _int, _vp, _vpp, _vpp]),
    "rtpb_moe_destroy": (_int, [_vp]),
    "rtpb_moe_set_rotation_mode": (_int, [_vp, _int]),
    "rtpb_moe_allocate_comm_spares": (_int, [_vp]),
    "rtpb_moe_release_comm_spares": (_int, [_vp]),
    "rtpb_moe_zero_grads": (_int, [_vp]),
    "rtpb_moe_shard_len": (_sz, [_vp]),
    "rtpb_moe_forward": (_int, [_vp, _vpp, _sz, _vpp, _int]),
    "rtpb_moe_backward": (_int, [_vp, _vpp, _sz, _vpp]),
    "rtpb_moe_slot": (_int, [_vp, _sz, C.POINTER(_i64), C.POINTER(_i64)]),
    "rtpb_moe_read_shard": (_int, [_vp, _sz, _int, C.POINTER(_dbl)]),
    "rtpb_moe_gate_grad": (_int, [_vp, _sz, C.POINTER(_dbl)]),
    "rtpb_linear_set_option": (_int, [_vp, _int, _int]),
    "rtpb_mlp_set_option": (_int, [_vp, _int, _int]),
    "rtpb_add": (_int, [_int, _vp, _vp, _vp, _sz, _vp]),
    "rtpb_model_create": (_int, [_vp, _sz, _sz, _sz, _sz, _sz, _sz, _int, _u64, _int, _int, _vpp]),
    "rtpb_model_destroy": (_int, [_vp]),
    "rtpb_model_begin_step": (_int, [_vp]),
    "rtpb_model_zero_grads": (_int, [_vp]),
    "rtpb_model_forward": (_int, [_vp, _vpp, C.POINTER(_sz), _vpp, _int]),
    "rtpb_model_backward": (_int, [_vp, _vpp, _sz]),
    "rtpb_model_layer_count": (_sz, [_vp]),
    "rtpb_model_layer_shard_len": (_sz, [_vp, _sz]),
    "rtpb_model_read_layer_shard": (_int, [_vp, _sz, _sz, _int, C.POINTER(_dbl)]),
    "rtpb_model_gate_grad": (_int, [_vp, _sz, _sz, C.POINTER(_dbl)]),
    "rtpb_wgrad_step_ex": (_int, [_int, _vp, _sz, _vp, _sz, _sz, _vp, _vp, _sz, _sz, _sz, _int, _vp, _sz, _vp]),
}


class RtpError(RuntimeError):
    """Base of the reference's exception taxonomy (errors.hpp:8-33)."""

    code = 1


class ConfigError(RtpError, ValueError):
    code = 2


class DimensionError(RtpError, ValueError):
    code = 3


class ProtocolError(RtpError):
    code = 4


class StateError(RtpError):
    code = 5


class IndexError_(RtpError, IndexError):
    code = 6


class CudaError(RtpError):
    code = 7


class NcclError(RtpError):
    code = 8


_BY_CODE = {c.code: c for c in (RtpError, ConfigError, DimensionError, ProtocolError, StateError, IndexError_,
                                CudaError, NcclError)}


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `make lib` (or __graft_entry__.build()); "
                          "there is no CPU fallback for the RTP hot path")
    lib = C.CDLL(LIB_PATH)
    missing = []
    for name, (res, args) in _SIGS.items():
        try:
            fn = getattr(lib, name)
        except AttributeError:
            missing.append(name)
            continue
        fn.restype = res
        fn.argtypes = args
    if missing:
        raise ImportError(f"{LIB_PATH} lacks exports {missing}; rebuild with `make lib`")
    return lib


lib = _load()


def check(rc: int) -> None:
    if rc != RTPB_OK:
        msg = lib.rtpb_last_error().decode(errors="replace")
        raise _BY_CODE.get(rc, RtpError)(msg)


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (or None)."""
    return None if t is None else t.data_ptr()


def ptr_array(tensors) -> C.Array:
    arr = (C.c_void_p * len(tensors))()
    for i, t in enumerate(tensors):
        arr[i] = None if t is None else (t if isinstance(t, int) else t.data_ptr())
    return arr
