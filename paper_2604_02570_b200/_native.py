"""ctypes binding of the C ABI in include/wsvd_b200.h (libwsvd_b200.so).

The library is built in-tree (paper_2604_02570_b200/build.py).  There is no
fallback: importing the package works everywhere, but every call that needs
the native library raises if it is missing, and every compute entry point
returns WSVD_ECUDA on a machine without an sm_100 device.
"""
from __future__ import annotations

import ctypes as C
import os

from .errors import ConfigError, CudaError, IoError, NumericError, ShapeError, WsvdError

LIB_PATH = os.environ.get("WSVD_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libwsvd_b200.so")

F32, BF16, I8, I4 = 0, 1, 2, 3
DTYPES = {"f32": F32, "bf16": BF16, "i8": I8, "i4": I4}

OK, ESHAPE, ECONFIG, ENUMERIC, ECUDA, EIO, ENCCL = 0, -1, -2, -3, -4, -5, -6


class LayerDesc(C.Structure):
    _fields_ = [("embed_dim", C.c_int32), ("head_dim", C.c_int32), ("n_heads", C.c_int32),
                ("head_offset", C.c_int32), ("weight_dtype", C.c_int32),
                ("act_rotation", C.c_int32), ("device", C.c_int32)]


# every exported symbol and its ctypes signature (restype, argtypes)
_vp, _i32, _i64, _fp, _dp = C.c_void_p, C.c_int32, C.c_int64, C.c_void_p, C.POINTER(C.c_double)
_u64p, _u8p, _i8p, _i32p = (C.POINTER(C.c_uint64), C.POINTER(C.c_uint8), C.POINTER(C.c_int8),
                            C.POINTER(C.c_int32))
SIGNATURES = {
    "wsvd_last_error": (C.c_char_p, []),
    "wsvd_abi_version": (C.c_int, []),
    "wsvd_device_count": (C.c_int, [_i32p]),
    "wsvd_layer_create": (C.c_int, [C.POINTER(LayerDesc), _i32p, C.POINTER(_vp)]),
    "wsvd_layer_destroy": (C.c_int, [_vp]),
    "wsvd_layer_rank_pad": (C.c_int, [_vp, _i32p]),
    "wsvd_layer_set_head": (C.c_int, [_vp, _i32, _i32, _dp, _dp]),
    "wsvd_layer_set_head_quantized": (C.c_int, [_vp, _i32, _i32, _i8p, _dp, _i8p, _dp]),
    "wsvd_layer_set_oproj": (C.c_int, [_vp, _dp, _i32, _i32]),
    "wsvd_cache_create": (C.c_int, [_vp, _i32, _i32, _i32, C.POINTER(_vp)]),
    "wsvd_cache_destroy": (C.c_int, [_vp]),
    "wsvd_cache_reset": (C.c_int, [_vp]),
    "wsvd_cache_bind_layer": (C.c_int, [_vp, _vp]),
    "wsvd_cache_length": (C.c_int, [_vp, _i32p]),
    "wsvd_cache_push_host": (C.c_int, [_vp, _dp, _dp]),
    "wsvd_cache_read_host": (C.c_int, [_vp, _i32, _i32, _dp, _dp]),
    "wsvd_cache_row_bytes": (C.c_int, [_vp, _i32p]),
    "wsvd_cache_step_info": (C.c_int, [_vp, _i32p, _i32p]),
    "wsvd_cache_sync_length": (C.c_int, [_vp, _i32p]),
    "wsvd_ckpt_info": (C.c_int, [C.c_char_p, C.POINTER(C.c_int64)]),
    "wsvd_ckpt_head": (C.c_int, [C.c_char_p, _i32, _i32, _i32, _i32p, _dp, _dp]),
    "wsvd_ckpt_head_quantized": (C.c_int, [C.c_char_p, _i32, _i32, _i32, _i32p, _i8p, _dp, _i8p, _dp]),
    "wsvd_ckpt_weight": (C.c_int, [C.c_char_p, C.c_char_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64), _dp]),
    "wsvd_layer_load_checkpoint": (C.c_int, [C.c_char_p, _i32, _i32, _i32, _i32, _i32, _i32, C.POINTER(_vp)]),
    "wsvd_cache_fill_synthetic": (C.c_int, [_vp, _i32, C.c_uint64, C.c_float]),
    "wsvd_cache_set_attention_mode": (C.c_int, [_vp, _i32]),
    "wsvd_cache_attention_mode": (C.c_int, [_vp, _i32p]),
    "wsvd_cache_read_raw": (C.c_int, [_vp, _i32, _i32, _vp, _vp]),
    "wsvd_append_token": (C.c_int, [_vp, _fp, _fp, _vp]),
    "wsvd_prefill": (C.c_int, [_vp, _fp, _i32, _vp]),
    "wsvd_fused_decode_step": (C.c_int, [_vp, _fp, _i32, _fp, _vp]),
    "wsvd_decode_attention": (C.c_int, [_vp, _fp, _vp]),
    "wsvd_layer_step": (C.c_int, [_vp, _fp, _fp, _fp, _vp]),
    "wsvd_layer_step_host": (C.c_int, [_vp, _fp, _fp, _vp]),
    "wsvd_layer_step_graph": (C.c_int, [_vp, _fp, _fp, _vp]),
    "wsvd_cache_debug_copy": (C.c_int, [_vp, _i32, _vp, C.POINTER(C.c_int64)]),
    "wsvd_quantize_weight": (C.c_int, [C.POINTER(C.c_double), _i64, _i64, _i32, _i8p,
                                       C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "wsvd_traffic_append": (C.c_int, [_vp, _u64p]),
    "wsvd_traffic_fused": (C.c_int, [_vp, _i32, _u64p]),
    "wsvd_nccl_unique_id": (C.c_int, [_u8p]),
    "wsvd_comm_create": (C.c_int, [_u8p, _i32, _i32, _i32, C.POINTER(_vp)]),
    "wsvd_comm_destroy": (C.c_int, [_vp]),
    "wsvd_allreduce_sum_f32": (C.c_int, [_vp, _fp, _i64, _vp]),
    "wsvd_cache_grow": (C.c_int, [_vp, _i32]),
    "wsvd_cache_capacity": (C.c_int, [_vp, _i32p]),
    "wsvd_cache_set_debug": (C.c_int, [_vp, _i32]),
    "wsvd_dense_cache_create": (C.c_int, [_i32, _i32, _i32, C.POINTER(_vp)]),
    "wsvd_dense_cache_destroy": (C.c_int, [_vp]),
    "wsvd_dense_cache_length": (C.c_int, [_vp, _i32p]),
    "wsvd_dense_cache_append": (C.c_int, [_vp, _fp, _fp, _vp]),
    "wsvd_dense_cache_read_host": (C.c_int, [_vp, _i32, _dp, _dp]),
    "wsvd_dense_decode_step": (C.c_int, [_vp, _fp, _i32, _fp, _vp]),
    "wsvd_dense_attend": (C.c_int, [_fp, _fp, _i32, _i32, _i32, _i32, _fp, _fp, _fp, _vp]),
    "wsvd_vecmat_f32": (C.c_int, [_fp, _fp, _i32, _i32, _fp, _vp]),
    "wsvd_matmul_f32": (C.c_int, [_fp, _fp, _i32, _i32, _i32, _fp, _vp]),
    "wsvd_chain_step": (C.c_int, [C.POINTER(_vp), _i32, _fp, C.POINTER(_vp), _vp]),
    "wsvd_chain_step_host": (C.c_int, [C.POINTER(_vp), _i32, _fp, _fp, _vp]),
    "wsvd_ffn_create": (C.c_int, [_i32, _i32, _fp, _fp, _i32, C.POINTER(_vp)]),
    "wsvd_ffn_destroy": (C.c_int, [_vp]),
    "wsvd_ffn_forward": (C.c_int, [_vp, _fp, _i32, _fp, _vp]),
}

_lib = None


def lib():
    """Load libwsvd_b200.so (raises loudly when it was never built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2604_02570_b200.build` "
                "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


_EXC = {ESHAPE: ShapeError, ECONFIG: ConfigError, ENUMERIC: NumericError, ECUDA: CudaError,
        EIO: IoError, ENCCL: CudaError}


def check(rc: int) -> None:
    if rc != OK:
        msg = lib().wsvd_last_error().decode(errors="replace")
        raise _EXC.get(rc, WsvdError)(msg)


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args))


def device_count() -> int:
    n = C.c_int32(0)
    call("wsvd_device_count", C.byref(n))
    return n.value
