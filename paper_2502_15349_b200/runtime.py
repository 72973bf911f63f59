"""ctypes binding of the C ABI declared in ``include/attn_b200.h``.

This is the only place Python touches the native library.  Structures mirror the header field by
field; every call checks the returned status and re-raises it as the attnforge-style exception of
the matching kind (``errors.py:30-82`` of the reference).  There is no fallback: if the library is
missing the import of :func:`lib` raises.
"""

from __future__ import annotations

import ctypes as C
import threading
from pathlib import Path

from . import errors

_LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libattn_b200.so"

AF_OK, AF_ERR_INPUT, AF_ERR_SHAPE, AF_ERR_UNSUPPORTED, AF_ERR_NAN, AF_ERR_CUDA = range(6)
AF_FAMILY_SOFTMAX, AF_FAMILY_ELEMENTWISE, AF_FAMILY_ABSSUM = 0, 1, 2
AF_ACT_IDENTITY, AF_ACT_SIGMOID, AF_ACT_RELU, AF_ACT_RELU2 = 0, 1, 2, 3
AF_DTYPE_BF16, AF_DTYPE_F32 = 0, 1
AF_BWD_DEFAULT, AF_BWD_SPLIT, AF_BWD_FUSED = 0, 1, 2
AF_ROWNORM_NONE, AF_ROWNORM_SOFTMAX, AF_ROWNORM_ABSSUM = 0, 1, 2
AF_FM_NONE, AF_FM_SILU, AF_FM_SIGMOID, AF_FM_RELU, AF_FM_TANH, AF_FM_EXP = range(6)

I64x4 = C.c_int64 * 4


class ParallelDesc(C.Structure):
    _fields_ = [
        ("batch", C.c_int32), ("heads_q", C.c_int32), ("heads_kv", C.c_int32),
        ("seq_q", C.c_int32), ("seq_k", C.c_int32), ("d_qk", C.c_int32), ("d_v", C.c_int32),
        ("dtype", C.c_int32),
        ("q_stride", I64x4), ("k_stride", I64x4), ("v_stride", I64x4), ("o_stride", I64x4),
        ("family", C.c_int32), ("act", C.c_int32), ("scale", C.c_float),
        ("causal", C.c_int32), ("diag_offset", C.c_int32), ("window", C.c_int32),
        ("slope", C.c_void_p), ("bias", C.c_float), ("cap_a", C.c_float), ("cap_b", C.c_float),
        ("kv_stages", C.c_int32), ("head_groups", C.c_int32), ("bwd_mode", C.c_int32),
    ]


I64x3 = C.c_int64 * 3


class LinearDesc(C.Structure):
    _fields_ = [
        ("batch", C.c_int32), ("heads", C.c_int32), ("seq", C.c_int32), ("d_k", C.c_int32),
        ("d_v", C.c_int32), ("chunk", C.c_int32), ("q_scale", C.c_float),
        ("q_stride", I64x4), ("k_stride", I64x4), ("v_stride", I64x4), ("o_stride", I64x4),
        ("log_decay_const", C.c_float), ("n_decay_factors", C.c_int32),
        ("decay_factor", C.c_void_p * 2), ("decay_factor_stride", I64x3 * 2),
        ("key_gate", C.c_void_p), ("key_gate_stride", I64x3), ("decay_hint", C.c_int32),
    ]


class MlaDesc(C.Structure):
    _fields_ = [
        ("batch", C.c_int32), ("heads", C.c_int32), ("seq_k", C.c_int32), ("d_qk", C.c_int32),
        ("d_v", C.c_int32), ("scale", C.c_float), ("splits", C.c_int32),
    ]


# Every symbol include/attn_b200.h declares, with its ctypes signature.
P = C.c_void_p
SIGNATURES: dict[str, tuple] = {
    "af_parallel_fwd": (C.c_int, [C.POINTER(ParallelDesc), P, P, P, P, P, P]),
    "af_parallel_bwd_workspace": (C.c_size_t, [C.POINTER(ParallelDesc)]),
    "af_parallel_bwd": (C.c_int, [C.POINTER(ParallelDesc), P, P, P, P, P, P, P, P, P, P,
                                  C.c_size_t, P]),
    "af_linear_fwd_workspace": (C.c_size_t, [C.POINTER(LinearDesc)]),
    "af_linear_fwd": (C.c_int, [C.POINTER(LinearDesc), P, P, P, P, P, P, C.c_size_t, P]),
    "af_linear_step": (C.c_int, [C.POINTER(LinearDesc), P, P, P, P, P, P]),
    "af_linear_bwd_workspace": (C.c_size_t, [C.POINTER(LinearDesc)]),
    "af_linear_bwd": (C.c_int, [C.POINTER(LinearDesc), P, P, P, P, P, P, P, P, P, P, C.c_size_t,
                                P]),  # (desc, q, k, v, dout, dq, dk, dv, d_factor**, d_gate, ws..)
    "af_mla_decode_workspace": (C.c_size_t, [C.POINTER(MlaDesc)]),
    "af_mla_decode": (C.c_int, [C.POINTER(MlaDesc), P, P, P, P, P, C.c_size_t, P]),
    "af_feature_map": (C.c_int, [C.c_int, C.c_int, P, P, P, C.c_int64, P]),
    "af_hook_eval": (C.c_int, [P, P, P, C.c_int32, C.c_int32, P, P, P, P]),
    "af_rownorm_fwd": (C.c_int, [C.c_int32, P, P, P, C.c_int64, C.c_int64, P]),
    "af_rownorm_bwd": (C.c_int, [C.c_int32, P, P, P, P, P, P, C.c_int64, C.c_int64, P]),
    "af_rowdot": (C.c_int, [P, P, P, P, P]),
    "af_status_string": (C.c_char_p, [C.c_int]),
    "af_last_error": (C.c_char_p, []),
    "af_device_sm_count": (C.c_int, []),
    "af_launch_count": (C.c_uint64, []),
}

_lock = threading.Lock()
_lib: C.CDLL | None = None


def library_path() -> Path:
    return _LIB_PATH


def lib() -> C.CDLL:
    """Load the sm_100a library (raises if it was never built — no fallback path exists)."""
    global _lib
    with _lock:
        if _lib is None:
            if not _LIB_PATH.exists():
                raise errors.UnsupportedError(
                    "native library missing; run __graft_entry__.build()", path=str(_LIB_PATH))
            handle = C.CDLL(str(_LIB_PATH))
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(handle, name)
                fn.restype = res
                fn.argtypes = args
            _lib = handle
    return _lib


_STATUS_ERR = {
    AF_ERR_INPUT: errors.InputError,
    AF_ERR_SHAPE: errors.ShapeError,
    AF_ERR_UNSUPPORTED: errors.UnsupportedError,
    AF_ERR_NAN: errors.NanError,
    AF_ERR_CUDA: errors.DeviceError,
}


def check(status: int, what: str) -> None:
    if status == AF_OK:
        return
    msg = lib().af_last_error().decode(errors="replace")
    raise _STATUS_ERR.get(status, errors.DeviceError)(f"{what}: {msg}", status=status)


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def strides4(t) -> I64x4:
    return I64x4(*[int(s) for s in t.stride()])


def step_strides(t) -> I64x3:
    """[b, h, s] element strides of a rank-4 per-step tensor [B|1, H|1, S, 1] (0 = broadcast)."""
    return I64x3(*[0 if t.shape[i] == 1 else int(t.stride(i)) for i in range(3)])


def launch_count() -> int:
    """Kernels the native library has launched in this process (its own counter)."""
    return int(lib().af_launch_count())
