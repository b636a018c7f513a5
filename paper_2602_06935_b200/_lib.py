"""ctypes binding of the C-ABI in include/cotten.h (libcotten.so, built in-tree).

There is no fallback: if the CUDA library is missing the import fails loudly,
and every call that reaches a kernel needs a CUDA device.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# COTTEN_LIB overrides the in-tree library (A/B builds of kernel variants).
LIB_PATH = os.environ.get("COTTEN_LIB") or os.path.join(_HERE, "libcotten.so")

COTTEN_OK = 0
COTTEN_ERR_INTERNAL = 1
COTTEN_ERR_USAGE = 2
COTTEN_ERR_NUMERIC = 4

F32, BF16, F64 = 0, 1, 2
DTYPES = {"f32": F32, "float32": F32, "bf16": BF16, "bfloat16": BF16, "f64": F64, "float64": F64}

FLAG_FORCE_GENERIC = 1
FLAG_FP32_PIPE = 2  # d_h=32 fp32: the FP32-pipe kernels instead of the tcgen05 ones
STATUS_EMPTY_SEQUENCE = 1


class UsageError(RuntimeError):
    """The reference's cosrec::UsageError (errors.hpp:10-12)."""


class ShapeError(UsageError):
    """The reference's cosrec::ShapeError (errors.hpp:14-16)."""


class NumericError(RuntimeError):
    """The reference's cosrec::NumericError (errors.hpp:22-24)."""


class CottenError(RuntimeError):
    """Internal / CUDA failure (COTTEN_ERR_INTERNAL)."""


class CottenDesc(ctypes.Structure):
    _fields_ = [
        ("batch", ctypes.c_int64),
        ("heads", ctypes.c_int64),
        ("seq_len", ctypes.c_int64),
        ("head_dim", ctypes.c_int64),
        ("dtype", ctypes.c_int32),
        ("flags", ctypes.c_int32),
        ("eps", ctypes.c_double),
        ("stride_b", ctypes.c_int64),
        ("stride_h", ctypes.c_int64),
        ("stride_n", ctypes.c_int64),
        ("mask_stride_b", ctypes.c_int64),
    ]


def make_desc(B, H, N, D, dtype="f32", eps=1e-6, strides=(0, 0, 0), mask_stride_b=0, flags=0):
    if isinstance(dtype, str):
        dtype = DTYPES[dtype]
    return CottenDesc(int(B), int(H), int(N), int(D), int(dtype), int(flags), float(eps),
                      int(strides[0]), int(strides[1]), int(strides[2]), int(mask_stride_b))


# Every exported symbol of include/cotten.h with its ctypes signature.
_vp, _i32, _i64, _dbl = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
_DP = ctypes.POINTER(CottenDesc)
SIGNATURES = {
    "cotten_version": (ctypes.c_char_p, []),
    "cotten_last_error": (ctypes.c_char_p, []),
    "cotten_last_launch_count": (ctypes.c_int, []),
    "cotten_fwd": (ctypes.c_int, [_DP, _vp, _vp, _vp, _vp, _dbl, _vp, _vp, _vp, _vp]),
    "cotten_bwd": (ctypes.c_int, [_DP, _vp, _vp, _vp, _vp, _dbl, _vp, _vp, _vp, _vp, _vp, _vp,
                                  _vp, _vp]),
    "cotten_fwd_mdev": (ctypes.c_int, [_DP, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "cotten_bwd_mdev": (ctypes.c_int, [_DP, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                       _vp, _vp, _vp]),
    "cotten_device_status": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(_i32), ctypes.c_int]),
    "cotten_fwd_host": (ctypes.c_int, [_DP, _vp, _vp, _vp, _vp, _dbl, _vp, _vp, _vp]),
    "cotten_bwd_host": (ctypes.c_int, [_DP, _vp, _vp, _vp, _vp, _dbl, _vp, _vp, _vp, _vp, _vp,
                                       _vp, _vp]),
    "cotten_fwd_bwd_host": (ctypes.c_int, [_DP, _vp, _vp, _vp, _vp, _dbl, _vp, _vp, _vp, _vp,
                                           _vp, _vp]),
    "cotten_fwd_host_cached": (ctypes.c_int, [_DP, _vp, _vp, _vp, _vp, _dbl, _vp, _vp,
                                              ctypes.POINTER(_vp)]),
    "cotten_bwd_host_cached": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "cotten_host_cache_free": (ctypes.c_int, [_vp]),
    "cotten_profile_begin": (ctypes.c_int, [_vp, ctypes.c_int]),
    "cotten_profile_end": (ctypes.c_int, []),
}

_lib = None


def load(path: str = LIB_PATH):
    """Load libcotten.so (raises ImportError with the build hint if absent)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(
            f"{path} not built: run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback for the cosine-attention operator)")
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int):
    """Map a C-ABI return code to the reference's exception taxonomy."""
    if rc == COTTEN_OK:
        return
    msg = (load().cotten_last_error() or b"").decode(errors="replace")
    if rc == COTTEN_ERR_USAGE:
        low = msg.lower()
        if "shape" in low or "empty matrix" in low or "mask length" in low or "stride" in low:
            raise ShapeError(msg)
        raise UsageError(msg)
    if rc == COTTEN_ERR_NUMERIC:
        raise NumericError(msg)
    raise CottenError(f"cotten error {rc}: {msg}")


def launches() -> int:
    return int(load().cotten_last_launch_count())
