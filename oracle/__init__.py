"""TEST INFRASTRUCTURE ONLY — ctypes loaders for the CPU checkers.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline / --impl
reference legs may import this package.  Libraries:

* ``libcosine_oracle.so`` — the plain-C float64 restatement (cosine_oracle.c),
  citing /root/reference/proj/src/attention.cpp line by line;
* ``_ref/libcosrec_ref.so`` — the unmodified reference operator compiled from
  its own sources (oracle/Makefile) behind ref_shim.cpp's extern "C" calls,
  with -O2 -ffp-contract=off (the bit-exact parity pin);
* ``_ref/libcosrec_ref_release.so`` — the same sources with the reference's
  stock Release flags (-O3 -DNDEBUG): the timed CPU baseline.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "libcosine_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libcosrec_ref.so")
# the same sources with the reference's stock Release flags (-O3 -DNDEBUG,
# proj/CMakeLists.txt:5-7): what bench.py times as the CPU baseline
REF_RELEASE_SO = os.path.join(HERE, "_ref", "libcosrec_ref_release.so")

_vp, _sz, _i64, _dbl = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int64, ctypes.c_double
_o = None
_r = {}


def _oracle():
    global _o
    if _o is None:
        if not os.path.exists(ORACLE_SO):
            raise ImportError(f"{ORACLE_SO} missing: run `make -C oracle`")
        lib = ctypes.CDLL(ORACLE_SO)
        lib.cos_oracle_fwd.argtypes = [_vp, _vp, _vp, _vp, _sz, _sz, _dbl, _dbl] + [_vp] * 6
        lib.cos_oracle_fwd_bwd.argtypes = [_vp, _vp, _vp, _vp, _sz, _sz, _dbl, _dbl] + [_vp] * 6
        lib.cos_oracle_naive.argtypes = [_vp, _vp, _vp, _sz, _sz, _dbl, _dbl, _vp]
        lib.cos_oracle_batched_f32.argtypes = ([_vp] * 5 + [_i64] * 8 + [_dbl, _dbl] + [_vp] * 5)
        for f in ("cos_oracle_fwd", "cos_oracle_fwd_bwd", "cos_oracle_naive",
                  "cos_oracle_batched_f32"):
            getattr(lib, f).restype = ctypes.c_int
        _o = lib
    return _o


def ref_available(release=False) -> bool:
    return os.path.exists(REF_RELEASE_SO if release else REF_SO)


def _ref(release=False):
    if release not in _r:
        path = REF_RELEASE_SO if release else REF_SO
        if not os.path.exists(path):
            raise ImportError(f"{path} missing: run `make -C oracle` where /root/reference exists")
        lib = ctypes.CDLL(path)
        lib.cosref_fwd.argtypes = [_vp, _vp, _vp, _vp, _i64, _i64, _dbl, _dbl, _i64] + [_vp] * 7
        lib.cosref_fwd_bwd.argtypes = [_vp, _vp, _vp, _vp, _i64, _i64, _dbl, _dbl, _i64] + [_vp] * 6
        lib.cosref_naive.argtypes = [_vp, _vp, _vp, _i64, _i64, _dbl, _dbl, _vp]
        lib.cosref_bwd_without_cache.argtypes = [_i64, _i64]
        lib.cosref_batched_f32.argtypes = ([_vp] * 5 + [_i64] * 8 + [_dbl, _dbl, _i64]
                                           + [_vp] * 5 + [ctypes.c_int])
        lib.cosref_last_error.restype = ctypes.c_char_p
        for f in ("cosref_fwd", "cosref_fwd_bwd", "cosref_naive", "cosref_bwd_without_cache",
                  "cosref_batched_f32", "cosref_hardware_threads"):
            getattr(lib, f).restype = ctypes.c_int
        _r[release] = lib
    return _r[release]


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _d(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _mask(valid):
    return None if valid is None else np.ascontiguousarray(valid, dtype=np.uint8)


class OracleError(RuntimeError):
    pass


def _rc(rc, lib=None):
    if rc != 0:
        msg = lib.cosref_last_error().decode() if lib is not None else ""
        raise OracleError(f"oracle rc={rc} {msg}")


# ---- C restatement -----------------------------------------------------------

def fwd(q, k, v, valid=None, m=1.0, eps=1e-6):
    """cosine_attention_fused with a full cache; returns dict of float64 arrays."""
    q, k, v = _d(q), _d(k), _d(v)
    n, d = q.shape
    r = {"out": np.empty((n, d)), "norm_q": np.empty(n), "norm_k": np.empty(n),
         "qn": np.empty((n, d)), "kn": np.empty((n, d)), "S": np.empty((d, d))}
    _rc(_oracle().cos_oracle_fwd(_p(q), _p(k), _p(v), _p(_mask(valid)), n, d, m, eps,
                                 _p(r["out"]), _p(r["norm_q"]), _p(r["norm_k"]), _p(r["qn"]),
                                 _p(r["kn"]), _p(r["S"])))
    return r


def fwd_bwd(q, k, v, d_out, valid=None, m=1.0, eps=1e-6):
    """Forward + backward of one unit; returns (out, dq, dk, dv, dm)."""
    q, k, v, g = _d(q), _d(k), _d(v), _d(d_out)
    n, d = q.shape
    out, dq, dk, dv = (np.empty((n, d)) for _ in range(4))
    dm = np.zeros(1)
    _rc(_oracle().cos_oracle_fwd_bwd(_p(q), _p(k), _p(v), _p(_mask(valid)), n, d, m, eps, _p(g),
                                     _p(out), _p(dq), _p(dk), _p(dv), _p(dm)))
    return out, dq, dk, dv, float(dm[0])


def naive(q, k, v, m=1.0, eps=1e-6):
    q, k, v = _d(q), _d(k), _d(v)
    n, d = q.shape
    out = np.empty((n, d))
    _rc(_oracle().cos_oracle_naive(_p(q), _p(k), _p(v), n, d, m, eps, _p(out)))
    return out


def batched_f32(q, k, v, d_out=None, valid=None, m=1.0, eps=1e-6):
    """Whole [B,H,N,D] float32 batch (contiguous) through the C restatement in
    float64.  Returns (out, dq, dk, dv, dm_unit) as float64 arrays (grads None
    without d_out)."""
    q = np.ascontiguousarray(q, np.float32)
    k = np.ascontiguousarray(k, np.float32)
    v = np.ascontiguousarray(v, np.float32)
    g = None if d_out is None else np.ascontiguousarray(d_out, np.float32)
    B, H, N, D = q.shape
    out = np.empty(q.shape)
    dq = dk = dv = None
    if g is not None:
        dq, dk, dv = np.empty(q.shape), np.empty(q.shape), np.empty(q.shape)
    dm = np.zeros(B * H)
    vm = _mask(valid)
    msb = 0 if vm is None else vm.shape[1]
    _rc(_oracle().cos_oracle_batched_f32(_p(q), _p(k), _p(v), _p(g), _p(vm), B, H, N, D,
                                         H * N * D, N * D, D, msb, m, eps, _p(out), _p(dq),
                                         _p(dk), _p(dv), _p(dm)))
    return out, dq, dk, dv, dm


# ---- the reference itself (oracle/_ref) ---------------------------------------

def ref_fwd(q, k, v, valid=None, m=1.0, eps=1e-6, tile=32):
    q, k, v = _d(q), _d(k), _d(v)
    n, d = q.shape
    r = {"out": np.empty((n, d)), "norm_q": np.empty(n), "norm_k": np.empty(n),
         "qn": np.empty((n, d)), "kn": np.empty((n, d)), "S": np.empty((d, d))}
    tn = np.zeros(1, np.int64)
    lib = _ref()
    _rc(lib.cosref_fwd(_p(q), _p(k), _p(v), _p(_mask(valid)), n, d, m, eps, tile, _p(r["out"]),
                       _p(r["norm_q"]), _p(r["norm_k"]), _p(r["qn"]), _p(r["kn"]), _p(r["S"]),
                       _p(tn)), lib)
    r["true_n"] = int(tn[0])
    return r


def ref_fwd_bwd(q, k, v, d_out, valid=None, m=1.0, eps=1e-6, tile=32):
    q, k, v, g = _d(q), _d(k), _d(v), _d(d_out)
    n, d = q.shape
    out, dq, dk, dv = (np.empty((n, d)) for _ in range(4))
    dm = np.zeros(1)
    lib = _ref()
    _rc(lib.cosref_fwd_bwd(_p(q), _p(k), _p(v), _p(_mask(valid)), n, d, m, eps, tile, _p(g),
                           _p(out), _p(dq), _p(dk), _p(dv), _p(dm)), lib)
    return out, dq, dk, dv, float(dm[0])


def ref_naive(q, k, v, m=1.0, eps=1e-6):
    q, k, v = _d(q), _d(k), _d(v)
    n, d = q.shape
    out = np.empty((n, d))
    lib = _ref()
    _rc(lib.cosref_naive(_p(q), _p(k), _p(v), n, d, m, eps, _p(out)), lib)
    return out


def ref_error_code(fn_name, *args):
    """Return code of a shim call expected to raise inside the reference."""
    return getattr(_ref(), fn_name)(*args)


def ref_hardware_threads() -> int:
    return int(_ref().cosref_hardware_threads())


def ref_batched_f32(q, k, v, d_out, valid, m=1.0, eps=1e-6, threads=0, outputs=None, tile=32,
                    release=False):
    """The reference operator over a contiguous float32 [B,H,N,D] batch on a
    persistent thread pool (threads <= 0: all host threads).  release=True
    uses the Release-flag build (the timed CPU baseline)."""
    B, H, N, D = q.shape
    if outputs is None:
        outputs = tuple(np.empty(q.shape, np.float32) for _ in range(4)) + (np.zeros(B * H),)
    out, dq, dk, dv, dm = outputs
    vm = _mask(valid)
    msb = 0 if vm is None else vm.shape[1]
    lib = _ref(release)
    _rc(lib.cosref_batched_f32(_p(q), _p(k), _p(v), _p(d_out), _p(vm), B, H, N, D, H * N * D,
                               N * D, D, msb, m, eps, tile, _p(out), _p(dq), _p(dk), _p(dv),
                               _p(dm), int(threads)), lib)
    return outputs
