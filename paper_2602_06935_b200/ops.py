"""Host-side mirror of the reference operator interface, over the C-ABI.

Same names, argument meaning and error behaviour as
/root/reference/proj/include/cosrec/attention.hpp:11-93:

    cosine_attention_fused(q, k, v, m, cfg, cache=None, mask=None)  (:84-86)
    cosine_attention_backward(cache, d_out)                         (:87)
    attention_forward / attention_backward                          (:90-93)
    AttentionConfig, RowMask, AttentionCache, AttentionGrads        (:16-59)

A reference ``Matrix`` (row-major float64, matrix.hpp:10-13) is a 2-D numpy
array here.  The math runs on the GPU through ``cotten_fwd_host`` /
``cotten_bwd_host`` in ``cfg.dtype`` (default "f64", so the reference's own
1e-10 tolerances apply unchanged; "f32" / "bf16" select the fast paths).

``forward`` / ``backward`` are the batched device entry points for torch
tensors laid out [B, H, N, D] (any strides with a contiguous last dim, so a
[B, N, H, D] projection output can be passed as a permuted view).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib
from ._lib import ShapeError, UsageError, check, load, make_desc

MECHANISMS = ("softmax", "elu_linear", "cosine")


def mechanism_from_string(name: str) -> str:
    """attention.cpp:10-15"""
    if name not in MECHANISMS:
        raise UsageError("unknown mechanism: " + name)
    return name


@dataclass
class AttentionConfig:
    """attention.hpp:16-23 (+ dtype: the device arithmetic type)."""
    mechanism: str = "cosine"
    eps: float = 1e-6
    alpha: float = 1.0
    tile_size: int = 32
    heads: int = 2
    linear_denominator: bool = True
    dtype: str = "f64"


@dataclass
class RowMask:
    """attention.hpp:27-32; from_valid counts the real rows (attention.cpp:26-33)."""
    valid: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint8))
    true_count: int = 0

    @staticmethod
    def from_valid(v) -> "RowMask":
        arr = np.ascontiguousarray(np.asarray(v, dtype=np.uint8))
        return RowMask(arr, int(np.count_nonzero(arr)))


@dataclass
class AttentionCache:
    """attention.hpp:35-54 (cosine fields)."""
    mechanism: Optional[str] = None
    q: Optional[np.ndarray] = None
    k: Optional[np.ndarray] = None
    v: Optional[np.ndarray] = None
    valid: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint8))
    true_n: int = 0
    eps: float = 0.0
    qn: Optional[np.ndarray] = None
    kn: Optional[np.ndarray] = None
    norm_q: Optional[np.ndarray] = None
    norm_k: Optional[np.ndarray] = None
    kv: Optional[np.ndarray] = None
    m: float = 1.0
    dtype: str = "f64"


@dataclass
class AttentionGrads:
    """attention.hpp:56-59"""
    dq: np.ndarray
    dk: np.ndarray
    dv: np.ndarray
    dm: float = 0.0


_NP = {"f32": np.float32, "f64": np.float64}


def _host(x, dt):
    if dt == "bf16":
        # bf16 host buffers: round-to-nearest-even from float32, as uint16 bits.
        f = np.ascontiguousarray(np.asarray(x, dtype=np.float32))
        bits = f.view(np.uint32).astype(np.uint64)
        rounded = ((bits + 0x7FFF + ((bits >> 16) & 1)) >> 16).astype(np.uint16)
        return rounded
    return np.ascontiguousarray(np.asarray(x, dtype=_NP[dt]))


def _from_host(x, dt):
    if dt == "bf16":
        return (x.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    return np.asarray(x, dtype=np.float64)


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _check_qkv(q, k, v, mask, what):
    """check_qkv (attention.cpp:37-46) + require_nonempty/same_shape (matrix.cpp:24-31)."""
    for x in (q, k, v):
        if x is None or x.ndim != 2 or x.shape[0] == 0 or x.shape[1] == 0:
            raise ShapeError(what + ": empty matrix")
    if q.shape != k.shape or q.shape != v.shape:
        raise ShapeError(what + ": shape mismatch")
    if mask is not None:
        if mask.valid.shape[0] != q.shape[0]:
            raise ShapeError(what + ": mask length")
        if mask.true_count == 0:
            raise UsageError(what + ": no real rows")


def cosine_attention_fused(q, k, v, m: float, cfg: AttentionConfig,
                           cache: Optional[AttentionCache] = None,
                           mask: Optional[RowMask] = None) -> np.ndarray:
    """attention.cpp:297-395 on the GPU; fills ``cache`` like :308-322,390-393."""
    q, k, v = (np.asarray(x, dtype=np.float64) for x in (q, k, v))
    _check_qkv(q, k, v, mask, "cosine_attention_fused")
    if cfg.tile_size == 0:
        raise UsageError("cosine_attention_fused: tile_size must be >= 1")
    n, d = q.shape
    dt = cfg.dtype
    lib = load()
    desc = make_desc(1, 1, n, d, dt, cfg.eps)
    hq, hk, hv = _host(q, dt), _host(k, dt), _host(v, dt)
    hout = np.empty_like(hq)
    acc = np.float64 if dt == "f64" else np.float32
    hS = np.empty((d, d), acc) if cache is not None else None
    hN = np.empty((2, n), acc) if cache is not None else None
    valid = None if mask is None else np.ascontiguousarray(mask.valid, dtype=np.uint8)
    check(lib.cotten_fwd_host(ctypes.byref(desc), _ptr(hq), _ptr(hk), _ptr(hv), _ptr(valid),
                              float(m), _ptr(hout), _ptr(hS), _ptr(hN)))
    out = _from_host(hout, dt)
    if cache is not None:
        nq = hN[0].astype(np.float64)
        nk = hN[1].astype(np.float64)
        vm = np.ones(n, bool) if valid is None else valid.astype(bool)
        qd, kd = _from_host(hq, dt), _from_host(hk, dt)
        cache.mechanism = "cosine"
        cache.q, cache.k, cache.v = q.copy(), k.copy(), v.copy()
        cache.qn = qd / nq[:, None]
        cache.kn = np.where(vm[:, None], kd / nk[:, None], 0.0)
        cache.norm_q, cache.norm_k = nq.reshape(n, 1), nk.reshape(n, 1)
        cache.kv = hS.astype(np.float64)
        cache.m, cache.eps = float(m), float(cfg.eps)
        cache.valid = np.zeros(0, np.uint8) if valid is None else valid.copy()
        cache.true_n = n if mask is None else mask.true_count
        cache.dtype = dt
    return out


def cosine_attention_backward(cache: AttentionCache, d_out) -> AttentionGrads:
    """attention.cpp:397-441 on the GPU (recomputes Q~/K~ from q, k; uses S)."""
    if cache is None or cache.mechanism != "cosine" or cache.qn is None:
        raise UsageError("cosine_attention_backward: cache missing")
    d_out = np.asarray(d_out, dtype=np.float64)
    if d_out.shape != cache.qn.shape:
        raise ShapeError("cosine_attention_backward: shape mismatch")
    n, d = d_out.shape
    dt = cache.dtype
    lib = load()
    desc = make_desc(1, 1, n, d, dt, cache.eps)
    hq, hk, hv, hg = (_host(x, dt) for x in (cache.q, cache.k, cache.v, d_out))
    acc = np.float64 if dt == "f64" else np.float32
    hS = np.ascontiguousarray(cache.kv, dtype=acc)
    valid = None if cache.valid.size == 0 else np.ascontiguousarray(cache.valid, np.uint8)
    dq, dk, dv = np.empty_like(hq), np.empty_like(hq), np.empty_like(hq)
    dm = np.zeros(1, np.float64)
    check(lib.cotten_bwd_host(ctypes.byref(desc), _ptr(hq), _ptr(hk), _ptr(hv), _ptr(valid),
                              float(cache.m), _ptr(hg), _ptr(hS), _ptr(dq), _ptr(dk), _ptr(dv),
                              None, _ptr(dm)))
    return AttentionGrads(_from_host(dq, dt), _from_host(dk, dt), _from_host(dv, dt), float(dm[0]))


def attention_forward(q, k, v, m, cfg: AttentionConfig, cache=None, mask=None):
    """attention.cpp:443-456 — only the cosine mechanism has a B200 path."""
    if cfg.mechanism == "cosine":
        return cosine_attention_fused(q, k, v, m, cfg, cache, mask)
    raise UsageError("attention_forward: mechanism '%s' is not on the B200 path" % cfg.mechanism)


def attention_backward(cache: AttentionCache, d_out):
    """attention.cpp:458-468"""
    if cache is not None and cache.mechanism == "cosine":
        return cosine_attention_backward(cache, d_out)
    if cache is None or cache.mechanism is None:
        raise UsageError("cosine_attention_backward: cache missing")
    raise UsageError("attention_backward: mechanism '%s' is not on the B200 path" % cache.mechanism)


# --------------------------------------------------------------------------
# Batched host entry points (numpy [B, H, N, D]; the e2e path of bench.py).

def fwd_bwd_host(q, k, v, valid, m, d_out, eps=1e-6, dtype="f32", out=None, dq=None, dk=None,
                 dv=None):
    """One op training step with host buffers: cotten_fwd_bwd_host.  Arrays
    must already be contiguous in the device dtype (e.g. pinned numpy views).
    Returns (out, dq, dk, dv, dm_total)."""
    B, H, N, D = q.shape
    lib = load()
    desc = make_desc(B, H, N, D, dtype, eps)
    out = np.empty_like(q) if out is None else out
    dq = np.empty_like(q) if dq is None else dq
    dk = np.empty_like(q) if dk is None else dk
    dv = np.empty_like(q) if dv is None else dv
    dm = np.zeros(1, np.float64)
    check(lib.cotten_fwd_bwd_host(ctypes.byref(desc), _ptr(q), _ptr(k), _ptr(v), _ptr(valid),
                                  float(m), _ptr(d_out), _ptr(out), _ptr(dq), _ptr(dk), _ptr(dv),
                                  _ptr(dm)))
    return out, dq, dk, dv, float(dm[0])


# --------------------------------------------------------------------------
# Device entry points for torch tensors (bench.py, tests).  torch is only the
# allocator/stream provider here; the arithmetic is libcotten.so.

def _tdesc(t, eps, flags, valid):
    import torch
    if t.dim() != 4 or t.stride(3) != 1:
        raise ShapeError("expected a [B, H, N, D] tensor with a contiguous last dim")
    dt = {torch.float32: "f32", torch.bfloat16: "bf16", torch.float64: "f64"}.get(t.dtype)
    if dt is None:
        raise UsageError("unsupported dtype %s" % t.dtype)
    B, H, N, D = t.shape
    msb = 0 if valid is None else valid.stride(0)
    return make_desc(B, H, N, D, dt, eps, (t.stride(0), t.stride(1), t.stride(2)), msb, flags)


def _same_layout(ref, *ts):
    for t in ts:
        if t is not None and (t.shape != ref.shape or t.stride() != ref.stride()
                              or t.dtype != ref.dtype or t.device != ref.device):
            raise ShapeError("shape mismatch: all operands must share shape, strides and dtype")


def _like(t):
    """An output with t's shape AND strides (storage covering t's span): the
    kernels write outputs at the inputs' strides, so a gapped q (a slice of a
    fused QKV projection) needs a gapped output, not empty_like's dense one."""
    import torch
    return torch.empty_strided(t.size(), t.stride(), dtype=t.dtype, device=t.device)


def _tp(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream):
    import torch
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def forward(q, k, v, valid=None, m=1.0, eps=1e-6, out=None, saved_S=None, saved_norms=None,
            stream=None, flags=0):
    """cotten_fwd on torch CUDA tensors [B, H, N, D]; valid is uint8 [B, >=N] or None."""
    import torch
    _same_layout(q, k, v, out)
    desc = _tdesc(q, eps, flags, valid)
    if out is None:
        out = _like(q)
    check(load().cotten_fwd(ctypes.byref(desc), _tp(q), _tp(k), _tp(v), _tp(valid), float(m),
                            _tp(out), _tp(saved_S), _tp(saved_norms), _stream(stream)))
    return out


def backward(q, k, v, valid, m, d_out, saved_S, dq=None, dk=None, dv=None, dm_unit=None,
             dm_total=None, eps=1e-6, stream=None, flags=0):
    """cotten_bwd on torch CUDA tensors; returns (dq, dk, dv)."""
    import torch
    _same_layout(q, k, v, d_out, dq, dk, dv)
    desc = _tdesc(q, eps, flags, valid)
    dq = _like(q) if dq is None else dq
    dk = _like(q) if dk is None else dk
    dv = _like(q) if dv is None else dv
    check(load().cotten_bwd(ctypes.byref(desc), _tp(q), _tp(k), _tp(v), _tp(valid), float(m),
                            _tp(d_out), _tp(saved_S), _tp(dq), _tp(dk), _tp(dv), _tp(dm_unit),
                            _tp(dm_total), _stream(stream)))
    return dq, dk, dv


def device_status(device=0, reset=True) -> int:
    bits = ctypes.c_int32(0)
    check(load().cotten_device_status(int(device), ctypes.byref(bits), int(reset)))
    return int(bits.value)
