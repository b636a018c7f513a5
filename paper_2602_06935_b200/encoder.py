"""Host-side mirror of the reference encoder step, over include/cotten_encoder.h.

Same names and argument meaning as the reference's model / training API
(/root/reference/proj/include/cosrec/encoder.hpp, training.hpp, data.hpp),
batched and device-resident:

    Encoder(ModelConfig...)                  EncoderParams + AdamState (encoder.hpp:18-50)
    Encoder.assemble(...)                    make_batches/fit_sequence (data.cpp:193-222),
                                             mask_sequence (training.cpp:15-56),
                                             mask_for_ids (encoder.cpp:268-272)
    Encoder.model_forward(ids, rows, ...)    model_forward (encoder.cpp:276-325)
    Encoder.nll_loss(targets)                nll_loss (training.cpp:58-87)
    Encoder.model_backward()                 model_backward (encoder.cpp:327-377)
    Encoder.clip_adam(max_norm, lr, wd)      clip_gradients + adam_step (training.cpp:89-143)

Tensors are torch CUDA tensors (device memory and streams only: the math is
libcotten.so).  ``params`` / ``grads`` are views of the library's flat
buffers in the reference's for_each_matrix order; ``m`` / ``m_grads`` the
per-layer exponents (float64).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional

import torch

from . import _lib
from ._lib import check, load

_vp, _i64, _dbl, _u64, _int = (ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_uint64,
                                ctypes.c_int)


class EncConfig(ctypes.Structure):
    _fields_ = [("vocab", _i64), ("dim", _i64), ("layers", _i64), ("heads", _i64),
                ("max_seq", _i64), ("dropout", _dbl), ("ln_eps", _dbl), ("attn_eps", _dbl)]


SIGNATURES = {
    "cotten_enc_create": (_int, [ctypes.POINTER(EncConfig), _i64, _i64, ctypes.POINTER(_vp)]),
    "cotten_enc_destroy": (_int, [_vp]),
    "cotten_enc_tensor_count": (_i64, [_vp]),
    "cotten_enc_layout": (_int, [_vp, _vp, _vp, _vp]),
    "cotten_enc_params": (_vp, [_vp]),
    "cotten_enc_grads": (_vp, [_vp]),
    "cotten_enc_m_params": (_vp, [_vp]),
    "cotten_enc_m_grads": (_vp, [_vp]),
    "cotten_enc_logits": (_vp, [_vp]),
    "cotten_enc_assemble": (_int, [_vp, _vp, _vp, _i64, _i64, _int, _dbl, _int, _u64, _vp, _vp,
                                   _vp, _vp, _vp, _vp]),
    "cotten_enc_forward": (_int, [_vp, _vp, _i64, _i64, _vp, _i64, _int, _u64, _vp, _vp, _vp]),
    "cotten_enc_loss": (_int, [_vp, _vp, _vp, _vp]),
    "cotten_enc_backward": (_int, [_vp, _vp, _vp]),
    "cotten_enc_clip_adam": (_int, [_vp, _dbl, _dbl, _dbl, _vp, _vp]),
}
_bound = False


def lib():
    global _bound
    L = load()
    if not _bound:
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _bound = True
    return L


class _DevView:
    """__cuda_array_interface__ over a library-owned device buffer."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"data": (ptr, False), "shape": tuple(shape),
                                         "typestr": typestr, "version": 3, "strides": None}


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


@dataclass
class ModelConfig:
    """encoder.hpp:18-30 (threads is the reference's CPU parallelism: unused)."""
    vocab: int
    dim: int = 64
    layers: int = 2
    max_seq: int = 50
    dropout: float = 0.1
    ln_eps: float = 1e-5
    heads: int = 2
    attn_eps: float = 1e-6

    def id_count(self) -> int:
        return self.vocab + 2


def expected_layout(cfg: ModelConfig):
    """(rows, cols) of every tensor in for_each_matrix order (encoder.hpp:52-72),
    as the library lays them out (checked against the reference's own count)."""
    d, dh, V2 = cfg.dim, cfg.dim // cfg.heads, cfg.id_count()
    out = [(V2, d), (cfg.max_seq, d)]
    for _ in range(cfg.layers):
        out += [(d, dh)] * (3 * cfg.heads)
        out += [(d, d), (d, 4 * d), (1, 4 * d), (4 * d, d), (1, d), (1, d), (1, d), (1, d), (1, d)]
    out += [(d, V2), (1, V2)]
    return out


class Encoder:
    def __init__(self, cfg: ModelConfig, max_batch: int, max_queries: int):
        L = lib()
        self.cfg = cfg
        c = EncConfig(cfg.vocab, cfg.dim, cfg.layers, cfg.heads, cfg.max_seq, cfg.dropout,
                      cfg.ln_eps, cfg.attn_eps)
        h = ctypes.c_void_p()
        check(L.cotten_enc_create(ctypes.byref(c), int(max_batch), int(max_queries),
                                  ctypes.byref(h)))
        self._h = h
        self.max_batch, self.max_queries = int(max_batch), int(max_queries)
        n = int(L.cotten_enc_tensor_count(h))
        offs = (ctypes.c_int64 * (n + 1))()
        rows = (ctypes.c_int64 * n)()
        cols = (ctypes.c_int64 * n)()
        check(L.cotten_enc_layout(h, offs, rows, cols))
        self.layout = [(int(offs[i]), int(rows[i]), int(cols[i])) for i in range(n)]
        self.count = int(offs[n])
        dev = torch.device("cuda", torch.cuda.current_device())
        self.params = torch.as_tensor(_DevView(L.cotten_enc_params(h), (self.count,), "<f4"),
                                      device=dev)
        self.grads = torch.as_tensor(_DevView(L.cotten_enc_grads(h), (self.count,), "<f4"),
                                     device=dev)
        self.m = torch.as_tensor(_DevView(L.cotten_enc_m_params(h), (cfg.layers,), "<f8"),
                                 device=dev)
        self.m_grads = torch.as_tensor(_DevView(L.cotten_enc_m_grads(h), (cfg.layers,), "<f8"),
                                       device=dev)
        self.K = 0

    def close(self):
        if self._h:
            lib().cotten_enc_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def tensor(self, i: int, grads: bool = False) -> torch.Tensor:
        off, r, c = self.layout[i]
        src = self.grads if grads else self.params
        return src[off:off + r * c].view(r, c)

    def logits(self) -> torch.Tensor:
        C = self.cfg.id_count()
        v = torch.as_tensor(_DevView(lib().cotten_enc_logits(self._h), (self.max_queries, C),
                                     "<f4"), device=self.params.device)
        return v[:self.K]

    # --- the reference API ------------------------------------------------
    def assemble(self, items: torch.Tensor, offsets: torch.Tensor, n: int, train: bool,
                 p_mask: float = 0.15, bert: bool = False, seed: int = 0):
        """Ragged histories (CSR, int32 items / int64 offsets) -> ids [B, n],
        valid [B, n], query rows [max_queries] (inactive = -1), targets,
        k_total (device int32)."""
        B = offsets.numel() - 1
        dev = items.device
        ids = torch.empty(B, n, dtype=torch.int32, device=dev)
        valid = torch.empty(B, n, dtype=torch.uint8, device=dev)
        rows = torch.empty(self.max_queries, dtype=torch.int32, device=dev)
        targets = torch.zeros(self.max_queries, dtype=torch.int32, device=dev)
        k_total = torch.empty(1, dtype=torch.int32, device=dev)
        check(lib().cotten_enc_assemble(self._h, _ptr(items), _ptr(offsets), B, n, int(train),
                                        float(p_mask), int(bert), int(seed) & (2**64 - 1),
                                        _ptr(ids), _ptr(valid), _ptr(rows), _ptr(targets),
                                        _ptr(k_total), _stream()))
        return ids, valid, rows, targets, k_total

    def model_forward(self, ids: torch.Tensor, query_rows: torch.Tensor, train: bool = False,
                      dropout_seed: int = 0, dropout_masks: Optional[torch.Tensor] = None,
                      logits: Optional[torch.Tensor] = None) -> torch.Tensor:
        B, n = ids.shape
        K = query_rows.numel()
        check(lib().cotten_enc_forward(self._h, _ptr(ids), B, n, _ptr(query_rows), K, int(train),
                                       int(dropout_seed) & (2**64 - 1), _ptr(dropout_masks),
                                       _ptr(logits), _stream()))
        self.K = K
        return logits if logits is not None else self.logits()

    def nll_loss(self, targets: torch.Tensor, loss: Optional[torch.Tensor] = None) -> torch.Tensor:
        if loss is None:
            loss = torch.empty(1, dtype=torch.float64, device=targets.device)
        check(lib().cotten_enc_loss(self._h, _ptr(targets), _ptr(loss), _stream()))
        return loss

    def model_backward(self, d_logits: Optional[torch.Tensor] = None):
        check(lib().cotten_enc_backward(self._h, _ptr(d_logits), _stream()))

    def clip_adam(self, max_norm: float = 1.0, lr: float = 1e-3, weight_decay: float = 1e-3,
                  norm: Optional[torch.Tensor] = None):
        check(lib().cotten_enc_clip_adam(self._h, float(max_norm), float(lr), float(weight_decay),
                                         _ptr(norm), _stream()))
        return norm


__all__ = ["Encoder", "ModelConfig", "expected_layout", "lib", "_lib"]
