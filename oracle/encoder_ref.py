"""TEST INFRASTRUCTURE ONLY — ctypes wrapper of oracle/_ref/libcosrec_encoder.so,
the UNMODIFIED reference encoder / nll_loss / clip + Adam / batch assembly
compiled from its own sources (oracle/Makefile, encoder_shim.cpp).

Used by tests/test_encoder*.py as the checker of the device encoder
(paper_2602_06935_b200/encoder.py) and by bench.py's CPU leg of the encoder
line; never by the product path.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ENC_SO = os.path.join(HERE, "_ref", "libcosrec_encoder.so")

_vp, _i64, _dbl, _u64, _int, _long = (ctypes.c_void_p, ctypes.c_int64, ctypes.c_double,
                                      ctypes.c_uint64, ctypes.c_int, ctypes.c_long)
_lib = None


def available() -> bool:
    return os.path.exists(ENC_SO)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise ImportError(f"{ENC_SO} missing: run `make -C oracle` where /root/reference exists")
        L = ctypes.CDLL(ENC_SO)
        L.ref_enc_last_error.restype = ctypes.c_char_p
        L.ref_enc_param_count.restype = _i64
        L.ref_enc_param_count.argtypes = [_i64] * 5
        L.ref_enc_init.restype = _int
        L.ref_enc_init.argtypes = [_i64] * 5 + [_u64, _vp, _vp]
        L.ref_enc_step.restype = _int
        L.ref_enc_step.argtypes = ([_i64] * 5 + [_dbl] * 3 + [_vp, _vp, _i64, _i64] + [_vp] * 4 +
                                   [_int, _u64] + [_vp] * 5)
        L.ref_enc_clip_adam.restype = _int
        L.ref_enc_clip_adam.argtypes = [_i64] * 5 + [_vp] * 8 + [_long, _dbl, _dbl, _dbl, _vp]
        L.ref_fit_mask_eval.restype = _int
        L.ref_fit_mask_eval.argtypes = [_vp, _vp, _i64, _i64, _i64, _vp, _vp, _vp]
        L.ref_enc_bench.restype = _int
        L.ref_enc_bench.argtypes = [_i64] * 5 + [_dbl, _i64, _i64, _i64] + [_vp] * 4 + [_int, _vp]
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _check(rc):
    if rc != 0:
        raise RuntimeError(f"reference error {rc}: {lib().ref_enc_last_error().decode()}")


def dims(cfg):
    return (cfg.vocab, cfg.dim, cfg.layers, cfg.heads, cfg.max_seq)


def init(cfg, seed):
    """init_encoder (encoder.cpp:26-60): flat float64 params, m."""
    n = lib().ref_enc_param_count(*dims(cfg))
    flat = np.empty(n, np.float64)
    m = np.empty(cfg.layers, np.float64)
    _check(lib().ref_enc_init(*dims(cfg), seed, _p(flat), _p(m)))
    return flat, m


def step(cfg, flat, m, ids, positions, targets, train=False, dropout_seed=0, want_masks=False):
    """model_forward + nll_loss + model_backward on float64 params.
    ids [B, n] int32; positions: list of per-sequence slot lists; targets
    concatenated.  Returns logits, loss, grads, grad_m, masks (or None)."""
    B, n = ids.shape
    ids = np.ascontiguousarray(ids, np.int32)
    off = np.zeros(B + 1, np.int64)
    off[1:] = np.cumsum([len(p) for p in positions])
    pos = np.ascontiguousarray(np.concatenate([np.asarray(p, np.int64) for p in positions]))
    tg = np.ascontiguousarray(targets, np.int32)
    K = int(off[-1])
    logits = np.empty((K, cfg.vocab + 2), np.float64)
    loss = np.empty(1, np.float64)
    grads = np.empty_like(flat)
    gm = np.empty(cfg.layers, np.float64)
    masks = (np.empty((1 + 2 * cfg.layers, B * n, cfg.dim), np.float64)
             if want_masks and train and cfg.dropout > 0 else None)
    _check(lib().ref_enc_step(*dims(cfg), cfg.dropout, cfg.ln_eps, cfg.attn_eps,
                              _p(np.ascontiguousarray(flat)), _p(np.ascontiguousarray(m)), B, n,
                              _p(ids), _p(off), _p(pos), _p(tg), int(train), dropout_seed,
                              _p(logits), _p(loss), _p(grads), _p(gm), _p(masks)))
    return logits, float(loss[0]), grads, gm, masks


def clip_adam(cfg, flat, m, g, gm, m1, m1m, m2, m2m, step_before, max_norm, lr, wd):
    """clip_gradients + adam_step (training.cpp:89-143), arrays updated in place."""
    norm = np.empty(1, np.float64)
    _check(lib().ref_enc_clip_adam(*dims(cfg), _p(flat), _p(m), _p(g), _p(gm), _p(m1), _p(m1m),
                                   _p(m2), _p(m2m), step_before, max_norm, lr, wd, _p(norm)))
    return float(norm[0])


def fit_mask_eval(items, offsets, n, vocab):
    """fit_sequence + mask_sequence(train_mode=false): ids [B, n], slot [B], target [B]."""
    B = len(offsets) - 1
    ids = np.empty((B, n), np.int32)
    slot = np.empty(B, np.int64)
    tg = np.empty(B, np.int32)
    _check(lib().ref_fit_mask_eval(_p(np.ascontiguousarray(items, np.int32)),
                                   _p(np.ascontiguousarray(offsets, np.int64)), B, n, vocab,
                                   _p(ids), _p(slot), _p(tg)))
    return ids, slot, tg


def bench(cfg, threads, ids, positions, targets, reps):
    """Per-rep seconds of the reference's training step on this batch
    (model_forward + nll_loss + model_backward + clip + Adam, cfg.threads)."""
    B, n = ids.shape
    off = np.zeros(B + 1, np.int64)
    off[1:] = np.cumsum([len(p) for p in positions])
    pos = np.ascontiguousarray(np.concatenate([np.asarray(p, np.int64) for p in positions]))
    secs = np.empty(reps, np.float64)
    _check(lib().ref_enc_bench(*dims(cfg), cfg.dropout, threads, B, n,
                               _p(np.ascontiguousarray(ids, np.int32)), _p(off), _p(pos),
                               _p(np.ascontiguousarray(targets, np.int32)), reps, _p(secs)))
    return secs
