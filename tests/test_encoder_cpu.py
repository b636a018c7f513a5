"""CPU checks of the encoder boundary and of its oracle: the
reference encoder library (oracle/_ref/libcosrec_encoder.so, built from the
reference's own sources) loads, its flat parameter count matches the layout
the device library uses, and its eval-mode batch assembly behaves like the
reference's tests (fit_sequence left-pads / truncates, the last real slot is
masked).  No compute call needs a GPU here."""
import ctypes

import numpy as np
import pytest

import oracle.encoder_ref as eref
from paper_2602_06935_b200 import _lib, encoder

pytestmark = pytest.mark.skipif(not eref.available(), reason="oracle/_ref not built")


@pytest.mark.parametrize("vocab,dim,layers,heads,max_seq",
                         [(40, 64, 2, 2, 24), (3706, 64, 2, 2, 200), (10, 32, 1, 4, 8),
                          (7, 48, 3, 3, 5)])
def test_layout_matches_reference_param_count(vocab, dim, layers, heads, max_seq):
    cfg = encoder.ModelConfig(vocab=vocab, dim=dim, layers=layers, heads=heads, max_seq=max_seq)
    lay = encoder.expected_layout(cfg)
    assert sum(r * c for r, c in lay) == eref.lib().ref_enc_param_count(vocab, dim, layers, heads,
                                                                       max_seq)
    # tensor count: 2 embeddings + per layer 3H projections + 9 + head w, b
    assert len(lay) == 2 + layers * (3 * heads + 9) + 2


def test_reference_init_is_deterministic_and_truncated():
    cfg = encoder.ModelConfig(vocab=30, dim=64, layers=2, heads=2, max_seq=16)
    a, ma = eref.init(cfg, 7)
    b, mb = eref.init(cfg, 7)
    assert np.array_equal(a, b) and np.all(ma == 1.0)  # attn.m = 1.0 (encoder.cpp:45)
    lay = encoder.expected_layout(cfg)
    off = np.cumsum([0] + [r * c for r, c in lay])
    w = a[off[0]:off[1]]
    assert np.abs(w).max() <= 0.04 + 1e-12  # truncated at 2 stddev (rng.hpp:24-30)
    # biases and LN gains/biases (encoder.cpp:50-57): b1 zero, gain one
    i_b1 = 2 + 3 * cfg.heads + 2
    assert np.all(a[off[i_b1]:off[i_b1 + 1]] == 0.0)
    i_g1 = 2 + 3 * cfg.heads + 5
    assert np.all(a[off[i_g1]:off[i_g1 + 1]] == 1.0)


def test_reference_fit_and_eval_mask():
    items = np.array([5, 6, 7, 8, 9, 1, 2, 3], np.int32)
    offs = np.array([0, 5, 6, 8], np.int64)
    ids, slot, tg = eref.fit_mask_eval(items, offs, 4, vocab=9)
    # seq 0: last 4 of [5..9] -> [6,7,8,9], the last slot masked with vocab+1
    assert ids[0].tolist() == [6, 7, 8, 10] and slot[0] == 3 and tg[0] == 9
    # seq 1: [1] left-padded
    assert ids[1].tolist() == [0, 0, 0, 10] and slot[1] == 3 and tg[1] == 1
    assert ids[2].tolist() == [0, 0, 2, 10] and tg[2] == 3


def test_reference_step_runs_and_grads_are_finite():
    cfg = encoder.ModelConfig(vocab=20, dim=64, layers=2, heads=2, max_seq=12, dropout=0.1)
    flat, m = eref.init(cfg, 1)
    rng = np.random.default_rng(0)
    ids = rng.integers(1, 21, size=(3, 12)).astype(np.int32)
    ids[0, :4] = 0
    pos = [[5, 9], [0], [3, 11]]
    tg = rng.integers(1, 21, size=5).astype(np.int32)
    logits, loss, g, gm, masks = eref.step(cfg, flat, m, ids, pos, tg, train=True,
                                           dropout_seed=3, want_masks=True)
    assert logits.shape == (5, 22) and np.isfinite(loss) and np.all(np.isfinite(g))
    assert masks.shape == (5, 36, 64)
    assert set(np.unique(masks)).issubset({0.0, 1.0 / 0.9})


def test_encoder_entry_points_reject_null_without_a_device():
    L = encoder.lib()
    h = ctypes.c_void_p()
    assert L.cotten_enc_create(None, 1, 1, ctypes.byref(h)) == _lib.COTTEN_ERR_USAGE
    c = encoder.EncConfig(0, 64, 2, 2, 10, 0.1, 1e-5, 1e-6)
    assert L.cotten_enc_create(ctypes.byref(c), 1, 1, ctypes.byref(h)) == _lib.COTTEN_ERR_USAGE
    assert b"vocab" in L.cotten_last_error()
    c = encoder.EncConfig(10, 63, 2, 2, 10, 0.1, 1e-5, 1e-6)
    assert L.cotten_enc_create(ctypes.byref(c), 1, 1, ctypes.byref(h)) == _lib.COTTEN_ERR_USAGE
    assert L.cotten_enc_forward(None, None, 1, 1, None, 1, 0, 0, None, None, None) == \
        _lib.COTTEN_ERR_USAGE
    assert L.cotten_enc_tensor_count(None) == -1
