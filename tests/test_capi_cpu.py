"""CPU-side checks of the C-ABI boundary: the library loads, exports every
symbol include/cotten.h declares, and rejects bad calls with the reference's
error taxonomy before touching a device (no compute without a GPU)."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from paper_2602_06935_b200 import _lib, encoder, ops

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "cotten.h")
HEADERS = [HEADER, os.path.join(ROOT, "include", "cotten_encoder.h")]


def declared_symbols():
    txt = "".join(open(h).read() for h in HEADERS)
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(cotten_[a-z_0-9]+)\s*\(", txt)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("cotten_fwd", "cotten_bwd", "cotten_fwd_host", "cotten_bwd_host",
              "cotten_fwd_bwd_host", "cotten_last_error", "cotten_device_status"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    for s in declared_symbols():
        assert hasattr(lib, s), s
        assert s in _lib.SIGNATURES or s in encoder.SIGNATURES, f"{s} has no ctypes signature"
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    for s in declared_symbols():
        assert re.search(r"\bT " + s + r"\b", out), s


def test_library_is_sm100a():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True, check=True).stdout
    assert "sm_100a" in out


def test_version_string():
    assert b"sm_100a" in _lib.load().cotten_version()


def test_null_descriptor_is_usage_error():
    lib = _lib.load()
    rc = lib.cotten_fwd(None, None, None, None, None, 1.0, None, None, None, None)
    assert rc == _lib.COTTEN_ERR_USAGE
    assert b"null descriptor" in lib.cotten_last_error()


@pytest.mark.parametrize("dims", [(0, 1, 4, 4), (1, 0, 4, 4), (1, 1, 0, 4), (1, 1, 4, 0)])
def test_empty_dims_are_shape_errors(dims):
    lib = _lib.load()
    desc = _lib.make_desc(*dims)
    rc = lib.cotten_fwd(ctypes.byref(desc), None, None, None, None, 1.0, None, None, None, None)
    assert rc == _lib.COTTEN_ERR_USAGE
    with pytest.raises(_lib.ShapeError):
        _lib.check(rc)


def test_bad_strides_and_mask_stride():
    lib = _lib.load()
    desc = _lib.make_desc(2, 2, 8, 4, strides=(64, 32, 2))  # stride_n < head_dim
    assert lib.cotten_fwd(ctypes.byref(desc), None, None, None, None, 1.0, None, None, None,
                          None) == _lib.COTTEN_ERR_USAGE
    desc = _lib.make_desc(2, 2, 8, 4, mask_stride_b=4)  # mask shorter than seq_len
    assert lib.cotten_fwd(ctypes.byref(desc), None, None, None, None, 1.0, None, None, None,
                          None) == _lib.COTTEN_ERR_USAGE


def test_host_entry_rejects_sequence_without_real_rows():
    # check_qkv: mask->true_count == 0 -> UsageError (attention.cpp:44), before any device work
    lib = _lib.load()
    B, H, N, D = 2, 1, 3, 2
    desc = _lib.make_desc(B, H, N, D, "f32")
    x = np.ones((B, H, N, D), np.float32)
    valid = np.array([[1, 1, 0], [0, 0, 0]], np.uint8)
    out = np.empty_like(x)
    p = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    rc = lib.cotten_fwd_host(ctypes.byref(desc), p(x), p(x), p(x), p(valid), 1.0, p(out), None,
                             None)
    assert rc == _lib.COTTEN_ERR_USAGE
    assert b"no real rows" in lib.cotten_last_error()


def test_reference_api_validation_mirrors_check_qkv():
    cfg = ops.AttentionConfig()
    a = np.ones((3, 2))
    with pytest.raises(ops.ShapeError):
        ops.cosine_attention_fused(a, np.ones((3, 3)), a, 1.0, cfg)
    with pytest.raises(ops.ShapeError):
        ops.cosine_attention_fused(np.ones((0, 2)), np.ones((0, 2)), np.ones((0, 2)), 1.0, cfg)
    with pytest.raises(ops.ShapeError):
        ops.cosine_attention_fused(a, a, a, 1.0, cfg, mask=ops.RowMask.from_valid([1, 1]))
    with pytest.raises(ops.UsageError):
        ops.cosine_attention_fused(a, a, a, 1.0, cfg, mask=ops.RowMask.from_valid([0, 0, 0]))
    with pytest.raises(ops.UsageError):
        ops.cosine_attention_fused(a, a, a, 1.0, ops.AttentionConfig(tile_size=0))
    # backward without a forward cache (test_attention.cpp:334-341)
    with pytest.raises(ops.UsageError):
        ops.cosine_attention_backward(ops.AttentionCache(), np.ones((2, 2)))
    with pytest.raises(ops.UsageError):
        ops.attention_backward(ops.AttentionCache(), np.ones((2, 2)))
    with pytest.raises(ops.UsageError):
        ops.mechanism_from_string("bogus")


def test_rowmask_from_valid_counts():  # attention.cpp:26-33
    m = ops.RowMask.from_valid([0, 1, 3, 0, 1])
    assert m.true_count == 3


def test_inputs_recipe():
    from paper_2602_06935_b200 import inputs
    # rng.hpp:9-21 splitmix64 / mix_seed known values (computed with the C++ formulas)
    assert inputs.splitmix64(0) == 0xE220A8397B1DCDAF
    vm = inputs.left_padded_mask(64, 200, 0)
    assert vm.shape == (64, 200)
    L = vm.sum(1)
    assert (L >= 1).all() and (L <= 200).all()
    for b in range(64):  # left padding: valid rows are a suffix
        assert vm[b, 200 - L[b]:].all() and not vm[b, :200 - L[b]].any()
