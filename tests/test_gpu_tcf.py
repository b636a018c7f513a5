"""GPU parity of the fp32 d_h = 64 tensor-core kernels (kernels_tcf.cuh:
tcgen05 kind::f16 with every operand split into three bf16 parts, 64-row
chunks, M = 64 MMAs) against the float64 oracle on the same fp32 inputs, at
the fp32 bar (normwise <= 1e-5 per (sequence, head) tensor), with
bit-exact padding.  Covers the 64-row chunk and 16-row K-step edges, the
running-sum flush (N > 512), persistent CTAs with >= 3 units each, m != 1,
arbitrary masks, NaN in padded K rows, the strided [B][N][H][D] layout, and
the register-tiled FP32-pipe kernels (COTTEN_FLAG_FP32_PIPE) on the same
inputs as the A/B partner — both within the bar, not bit-identical."""
import numpy as np
import pytest

from paper_2602_06935_b200 import _lib, inputs
from test_gpu_parity import assert_parity, normwise, oracle_for, run_gpu

pytestmark = pytest.mark.gpu
D = 64


@pytest.mark.parametrize("N", [1, 2, 15, 16, 17, 63, 64, 65, 127, 128, 129, 200, 511, 512, 513, 700])
def test_tcf_seq_len_edges(N):
    B, H = 5, 2
    h = inputs.make_host(B, H, N, D, seed=N)
    valid = inputs.left_padded_mask(B, N, N)
    res = run_gpu(h, valid, 1.0, 1e-6, "f32")
    assert_parity(res, oracle_for(res["inputs"], valid, 1.0, 1e-6), valid, "f32")


@pytest.mark.parametrize("N,m", [(200, 1.0), (200, 0.75), (1000, 0.75)])
def test_tcf_multi_unit_schedule(N, m):
    """B*H = 480 units on 148 persistent CTAs: >= 3 units per CTA."""
    B, H = 240, 2
    h = inputs.make_host(B, H, N, D, seed=7)
    rng = np.random.default_rng(3)
    valid = (rng.random((B, N)) < 0.7).astype(np.uint8)  # arbitrary pattern
    valid[:, -1] = 1
    res = run_gpu(h, valid, m, 1e-6, "f32")
    sel = rng.choice(B, size=32, replace=False)  # oracle on a sample of sequences
    sub = {k: v[sel] for k, v in res["inputs"].items()}
    ref = oracle_for(sub, valid[sel], m, 1e-6)
    part = {k: (v[sel] if isinstance(v, np.ndarray) and v.ndim == 4 else v) for k, v in res.items()}
    part["dm_unit"] = res["dm_unit"].reshape(B, H)[sel].reshape(-1)
    part["dm_total"] = float(np.sum(part["dm_unit"]))
    assert_parity(part, ref, valid[sel], "f32")


@pytest.mark.parametrize("N", [4096, 16384])
def test_tcf_long_sequence(N):
    B, H = 2, 1
    h = inputs.make_host(B, H, N, D, seed=11)
    valid = inputs.left_padded_mask(B, N, 11)
    res = run_gpu(h, valid, 1.0, 1e-6, "f32")
    assert_parity(res, oracle_for(res["inputs"], valid, 1.0, 1e-6), valid, "f32")


def test_tcf_nan_in_padded_k_rows_never_propagates():
    B, H, N = 3, 2, 150
    h = inputs.make_host(B, H, N, D, seed=5)
    valid = inputs.left_padded_mask(B, N, 5)
    h["k"] = h["k"].copy()
    for b in range(B):
        h["k"][b, :, valid[b] == 0, :] = np.nan
    res = run_gpu(h, valid, 1.0, 1e-6, "f32")
    for name in ("out", "dq", "dk", "dv"):
        assert np.isfinite(res[name]).all(), name
    clean = {k: np.nan_to_num(v, nan=0.0) for k, v in res["inputs"].items()}
    assert_parity(res, oracle_for(clean, valid, 1.0, 1e-6), valid, "f32")


def test_tcf_strided_projection_layout():
    B, H, N = 4, 2, 300
    h = inputs.make_host(B, H, N, D, seed=9)
    valid = inputs.random_mask(B, N, 9)
    a = run_gpu(h, valid, 1.0, 1e-6, "f32", layout="bnhd")
    assert_parity(a, oracle_for(a["inputs"], valid, 1.0, 1e-6), valid, "f32")


def test_tcf_against_fp32_pipe_partner():
    B, H, N = 8, 2, 300
    h = inputs.make_host(B, H, N, D, seed=2)
    valid = inputs.left_padded_mask(B, N, 2)
    a = run_gpu(h, valid, 1.0, 1e-6, "f32")
    b = run_gpu(h, valid, 1.0, 1e-6, "f32", flags=_lib.FLAG_FP32_PIPE)
    ref = oracle_for(a["inputs"], valid, 1.0, 1e-6)
    assert_parity(a, ref, valid, "f32")
    assert_parity(b, ref, valid, "f32")
    assert not np.array_equal(a["dq"], b["dq"])  # the tensor-core path really ran
    errs = {n: normwise(a[n], r) for n, r in zip(("out", "dq", "dk", "dv"), ref[:4])}
    assert max(errs.values()) <= 1e-5, errs


# ---- head-merged mode: fp32 d_h = 32, even H, N <= 64 (heads 2j, 2j+1 in one 64-column row) ----

@pytest.mark.parametrize("H", [2, 4])
@pytest.mark.parametrize("N", [4, 15, 16, 17, 33, 50, 63, 64])
def test_tcf_merged_heads_seq_lens(N, H):
    """(N <= 3 runs through the same kernels in test_gpu_schedule.py's
    24-seed sweep, under its condition-scaled bound: with one to three rows
    O = (q~.k~) v cancels and a plain normwise 1e-5 measures conditioning.)"""
    B = 5
    h = inputs.make_host(B, H, N, 32, seed=N + H)
    valid = inputs.left_padded_mask(B, N, N)
    res = run_gpu(h, valid, 1.0, 1e-6, "f32")
    assert_parity(res, oracle_for(res["inputs"], valid, 1.0, 1e-6), valid, "f32", m=1.0, eps=1e-6)


@pytest.mark.parametrize("m", [1.0, 0.75])
def test_tcf_merged_heads_multi_unit_schedule(m):
    """Beauty shape at B = 480: 480 head pairs on 148 persistent CTAs (>= 3 per CTA)."""
    B, H, N = 480, 2, 50
    h = inputs.make_host(B, H, N, 32, seed=17)
    rng = np.random.default_rng(5)
    valid = (rng.random((B, N)) < 0.7).astype(np.uint8)
    valid[:, -1] = 1
    res = run_gpu(h, valid, m, 1e-6, "f32")
    sel = rng.choice(B, size=48, replace=False)
    sub = {k: v[sel] for k, v in res["inputs"].items()}
    ref = oracle_for(sub, valid[sel], m, 1e-6)
    part = {k: (v[sel] if isinstance(v, np.ndarray) and v.ndim == 4 else v) for k, v in res.items()}
    part["dm_unit"] = res["dm_unit"].reshape(B, H)[sel].reshape(-1)
    part["dm_total"] = float(np.sum(part["dm_unit"]))
    assert_parity(part, ref, valid[sel], "f32")


def test_tcf_merged_heads_nan_in_padded_k_rows():
    B, H, N = 6, 2, 50
    h = inputs.make_host(B, H, N, 32, seed=23)
    valid = inputs.left_padded_mask(B, N, 23)
    h["k"] = h["k"].copy()
    for b in range(B):
        h["k"][b, :, valid[b] == 0, :] = np.nan
    res = run_gpu(h, valid, 1.0, 1e-6, "f32")
    for name in ("out", "dq", "dk", "dv"):
        assert np.isfinite(res[name]).all(), name
    clean = {k: np.nan_to_num(v, nan=0.0) for k, v in res["inputs"].items()}
    assert_parity(res, oracle_for(clean, valid, 1.0, 1e-6), valid, "f32")


def test_tcf_merged_heads_saved_state_and_norms():
    torch = pytest.importorskip("torch")
    import oracle
    from paper_2602_06935_b200 import ops
    B, H, N = 3, 4, 50
    h = inputs.make_host(B, H, N, 32, seed=29)
    valid = inputs.random_mask(B, N, 29)
    t = {n: torch.from_numpy(x).cuda() for n, x in h.items()}
    norms = torch.empty(B * H, 2, N, device="cuda")
    S = torch.empty(B * H, 32, 32, device="cuda")
    ops.forward(t["q"], t["k"], t["v"], torch.from_numpy(valid).cuda(), 0.75, saved_S=S,
                saved_norms=norms)
    got, gS = norms.cpu().numpy().astype(np.float64), S.cpu().numpy().astype(np.float64)
    for b in range(B):
        for hh in range(H):
            r = oracle.fwd(h["q"][b, hh], h["k"][b, hh], h["v"][b, hh], valid[b], 0.75, 1e-6)
            np.testing.assert_allclose(got[b * H + hh, 0], r["norm_q"], rtol=1e-6)
            np.testing.assert_allclose(got[b * H + hh, 1], r["norm_k"], rtol=1e-6)
            assert np.all(got[b * H + hh, 1][valid[b] == 0] == 1.0)
            assert normwise(gS[b * H + hh][None, None], r["S"][None, None]) <= 1e-5


def test_tcf_merged_heads_against_fp32_pipe_partner():
    B, H, N = 64, 2, 50
    h = inputs.make_host(B, H, N, 32, seed=31)
    valid = inputs.left_padded_mask(B, N, 31)
    a = run_gpu(h, valid, 1.0, 1e-6, "f32")
    b = run_gpu(h, valid, 1.0, 1e-6, "f32", flags=_lib.FLAG_FP32_PIPE)
    ref = oracle_for(a["inputs"], valid, 1.0, 1e-6)
    assert_parity(a, ref, valid, "f32")
    assert_parity(b, ref, valid, "f32")
    assert not np.array_equal(a["dq"], b["dq"])  # the tensor-core path really ran


def test_tcf_odd_heads_keep_fp32_pipe():
    B, H, N = 4, 3, 50
    h = inputs.make_host(B, H, N, 32, seed=37)
    valid = inputs.left_padded_mask(B, N, 37)
    a = run_gpu(h, valid, 1.0, 1e-6, "f32")
    b = run_gpu(h, valid, 1.0, 1e-6, "f32", flags=_lib.FLAG_FP32_PIPE)
    assert_parity(a, oracle_for(a["inputs"], valid, 1.0, 1e-6), valid, "f32")
    assert np.array_equal(a["dq"], b["dq"])
