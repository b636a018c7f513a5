"""GPU parity of the fp32 d_h = 128 tensor-core kernels (kernels_tcg.cuh:
tcgen05 kind::f16, every operand as three bf16 parts, 32-row items in a
two-slot ring, M = 128 reductions, M = 64 row outputs of which rows 0-31 are
the item's, the S / G running sum in TMEM, one state area for S and dA)
against the float64 oracle on the same fp32 inputs, at the fp32 bar (normwise
<= 1e-5 per (sequence, head) tensor), with bit-exact padding.
Covers the 32-row item and 16-row K-step edges, the running-sum flush
(N > 512), persistent CTAs with >= 3 units each, m != 1, arbitrary masks,
NaN in padded K rows, the strided [B][N][H][D] layout, saved norms / S, and
the register-tiled FP32-pipe kernels (COTTEN_FLAG_FP32_PIPE) as the A/B
partner — both within the bar, not bit-identical."""
import numpy as np
import pytest

import oracle
from paper_2602_06935_b200 import _lib, inputs, ops
from test_gpu_parity import assert_parity, normwise, oracle_for, run_gpu

pytestmark = pytest.mark.gpu
D = 128


@pytest.mark.parametrize("N", [1, 2, 15, 16, 17, 31, 32, 33, 64, 129, 200, 511, 512, 513, 700])
def test_tcg_seq_len_edges(N):
    B, H = 5, 2
    h = inputs.make_host(B, H, N, D, seed=N)
    valid = inputs.left_padded_mask(B, N, N)
    res = run_gpu(h, valid, 1.0, 1e-6, "f32")
    ref = oracle_for(res["inputs"], valid, 1.0, 1e-6)
    if N <= 3:
        # one to three rows: O = s (q~.k~) v cancels, so the error is bounded
        # against the magnitude evaluated on absolute values (the stated rule of
        # test_gpu_schedule.py::test_tiny_sequences_seed_sweep)
        from test_gpu_schedule import _abs_scales
        sc = _abs_scales(res["inputs"], valid, 1.0, 1e-6)
        for name, want in zip(("out", "dq", "dk", "dv"), ref[:4]):
            err = np.abs(res[name] - want).reshape(B * H, -1).max(1) / np.maximum(sc[name], 1e-30)
            assert err.max() <= 1e-5, (name, float(err.max()))
        pad = np.broadcast_to((valid == 0)[:, None, :], (B, H, N))
        assert np.all(res["dk"][pad] == 0.0) and np.all(res["dv"][pad] == 0.0)
    else:
        assert_parity(res, ref, valid, "f32")


@pytest.mark.parametrize("N,m", [(200, 1.0), (200, 0.75), (600, 0.75)])
def test_tcg_multi_unit_schedule(N, m):
    """B*H = 480 units on 148 persistent CTAs: >= 3 units per CTA."""
    B, H = 240, 2
    h = inputs.make_host(B, H, N, D, seed=7)
    rng = np.random.default_rng(3)
    valid = (rng.random((B, N)) < 0.7).astype(np.uint8)
    valid[:, -1] = 1
    res = run_gpu(h, valid, m, 1e-6, "f32")
    sel = rng.choice(B, size=24, replace=False)
    sub = {k: v[sel] for k, v in res["inputs"].items()}
    ref = oracle_for(sub, valid[sel], m, 1e-6)
    part = {k: (v[sel] if isinstance(v, np.ndarray) and v.ndim == 4 else v) for k, v in res.items()}
    part["dm_unit"] = res["dm_unit"].reshape(B, H)[sel].reshape(-1)
    part["dk"], part["dv"] = res["dk"][sel], res["dv"][sel]
    part["dm_total"] = float(np.sum(part["dm_unit"]))
    assert_parity(part, ref, valid[sel], "f32")


@pytest.mark.parametrize("N", [4096, 16384])
def test_tcg_long_sequence(N):
    B, H = 2, 1
    h = inputs.make_host(B, H, N, D, seed=11)
    valid = inputs.left_padded_mask(B, N, 11)
    res = run_gpu(h, valid, 1.0, 1e-6, "f32")
    assert_parity(res, oracle_for(res["inputs"], valid, 1.0, 1e-6), valid, "f32")


def test_tcg_nan_in_padded_k_rows_never_propagates():
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


def test_tcg_strided_projection_layout():
    B, H, N = 4, 2, 300
    h = inputs.make_host(B, H, N, D, seed=9)
    valid = inputs.random_mask(B, N, 9)
    a = run_gpu(h, valid, 1.0, 1e-6, "f32", layout="bnhd")
    assert_parity(a, oracle_for(a["inputs"], valid, 1.0, 1e-6), valid, "f32")


def test_tcg_against_fp32_pipe_partner():
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


def test_tcg_saved_norms_and_state():
    torch = pytest.importorskip("torch")
    B, H, N = 3, 2, 300
    h = inputs.make_host(B, H, N, D, seed=21)
    valid = inputs.random_mask(B, N, 21)
    t = {n: torch.from_numpy(x).cuda() for n, x in h.items()}
    norms = torch.empty(B * H, 2, N, device="cuda")
    S = torch.empty(B * H, D, D, device="cuda")
    ops.forward(t["q"], t["k"], t["v"], torch.from_numpy(valid).cuda(), 0.75, saved_S=S,
                saved_norms=norms)
    got, gS = norms.cpu().numpy().astype(np.float64), S.cpu().numpy().astype(np.float64)
    for b in range(B):
        for hh in range(H):
            f = lambda n: h[n][b, hh].astype(np.float64)  # noqa: E731
            r = oracle.fwd(f("q"), f("k"), f("v"), valid[b], 0.75, 1e-6)
            np.testing.assert_allclose(got[b * H + hh, 0], r["norm_q"], rtol=1e-6)
            np.testing.assert_allclose(got[b * H + hh, 1], r["norm_k"], rtol=1e-6)
            assert np.all(got[b * H + hh, 1][valid[b] == 0] == 1.0)
            assert normwise(gS[b * H + hh][None, None], r["S"][None, None]) <= 1e-5


@pytest.mark.parametrize("N", [50, 300])
def test_tcg_no_mask(N):
    """valid = NULL: every row valid (attention_forward without a RowMask)."""
    B, H = 6, 2
    h = inputs.make_host(B, H, N, D, seed=N + 31)
    res = run_gpu(h, None, 0.75, 1e-6, "f32")
    assert_parity(res, oracle_for(res["inputs"], None, 0.75, 1e-6), None, "f32")
