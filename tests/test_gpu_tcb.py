"""GPU parity of the bf16 tensor-core kernels (kernels_tcb.cuh: tcgen05
kind::f16, d_h = 64, and d_h = 32 as paired rows — [N][32] read as
[N/2][64], block-diagonal state operand) against the float64 oracle on the
same bf16-rounded inputs, at the bf16 bar (normwise <= 1e-2 per (sequence, head) tensor,
SURVEY §8c), with bit-exact padding.  Covers chunk edges (N = 1 ... 4096),
the 16-row MMA K-step edges, the running-sum flush (N > 512), persistent
CTAs with >= 3 units each, m != 1, arbitrary masks, NaN in padded K rows,
and the FP32-pipe kernels on the same inputs (COTTEN_FLAG_FP32_PIPE) as the
A/B partner — both within the bar, and not bit-identical (two paths ran)."""
import numpy as np
import pytest

import oracle
from paper_2602_06935_b200 import _lib, inputs, ops
from test_gpu_parity import assert_parity, normwise, oracle_for, run_gpu

pytestmark = pytest.mark.gpu
DS = [32, 64]
# d_h = 32 pairs rows, so its chunk / K-step edges sit at twice the row counts
EDGES = {64: [1, 2, 15, 16, 17, 64, 127, 128, 129, 200, 255, 257, 513, 700],
         32: [2, 30, 32, 34, 126, 128, 130, 200, 254, 256, 258, 510, 512, 514, 1026, 1400]}


@pytest.mark.parametrize("D,N", [(d, n) for d in DS for n in EDGES[d]])
def test_tcb_seq_len_edges(D, N):
    B, H = 5, 2
    h = inputs.make_host(B, H, N, D, seed=N)
    valid = inputs.left_padded_mask(B, N, N)
    res = run_gpu(h, valid, 1.0, 1e-6, "bf16")
    assert_parity(res, oracle_for(res["inputs"], valid, 1.0, 1e-6), valid, "bf16")


@pytest.mark.parametrize("D", DS)
@pytest.mark.parametrize("N,m", [(200, 1.0), (200, 0.75), (1000, 0.75)])
def test_tcb_multi_unit_schedule(N, m, D):
    """B*H = 480 units on 148 persistent CTAs: >= 3 units per CTA."""
    B, H = 240, 2
    h = inputs.make_host(B, H, N, D, seed=7)
    rng = np.random.default_rng(3)
    valid = (rng.random((B, N)) < 0.7).astype(np.uint8)  # arbitrary pattern
    valid[:, -1] = 1
    res = run_gpu(h, valid, m, 1e-6, "bf16")
    sel = rng.choice(B, size=32, replace=False)  # oracle on a sample of sequences
    sub = {k: v[sel] for k, v in res["inputs"].items()}
    ref = oracle_for(sub, valid[sel], m, 1e-6)
    part = {k: (v[sel] if isinstance(v, np.ndarray) and v.ndim == 4 else v) for k, v in res.items()}
    part["dm_unit"] = res["dm_unit"].reshape(B, H)[sel].reshape(-1)
    part["dk"], part["dv"] = res["dk"][sel], res["dv"][sel]
    part["dm_total"] = float(np.sum(part["dm_unit"]))
    assert_parity(part, ref, valid[sel], "bf16")


@pytest.mark.parametrize("D", DS)
def test_tcb_long_sequence(D):
    B, H, N = 2, 2, 4096
    h = inputs.make_host(B, H, N, D, seed=11)
    valid = inputs.left_padded_mask(B, N, 11)
    res = run_gpu(h, valid, 1.0, 1e-6, "bf16")
    assert_parity(res, oracle_for(res["inputs"], valid, 1.0, 1e-6), valid, "bf16")


@pytest.mark.parametrize("D", DS)
def test_tcb_nan_in_padded_k_rows_never_propagates(D):
    torch = pytest.importorskip("torch")
    B, H, N = 3, 2, 150
    h = inputs.make_host(B, H, N, D, seed=5)
    valid = inputs.left_padded_mask(B, N, 5)
    h["k"] = h["k"].copy()
    for b in range(B):
        h["k"][b, :, valid[b] == 0, :] = np.nan
    res = run_gpu(h, valid, 1.0, 1e-6, "bf16")
    for name in ("out", "dq", "dk", "dv"):
        assert np.isfinite(res[name]).all(), name
    clean = {k: np.nan_to_num(v, nan=0.0) for k, v in res["inputs"].items()}
    assert_parity(res, oracle_for(clean, valid, 1.0, 1e-6), valid, "bf16")


@pytest.mark.parametrize("D", DS)
def test_tcb_against_fp32_pipe_partner(D):
    B, H, N = 8, 2, 300
    h = inputs.make_host(B, H, N, D, seed=2)
    valid = inputs.left_padded_mask(B, N, 2)
    a = run_gpu(h, valid, 1.0, 1e-6, "bf16")
    b = run_gpu(h, valid, 1.0, 1e-6, "bf16", flags=_lib.FLAG_FP32_PIPE)
    ref = oracle_for(a["inputs"], valid, 1.0, 1e-6)
    assert_parity(a, ref, valid, "bf16")
    assert_parity(b, ref, valid, "bf16")
    assert not np.array_equal(a["dq"], b["dq"])  # the tensor-core path really ran
    # the tensor-core path is at least as close to the oracle as the bf16 bar needs
    errs = {n: normwise(a[n], r) for n, r in zip(("out", "dq", "dk", "dv"), ref[:4])}
    assert max(errs.values()) <= 1e-2, errs


def test_tcb_pair_saved_norms_and_state():
    """Paired rows: saved norms per sequence row (norm_k = 1 on padded rows,
    attention.cpp:336) and the 32 x 32 saved S = S'00 + S'11."""
    torch = pytest.importorskip("torch")
    B, H, N, D = 3, 2, 300, 32
    h = inputs.make_host(B, H, N, D, seed=21)
    valid = inputs.random_mask(B, N, 21)
    t = {n: torch.from_numpy(x).to("cuda", torch.bfloat16) for n, x in h.items()}
    norms = torch.empty(B * H, 2, N, device="cuda")
    S = torch.empty(B * H, D, D, device="cuda")
    ops.forward(t["q"], t["k"], t["v"], torch.from_numpy(valid).cuda(), 0.75, saved_S=S,
                saved_norms=norms)
    got, gS = norms.cpu().numpy().astype(np.float64), S.cpu().numpy().astype(np.float64)
    for b in range(B):
        for hh in range(H):
            f = lambda n: t[n][b, hh].double().cpu().numpy()  # noqa: E731
            r = oracle.fwd(f("q"), f("k"), f("v"), valid[b], 0.75, 1e-6)
            np.testing.assert_allclose(got[b * H + hh, 0], r["norm_q"], rtol=1e-6)
            np.testing.assert_allclose(got[b * H + hh, 1], r["norm_k"], rtol=1e-6)
            assert np.all(got[b * H + hh, 1][valid[b] == 0] == 1.0)
            assert normwise(gS[b * H + hh][None, None], r["S"][None, None]) <= 1e-5


@pytest.mark.parametrize("N", [199, 301])
def test_bf16_d32_odd_seq_len_keeps_register_tiled_path(N):
    """Odd N cannot be read as row pairs; the register-tiled kernels serve it."""
    B, H, D = 4, 2, 32
    h = inputs.make_host(B, H, N, D, seed=N)
    valid = inputs.left_padded_mask(B, N, N)
    a = run_gpu(h, valid, 1.0, 1e-6, "bf16")
    b = run_gpu(h, valid, 1.0, 1e-6, "bf16", flags=_lib.FLAG_FP32_PIPE)
    assert_parity(a, oracle_for(a["inputs"], valid, 1.0, 1e-6), valid, "bf16")
    assert np.array_equal(a["dq"], b["dq"])
