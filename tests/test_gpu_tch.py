"""GPU parity of the bf16 d_h = 128 tensor-core kernels (kernels_tch.cuh:
tcgen05 kind::f16, 64-row chunks, M = 128 reductions and M = 64 row outputs,
the S / G running sum in TMEM, one state area shared by S and dA) against the
float64 oracle on the same bf16-rounded inputs, at the bf16 bar (normwise
<= 1e-2 per (sequence, head) tensor), with bit-exact padding.
Covers chunk edges (N = 1 ... 4096), the 16-row MMA K-step edges, the
running-sum flush (N > 512: 8 chunks), persistent CTAs with >= 3 units each
(the S / dA hand-over between units), m != 1, arbitrary masks, NaN in padded
K rows, saved norms / S, and the FP32-pipe kernels on the same inputs
(COTTEN_FLAG_FP32_PIPE) as the A/B partner."""
import numpy as np
import pytest

import oracle
from paper_2602_06935_b200 import _lib, inputs, ops
from test_gpu_parity import assert_parity, normwise, oracle_for, run_gpu

pytestmark = pytest.mark.gpu
D = 128
EDGES = [1, 2, 15, 16, 17, 63, 64, 65, 127, 128, 129, 200, 511, 512, 513, 700, 1025]


@pytest.mark.parametrize("N", EDGES)
def test_tch_seq_len_edges(N):
    B, H = 5, 2
    h = inputs.make_host(B, H, N, D, seed=N)
    valid = inputs.left_padded_mask(B, N, N)
    res = run_gpu(h, valid, 1.0, 1e-6, "bf16")
    assert_parity(res, oracle_for(res["inputs"], valid, 1.0, 1e-6), valid, "bf16")


@pytest.mark.parametrize("N,m", [(200, 1.0), (200, 0.75), (600, 0.75)])
def test_tch_multi_unit_schedule(N, m):
    """B*H = 480 units on 148 persistent CTAs: >= 3 units per CTA."""
    B, H = 240, 2
    h = inputs.make_host(B, H, N, D, seed=7)
    rng = np.random.default_rng(3)
    valid = (rng.random((B, N)) < 0.7).astype(np.uint8)  # arbitrary pattern
    valid[:, -1] = 1
    res = run_gpu(h, valid, m, 1e-6, "bf16")
    sel = rng.choice(B, size=24, replace=False)  # oracle on a sample of sequences
    sub = {k: v[sel] for k, v in res["inputs"].items()}
    ref = oracle_for(sub, valid[sel], m, 1e-6)
    part = {k: (v[sel] if isinstance(v, np.ndarray) and v.ndim == 4 else v) for k, v in res.items()}
    part["dm_unit"] = res["dm_unit"].reshape(B, H)[sel].reshape(-1)
    part["dk"], part["dv"] = res["dk"][sel], res["dv"][sel]
    part["dm_total"] = float(np.sum(part["dm_unit"]))
    assert_parity(part, ref, valid[sel], "bf16")


def test_tch_long_sequence():
    B, H, N = 2, 2, 4096
    h = inputs.make_host(B, H, N, D, seed=11)
    valid = inputs.left_padded_mask(B, N, 11)
    res = run_gpu(h, valid, 1.0, 1e-6, "bf16")
    assert_parity(res, oracle_for(res["inputs"], valid, 1.0, 1e-6), valid, "bf16")


def test_tch_nan_in_padded_k_rows_never_propagates():
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


def test_tch_against_fp32_pipe_partner():
    B, H, N = 8, 2, 300
    h = inputs.make_host(B, H, N, D, seed=2)
    valid = inputs.left_padded_mask(B, N, 2)
    a = run_gpu(h, valid, 1.0, 1e-6, "bf16")
    b = run_gpu(h, valid, 1.0, 1e-6, "bf16", flags=_lib.FLAG_FP32_PIPE)
    ref = oracle_for(a["inputs"], valid, 1.0, 1e-6)
    assert_parity(a, ref, valid, "bf16")
    assert_parity(b, ref, valid, "bf16")
    assert not np.array_equal(a["dq"], b["dq"])  # the tensor-core path really ran
    errs = {n: normwise(a[n], r) for n, r in zip(("out", "dq", "dk", "dv"), ref[:4])}
    assert max(errs.values()) <= 1e-2, errs


def test_tch_saved_norms_and_state():
    """Saved norms per row (norm_k = 1 on padded rows, attention.cpp:336) and
    the 128 x 128 saved S in fp32."""
    torch = pytest.importorskip("torch")
    B, H, N = 3, 2, 300
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
            assert normwise(gS[b * H + hh][None, None], r["S"][None, None]) <= 1e-4


@pytest.mark.parametrize("N", [1, 64, 700])
def test_tch_forward_only_without_outputs(N):
    """out = saved_norms = NULL (one pass per unit): saved S only, unit after
    unit on the same state area; equal to the S of the two-pass forward."""
    import ctypes
    torch = pytest.importorskip("torch")
    B, H = 200, 2
    h = inputs.make_host(B, H, N, D, seed=N + 3)
    valid = inputs.left_padded_mask(B, N, N + 3)
    t = {n: torch.from_numpy(x).to("cuda", torch.bfloat16) for n, x in h.items()}
    S = torch.empty(B * H, D, D, device="cuda")
    S2 = torch.empty(B * H, D, D, device="cuda")
    vm = torch.from_numpy(valid).cuda()
    lib = _lib.load()
    desc = _lib.make_desc(B, H, N, D, "bf16", 1e-6)
    p = lambda x: ctypes.c_void_p(x.data_ptr())  # noqa: E731
    _lib.check(lib.cotten_fwd(ctypes.byref(desc), p(t["q"]), p(t["k"]), p(t["v"]), p(vm), 1.0,
                              None, p(S), None, None))
    ops.forward(t["q"], t["k"], t["v"], vm, 1.0, saved_S=S2)
    torch.cuda.synchronize()
    assert torch.equal(S, S2)


def test_tch_strided_projection_layout():
    """[B][N][H][D] storage (stride_n = H*D): the projection output read in place."""
    B, H, N = 4, 2, 300
    h = inputs.make_host(B, H, N, D, seed=9)
    valid = inputs.random_mask(B, N, 9)
    a = run_gpu(h, valid, 1.0, 1e-6, "bf16", layout="bnhd")
    assert_parity(a, oracle_for(a["inputs"], valid, 1.0, 1e-6), valid, "bf16")


@pytest.mark.parametrize("N", [50, 300])
def test_tch_no_mask(N):
    """valid = NULL: every row valid (attention_forward without a RowMask)."""
    B, H = 6, 2
    h = inputs.make_host(B, H, N, D, seed=N + 31)
    res = run_gpu(h, None, 0.75, 1e-6, "bf16")
    assert_parity(res, oracle_for(res["inputs"], None, 0.75, 1e-6), None, "bf16")
