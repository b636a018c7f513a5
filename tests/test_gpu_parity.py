"""GPU parity: libcotten.so (through the C-ABI) vs the float64 CPU oracle.

Tolerances (north star), per (sequence, head) tensor, normwise
max|x - y| / max|y| against the oracle run on the SAME rounded inputs:
    f32  <= 1e-5        bf16 <= 1e-2        f64 <= 1e-12
Mask handling is bit-exact: dK / dV rows of padded positions are exactly 0,
padded K rows are never read (NaN there must not propagate), true_n is exact.
"""
import numpy as np
import pytest

import oracle
from paper_2602_06935_b200 import _lib, inputs, ops

pytestmark = pytest.mark.gpu

TOL = {"f32": 1e-5, "bf16": 1e-2, "f64": 1e-12}


def torch_mod():
    import torch
    return torch


def normwise(got, want, scale=None):
    """Max over units of max|got-want| / max|want| (units = leading two dims).
    ``scale`` (per unit) raises the denominator to the magnitude of the
    un-projected gradient for dQ/dK: (g - (g.x~)x~)/n cancels to O(eps) when
    d_h is 1 or 2, so there max|dQ| says nothing about the rounding budget."""
    g = got.reshape(got.shape[0] * got.shape[1], -1).astype(np.float64)
    w = want.reshape(want.shape[0] * want.shape[1], -1).astype(np.float64)
    den = np.abs(w).max(1)
    if scale is not None:
        den = np.maximum(den, scale)
    den = np.maximum(den, 1e-30)
    return float((np.abs(g - w).max(1) / den).max())


def proj_scales(inp, valid, m, eps):
    """Per unit: max_i |s dO_i S^T| / n_q,i and max_valid_i |V_i dA^T| / n_k,i."""
    B, H, N, D = inp["q"].shape
    sq, sk = np.zeros(B * H), np.zeros(B * H)
    for b in range(B):
        vm = None if valid is None else valid[b]
        for hh in range(H):
            r = oracle.fwd(inp["q"][b, hh], inp["k"][b, hh], inp["v"][b, hh], vm, m, eps)
            tn = N if vm is None else int(vm.sum())
            s = np.exp(-m * np.log(tn))
            g = s * inp["d_out"][b, hh] @ r["S"].T
            sq[b * H + hh] = np.abs(g / r["norm_q"][:, None]).max()
            dA = s * r["qn"].T @ inp["d_out"][b, hh]
            gk = inp["v"][b, hh] @ dA.T / r["norm_k"][:, None]
            if vm is not None:
                gk = gk[vm != 0]
            sk[b * H + hh] = np.abs(gk).max()
    return sq, sk


def run_gpu(h, valid, m, eps, dtype="f32", flags=0, layout="bhnd"):
    torch = torch_mod()
    tdt = {"f32": torch.float32, "bf16": torch.bfloat16, "f64": torch.float64}[dtype]
    B, H, N, D = h["q"].shape

    def dev(x):
        t = torch.from_numpy(np.ascontiguousarray(x)).to("cuda", tdt)
        if layout == "bnhd":  # [B, N, H, D] storage viewed as [B, H, N, D]
            t = t.permute(0, 2, 1, 3).contiguous().permute(0, 2, 1, 3)
        return t

    q, k, v, g = (dev(h[n]) for n in ("q", "k", "v", "d_out"))
    vm = None if valid is None else torch.from_numpy(valid).cuda()
    acc = torch.float64 if dtype == "f64" else torch.float32
    S = torch.empty((B * H, D, D), dtype=acc, device="cuda")
    out = torch.empty_like(q)
    ops.forward(q, k, v, vm, m, eps, out=out, saved_S=S, flags=flags)
    dm_unit = torch.empty(B * H, dtype=torch.float64, device="cuda")
    dm_total = torch.empty(1, dtype=torch.float64, device="cuda")
    dq, dk, dv = (torch.empty_like(q) for _ in range(3))
    ops.backward(q, k, v, vm, m, g, S, dq, dk, dv, dm_unit, dm_total, eps=eps, flags=flags)
    torch.cuda.synchronize()
    f = lambda t: t.double().cpu().numpy()  # noqa: E731
    return {"out": f(out), "dq": f(dq), "dk": f(dk), "dv": f(dv), "S": f(S),
            "dm_unit": dm_unit.cpu().numpy(), "dm_total": float(dm_total.item()),
            "inputs": {n: f(t) for n, t in (("q", q), ("k", k), ("v", v), ("d_out", g))}}


def oracle_for(inp, valid, m, eps):
    """Oracle over the exact values the device saw (already dtype-rounded)."""
    o = oracle.batched_f32
    if any(x.dtype == np.float64 and not np.array_equal(x, x.astype(np.float32))
           for x in inp.values()):
        return oracle_f64(inp, valid, m, eps)
    return o(inp["q"], inp["k"], inp["v"], inp["d_out"], valid, m, eps)


def oracle_f64(inp, valid, m, eps):
    B, H, N, D = inp["q"].shape
    outs = [np.empty((B, H, N, D)) for _ in range(4)]
    dm = np.empty(B * H)
    for b in range(B):
        for hh in range(H):
            r = oracle.fwd_bwd(inp["q"][b, hh], inp["k"][b, hh], inp["v"][b, hh],
                               inp["d_out"][b, hh], None if valid is None else valid[b], m, eps)
            for i in range(4):
                outs[i][b, hh] = r[i]
            dm[b * H + hh] = r[4]
    return (*outs, dm)


def assert_parity(res, ref, valid, dtype, m=None, eps=None):
    tol = TOL[dtype]
    out, dq, dk, dv, dm = ref
    scales = {}
    if m is not None and res["inputs"]["q"].shape[-1] <= 2:
        scales["dq"], scales["dk"] = proj_scales(res["inputs"], valid, m, eps)
    for name, want in (("out", out), ("dq", dq), ("dk", dk), ("dv", dv)):
        err = normwise(res[name], want, scales.get(name))
        assert err <= tol, f"{name}: normwise {err:.3e} > {tol}"
    # dm per unit, normwise over the batch of units (a sum of d^2 products can
    # cancel, so a per-unit relative error is not meaningful near zero)
    dm_err = np.abs(res["dm_unit"] - dm).max() / max(np.abs(dm).max(), 1e-30)
    assert dm_err <= tol, f"dm: normwise {dm_err:.3e}"
    if valid is not None:  # bit-exact padding: dK, dV exactly 0 on padded rows
        B, H = res["dk"].shape[:2]
        pad = np.broadcast_to((valid == 0)[:, None, :], (B, H, valid.shape[1]))
        assert np.all(res["dk"][pad] == 0.0) and np.all(res["dv"][pad] == 0.0)
    assert np.isfinite(res["dm_total"])
    assert res["dm_total"] == pytest.approx(float(np.sum(res["dm_unit"])), rel=1e-12, abs=1e-12)


PATHS = [0, _lib.FLAG_FP32_PIPE, _lib.FLAG_FORCE_GENERIC]
PATH_IDS = ["tcgen05", "fp32pipe", "generic"]


@pytest.mark.parametrize("flags", PATHS, ids=PATH_IDS)
@pytest.mark.parametrize("mask_kind", ["left", "random", "none"])
def test_ml1m_unit_shape_f32(flags, mask_kind):
    B, H, N, D = 24, 2, 200, 32
    h = inputs.make_host(B, H, N, D, seed=0)
    valid = {"left": inputs.left_padded_mask(B, N, 0), "random": inputs.random_mask(B, N, 1),
             "none": None}[mask_kind]
    res = run_gpu(h, valid, 1.0, 1e-6, "f32", flags)
    ref = oracle_for(res["inputs"], valid, 1.0, 1e-6)
    assert_parity(res, ref, valid, "f32")


@pytest.mark.parametrize("flags", PATHS[:2], ids=PATH_IDS[:2])
@pytest.mark.parametrize("N", [1, 2, 7, 8, 9, 31, 32, 33, 50, 65, 72, 96, 100, 127, 128, 129, 200, 255, 256, 257,
                               513, 1000, 2048, 4096, 16384])
def test_seq_len_edges_f32(N, flags):
    B, H, D = (5, 2, 32) if N <= 2048 else (2, 2, 32)
    h = inputs.make_host(B, H, N, D, seed=N)
    valid = inputs.left_padded_mask(B, N, N)
    res = run_gpu(h, valid, 0.75, 1e-6, "f32", flags)
    ref = oracle_for(res["inputs"], valid, 0.75, 1e-6)
    if N <= 3:
        # one to three rows: O = s (q~.k~) v cancels, so the error is bounded
        # against the magnitude evaluated on absolute values (the stated rule of
        # test_gpu_schedule.py::test_tiny_sequences_seed_sweep)
        from test_gpu_schedule import _abs_scales
        sc = _abs_scales(res["inputs"], valid, 0.75, 1e-6)
        for name, want in zip(("out", "dq", "dk", "dv"), ref[:4]):
            err = np.abs(res[name] - want).reshape(B * H, -1).max(1) / np.maximum(sc[name], 1e-30)
            assert err.max() <= 1e-5, (name, float(err.max()))
        pad = np.broadcast_to((valid == 0)[:, None, :], (B, H, N))
        assert np.all(res["dk"][pad] == 0.0) and np.all(res["dv"][pad] == 0.0)
    else:
        assert_parity(res, ref, valid, "f32")


@pytest.mark.parametrize("D", [1, 2, 3, 5, 8, 16, 24, 32, 48, 64, 96, 128])
def test_head_dims_f32(D):
    B, H, N = 3, 2, 70
    h = inputs.make_host(B, H, N, D, seed=D)
    valid = inputs.random_mask(B, N, D)
    res = run_gpu(h, valid, 1.25, 1e-6, "f32")
    assert_parity(res, oracle_for(res["inputs"], valid, 1.25, 1e-6), valid, "f32", 1.25, 1e-6)


@pytest.mark.parametrize("D", [1, 4, 16, 32, 64])
def test_f64_matches_oracle_tightly(D):
    B, H, N = 3, 2, 45
    rng = np.random.default_rng(D)
    h = {n: rng.uniform(-2, 2, (B, H, N, D)) for n in ("q", "k", "v", "d_out")}
    valid = inputs.random_mask(B, N, 100 + D)
    res = run_gpu(h, valid, 0.6, 1e-9, "f64")
    assert_parity(res, oracle_f64(res["inputs"], valid, 0.6, 1e-9), valid, "f64", 0.6, 1e-9)


@pytest.mark.parametrize("D", [32, 64])
def test_bf16_within_stated_tolerance(D):
    B, H, N = 8, 2, 200
    h = inputs.make_host(B, H, N, D, seed=3)
    valid = inputs.left_padded_mask(B, N, 3)
    res = run_gpu(h, valid, 1.0, 1e-6, "bf16")
    assert_parity(res, oracle_for(res["inputs"], valid, 1.0, 1e-6), valid, "bf16")


@pytest.mark.parametrize("flags", [0, _lib.FLAG_FP32_PIPE], ids=["tcgen05", "fp32pipe"])
@pytest.mark.parametrize("D", [64, 128])
@pytest.mark.parametrize("N", [7, 33, 64, 65, 200, 513, 1000, 4096])
def test_head_dim_64_128_seq_lens_f32(D, N, flags):
    """Both paths at d_h 64 / 128: the tensor-core kernels (kernels_tcf.cuh,
    kernels_tcg.cuh) and kernels_rt.cuh (register-tiled FP32 pipe, tile edges
    TR = 64 / 32 rows); the 512-row running-sum flush, left-padded masks."""
    B, H = (3, 2) if N <= 1000 else (2, 1)
    h = inputs.make_host(B, H, N, D, seed=N + D)
    valid = inputs.left_padded_mask(B, N, N)
    res = run_gpu(h, valid, 0.75, 1e-6, "f32", flags)
    assert_parity(res, oracle_for(res["inputs"], valid, 0.75, 1e-6), valid, "f32")


@pytest.mark.parametrize("D", [64, 128])
def test_head_dim_64_128_single_row(D):
    """N = 1 reduces every output to one d_h-term dot product times a vector:
    O and dV scale with q~.k~, dQ and dK with dO.v (S = k~ v^T, G = q~ dO^T).
    Those dots cancel for some units, and an fp32 sum of d_h terms is accurate
    to ~d_h u sum|terms|, not to 1e-5 of a cancelled result; each output's
    error is therefore scaled by its dot's condition number sum|x_a y_a| /
    |x.y| (the same kind of scaling the d_h <= 2 tests use)."""
    B, H, N = 3, 2, 1
    h = inputs.make_host(B, H, N, D, seed=N + D)
    valid = inputs.left_padded_mask(B, N, N)
    res = run_gpu(h, valid, 0.75, 1e-6, "f32")
    out, dq, dk, dv, dm = oracle_for(res["inputs"], valid, 0.75, 1e-6)
    x = {n: res["inputs"][n][:, :, 0, :].astype(np.float64) for n in ("q", "k", "v", "d_out")}
    unit = lambda a: a / np.linalg.norm(a, axis=-1, keepdims=True)  # noqa: E731

    def cond(a, b):
        prod = a * b
        return np.maximum((np.abs(prod).sum(-1) / np.abs(prod.sum(-1))).reshape(-1), 1.0)

    c_qk, c_dov = cond(unit(x["q"]), unit(x["k"])), cond(x["d_out"], x["v"])
    for name, want, c in (("out", out, c_qk), ("dv", dv, c_qk), ("dq", dq, c_dov), ("dk", dk, c_dov)):
        g = res[name].reshape(B * H, -1).astype(np.float64)
        w = want.reshape(B * H, -1)
        err = np.abs(g - w).max(1) / np.abs(w).max(1)
        assert np.all(err / c <= 1e-5), (name, err, c)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_head_dim_128_random_mask(dtype):
    B, H, N, D = 4, 2, 300, 128
    h = inputs.make_host(B, H, N, D, seed=21)
    valid = inputs.random_mask(B, N, 21)
    res = run_gpu(h, valid, 1.0, 1e-6, dtype)
    assert_parity(res, oracle_for(res["inputs"], valid, 1.0, 1e-6), valid, dtype)


@pytest.mark.parametrize("flags", [0, _lib.FLAG_FP32_PIPE], ids=["default", "fp32pipe"])
@pytest.mark.parametrize("D", [32, 64, 128])
@pytest.mark.parametrize("N", [5, 129, 1000])
def test_bf16_register_tiled_seq_lens(D, N, flags):
    """bf16 in HBM on kernels_rt.cuh (d_h 32 / 64 / 128, FP32_PIPE: tile edges
    of the 128 / 64 / 32-row tiles) and on the default path (the tensor-core
    kernels where the shape allows), random masks."""
    B, H = 3, 2
    h = inputs.make_host(B, H, N, D, seed=7 * N + D)
    valid = inputs.random_mask(B, N, N + D)
    res = run_gpu(h, valid, 1.0, 1e-6, "bf16", flags)
    assert_parity(res, oracle_for(res["inputs"], valid, 1.0, 1e-6), valid, "bf16")


@pytest.mark.parametrize("D", [64, 128])
def test_nan_in_padded_key_rows_never_read_rt(D):
    B, H, N = 3, 2, 150
    h = inputs.make_host(B, H, N, D, seed=22)
    valid = inputs.left_padded_mask(B, N, 22)
    clean = run_gpu(h, valid, 1.0, 1e-6)
    h2 = {n: x.copy() for n, x in h.items()}
    h2["k"][np.broadcast_to((valid == 0)[:, None, :], (B, H, N))] = np.nan
    dirty = run_gpu(h2, valid, 1.0, 1e-6)
    for n in ("out", "dq", "dk", "dv"):
        np.testing.assert_array_equal(clean[n], dirty[n])


def test_bnhd_strided_layout_equals_contiguous():
    B, H, N, D = 6, 2, 200, 32
    h = inputs.make_host(B, H, N, D, seed=5)
    valid = inputs.left_padded_mask(B, N, 5)
    a = run_gpu(h, valid, 1.0, 1e-6, "f32", layout="bhnd")
    b = run_gpu(h, valid, 1.0, 1e-6, "f32", layout="bnhd")
    for n in ("out", "dq", "dk", "dv"):
        np.testing.assert_array_equal(a[n], b[n])


@pytest.mark.parametrize("D,dtype", [(64, "f32"), (128, "f32"), (32, "bf16"), (64, "bf16")])
def test_bnhd_strided_layout_register_tiled(D, dtype):
    """The register-tiled kernels read a [B][N][H*D] projection output in
    place (stride_n = H*D): identical results to the contiguous layout.
    (COTTEN_FLAG_FP32_PIPE keeps both layouts on them: contiguous bf16 d_h 32
    would otherwise take the paired-row tensor-core kernel, fp32 d_h 64 the
    three-part one.)  The default path on the strided layout stays within
    the bar of the oracle."""
    B, H, N = 4, 2, 150
    h = inputs.make_host(B, H, N, D, seed=40 + D)
    valid = inputs.left_padded_mask(B, N, 40)
    fl = _lib.FLAG_FP32_PIPE
    a = run_gpu(h, valid, 1.0, 1e-6, dtype, layout="bhnd", flags=fl)
    b = run_gpu(h, valid, 1.0, 1e-6, dtype, layout="bnhd", flags=fl)
    for n in ("out", "dq", "dk", "dv"):
        np.testing.assert_array_equal(a[n], b[n])
    c = run_gpu(h, valid, 1.0, 1e-6, dtype, layout="bnhd")
    assert_parity(c, oracle_for(c["inputs"], valid, 1.0, 1e-6), valid, dtype)


def test_head_dim_64_long_sequence_accuracy():
    """N = 16384 at d_h = 64: the 512-row running-sum flush keeps the fp32
    reductions within the 1e-5 bar over 32 flushes."""
    B, H, N, D = 1, 1, 16384, 64
    h = inputs.make_host(B, H, N, D, seed=44)
    valid = inputs.left_padded_mask(B, N, 44)
    res = run_gpu(h, valid, 0.75, 1e-6, "f32")
    assert_parity(res, oracle_for(res["inputs"], valid, 0.75, 1e-6), valid, "f32")


def test_nan_in_padded_key_rows_never_read():
    # attention.cpp:334-338: padded K rows are selected to zero, never read
    B, H, N, D = 4, 2, 64, 32
    h = inputs.make_host(B, H, N, D, seed=9)
    valid = inputs.left_padded_mask(B, N, 9)
    clean = run_gpu(h, valid, 1.0, 1e-6)
    h2 = {n: x.copy() for n, x in h.items()}
    h2["k"][np.broadcast_to((valid == 0)[:, None, :], (B, H, N))] = np.nan
    dirty = run_gpu(h2, valid, 1.0, 1e-6)
    for n in ("out", "dq", "dk", "dv"):
        np.testing.assert_array_equal(clean[n], dirty[n])


def test_single_valid_row_and_true_n():
    B, H, N, D = 3, 2, 40, 32
    h = inputs.make_host(B, H, N, D, seed=10)
    valid = np.zeros((B, N), np.uint8)
    valid[0, 5] = valid[1, 39] = valid[2, 0] = 1
    res = run_gpu(h, valid, 1.5, 1e-6)
    assert_parity(res, oracle_for(res["inputs"], valid, 1.5, 1e-6), valid, "f32")


def test_dm_total_is_deterministic():
    B, H, N, D = 64, 2, 200, 32
    h = inputs.make_host(B, H, N, D, seed=11)
    valid = inputs.left_padded_mask(B, N, 11)
    a = run_gpu(h, valid, 1.0, 1e-6)
    b = run_gpu(h, valid, 1.0, 1e-6)
    assert a["dm_total"] == b["dm_total"]
    np.testing.assert_array_equal(a["dm_unit"], b["dm_unit"])


def test_empty_sequence_sets_status_on_device_path():
    torch = torch_mod()
    ops.device_status(0, reset=True)
    B, H, N, D = 2, 2, 16, 32
    q = torch.rand(B, H, N, D, device="cuda")
    valid = torch.ones(B, N, dtype=torch.uint8, device="cuda")
    valid[1] = 0
    out = ops.forward(q, q, q, valid, 1.0)
    torch.cuda.synchronize()
    assert ops.device_status(0, reset=True) & _lib.STATUS_EMPTY_SEQUENCE
    assert torch.isnan(out[1]).all() and torch.isfinite(out[0]).all()
    assert ops.device_status(0) == 0


def test_recomputed_state_equals_saved_state():
    torch = torch_mod()
    B, H, N, D = 8, 2, 200, 32
    h = inputs.make_host(B, H, N, D, seed=12)
    t = {n: torch.from_numpy(x).cuda() for n, x in h.items()}
    S = torch.empty(B * H, D, D, device="cuda")
    ops.forward(t["q"], t["k"], t["v"], None, 1.0, saved_S=S)
    a = ops.backward(t["q"], t["k"], t["v"], None, 1.0, t["d_out"], S)
    b = ops.backward(t["q"], t["k"], t["v"], None, 1.0, t["d_out"], None)
    for x, y in zip(a, b):
        assert torch.equal(x, y)


def test_saved_norms_match_cache_semantics():
    torch = torch_mod()
    B, H, N, D = 2, 2, 30, 32
    h = inputs.make_host(B, H, N, D, seed=13)
    valid = inputs.random_mask(B, N, 13)
    t = {n: torch.from_numpy(x).cuda() for n, x in h.items()}
    norms = torch.empty(B * H, 2, N, device="cuda")
    ops.forward(t["q"], t["k"], t["v"], torch.from_numpy(valid).cuda(), 1.0, saved_norms=norms)
    got = norms.cpu().numpy().astype(np.float64)
    for b in range(B):
        for hh in range(H):
            r = oracle.fwd(h["q"][b, hh], h["k"][b, hh], h["v"][b, hh], valid[b], 1.0, 1e-6)
            np.testing.assert_allclose(got[b * H + hh, 0], r["norm_q"], rtol=1e-6)
            np.testing.assert_allclose(got[b * H + hh, 1], r["norm_k"], rtol=1e-6)
            assert np.all(got[b * H + hh, 1][valid[b] == 0] == 1.0)  # attention.cpp:336


@pytest.mark.parametrize("config", ["beauty", "ml20m"])
def test_full_size_properties(config):
    """BASELINE configs at full size: sampled units vs the oracle, exact
    linearity in V (scaling by 2 is exact in fp32), exact zero padded
    gradients, and dm_total == ordered sum of dm_unit."""
    torch = torch_mod()
    B, H, N, D = {"beauty": (8192, 2, 50, 32), "ml20m": (65536, 2, 200, 32)}[config]
    t = inputs.make_device(B, H, N, D, seed=0)
    valid_np = inputs.left_padded_mask(B, N, 0)
    vm = torch.from_numpy(valid_np).cuda()
    S = torch.empty(B * H, D, D, device="cuda")
    out = ops.forward(t["q"], t["k"], t["v"], vm, 1.0, saved_S=S)
    dm_unit = torch.empty(B * H, dtype=torch.float64, device="cuda")
    dm_total = torch.empty(1, dtype=torch.float64, device="cuda")
    dq, dk, dv = ops.backward(t["q"], t["k"], t["v"], vm, 1.0, t["d_out"], S,
                              dm_unit=dm_unit, dm_total=dm_total)
    out2 = ops.forward(t["q"], t["k"], t["v"] * 2, vm, 1.0)
    assert torch.equal(out2, out * 2)
    pad = (vm == 0)[:, None, :].expand(B, H, N)
    assert bool((dk[pad] == 0).all()) and bool((dv[pad] == 0).all())
    rng = np.random.default_rng(0)
    dms, dms_ref = [], []
    for b in rng.choice(B, 24, replace=False):
        b = int(b)
        for hh in range(H):
            g = lambda x: x[b, hh].double().cpu().numpy()  # noqa: E731
            o = oracle.fwd_bwd(g(t["q"]), g(t["k"]), g(t["v"]), g(t["d_out"]), valid_np[b],
                               1.0, 1e-6)
            for got, want in zip((out, dq, dk, dv), o[:4]):
                assert np.abs(g(got) - want).max() / np.abs(want).max() <= 1e-5
            dms.append(dm_unit[b * H + hh].item())
            dms_ref.append(o[4])
    dms, dms_ref = np.array(dms), np.array(dms_ref)
    assert np.abs(dms - dms_ref).max() / np.abs(dms_ref).max() <= 1e-5
    assert dm_total.item() == pytest.approx(dm_unit.sum().item(), rel=1e-9)


@pytest.mark.parametrize("D,dtype", [(32, "f32"), (64, "f32"), (32, "bf16")])
def test_host_entry_slices_match_device_entry(D, dtype):
    """cotten_fwd_host / cotten_bwd_host stage the batch in pipelined slices of
    whole sequences (3 streams); the results must equal the single device call
    bit for bit: out, S, dQ, dK, dV, dm per unit and the fixed-order dm total,
    with the state given and recomputed, and an uneven last slice."""
    import ctypes
    torch = torch_mod()
    B, H, N = (301, 2, 200) if D == 32 else (151, 2, 200)
    h = inputs.make_host(B, H, N, D, seed=31)
    valid = inputs.left_padded_mask(B, N, 31)
    ref = run_gpu(h, valid, 1.0, 1e-6, dtype)
    lib = _lib.load()
    tdt = {"f32": torch.float32, "bf16": torch.bfloat16}[dtype]
    host = {n: torch.from_numpy(h[n]).to(tdt).contiguous().pin_memory() for n in ("q", "k", "v", "d_out")}
    vm = torch.from_numpy(valid).contiguous().pin_memory()
    outs = {n: torch.empty((B, H, N, D), dtype=tdt).pin_memory() for n in ("out", "dq", "dk", "dv")}
    S = torch.empty((B * H, D, D), dtype=torch.float32).pin_memory()
    dm_unit = torch.empty(B * H, dtype=torch.float64).pin_memory()
    dm_total = torch.empty(1, dtype=torch.float64).pin_memory()
    desc = _lib.make_desc(B, H, N, D, dtype, 1e-6)
    p = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    _lib.check(lib.cotten_fwd_host(ctypes.byref(desc), p(host["q"]), p(host["k"]), p(host["v"]), p(vm),
                                   1.0, p(outs["out"]), p(S), None))
    for saved in (S, None):
        _lib.check(lib.cotten_bwd_host(ctypes.byref(desc), p(host["q"]), p(host["k"]), p(host["v"]),
                                       p(vm), 1.0, p(host["d_out"]), None if saved is None else p(saved),
                                       p(outs["dq"]), p(outs["dk"]), p(outs["dv"]), p(dm_unit),
                                       p(dm_total)))
        for n in ("out", "dq", "dk", "dv"):
            np.testing.assert_array_equal(outs[n].double().numpy(), ref[n], err_msg=n)
        np.testing.assert_array_equal(S.double().numpy(), ref["S"])
        np.testing.assert_array_equal(dm_unit.numpy(), ref["dm_unit"])
        assert float(dm_total.item()) == ref["dm_total"]
