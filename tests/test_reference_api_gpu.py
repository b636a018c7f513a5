"""The reference's own hot-path tests, re-expressed against the GPU operator
through the reference-shaped API (paper_2602_06935_b200.ops -> C-ABI host
entry points -> sm_100a kernels).  cfg.dtype = "f64" runs the float64
kernels, so the reference's tolerances apply unchanged; the f32 variants use
the north-star 1e-5 normwise bar.

Sources: /root/reference/proj/tests/test_attention.cpp:93-187,212-251,334-341,
test_attention_grad.cpp:62-123,153-189, acceptance.cpp:60-116.
"""
import os

import numpy as np
import pytest

import oracle
from paper_2602_06935_b200 import ops
from paper_2602_06935_b200.ops import AttentionCache, AttentionConfig, RowMask

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "cosine_golden.npz")


def cfg(eps=1e-9, tile=32, dtype="f64"):
    return AttentionConfig(mechanism="cosine", eps=eps, tile_size=tile, dtype=dtype)


def rand(rng, n, d, lo=-1.0, hi=1.0):
    return rng.uniform(lo, hi, (n, d))


def test_n1_q_equals_k_returns_v():  # test_attention.cpp:142-148
    rng = np.random.default_rng(9)
    q, v = rand(rng, 1, 8), rand(rng, 1, 8)
    out = ops.cosine_attention_fused(q, q, v, 1.3, cfg(1e-12))
    assert np.abs(out - v).max() < 1e-10


def test_orthogonal_q_k_give_zeros():  # test_attention.cpp:101-110
    q, k, v = np.zeros((2, 4)), np.zeros((2, 4)), np.full((2, 4), 5.0)
    q[0, 0], q[1, 1], k[0, 2], k[1, 3] = 1.0, 2.0, 3.0, -1.0
    assert np.abs(ops.cosine_attention_fused(q, k, v, 1.0, cfg(1e-12))).max() < 1e-12


def test_2x2_hand_computation():  # test_attention.cpp:112-123
    out = ops.cosine_attention_fused(np.eye(2), np.eye(2), np.diag([2.0, 4.0]), 1.0, cfg(1e-13))
    np.testing.assert_allclose(out, np.diag([1.0, 2.0]), atol=1e-9)


@pytest.mark.parametrize("dtype,tol", [("f64", 1e-10), ("f32", 1e-5)])
def test_fused_equals_naive_oracle(dtype, tol):  # test_attention.cpp:125-140 / acceptance C1
    rng = np.random.default_rng(8)
    worst = 0.0
    for it in range(60):
        n, d = int(rng.integers(1, 129)), int(rng.integers(1, 17))
        q, k, v = (rand(rng, n, d, -2, 2) for _ in range(3))
        m = 0.25 * (it % 8)
        want = oracle.naive(q, k, v, m, 1e-9)
        got = ops.cosine_attention_fused(q, k, v, m, cfg(1e-9, dtype=dtype))
        err = np.abs(got - want).max()
        worst = max(worst, err if dtype == "f64" else err / max(np.abs(want).max(), 1e-30))
    assert worst < tol


def test_row_scale_invariance():  # test_attention.cpp:150-160
    rng = np.random.default_rng(10)
    q, k, v = (rand(rng, 7, 5) for _ in range(3))
    base = ops.cosine_attention_fused(q, k, v, 1.0, cfg(1e-14, 4))
    q2 = q.copy()
    q2[3] *= 17.5
    k2 = k.copy()
    k2[5] *= 0.004
    assert np.abs(ops.cosine_attention_fused(q2, k, v, 1.0, cfg(1e-14, 4)) - base).max() < 1e-9
    assert np.abs(ops.cosine_attention_fused(q, k2, v, 1.0, cfg(1e-14, 4)) - base).max() < 1e-9


def test_output_bounded_by_max_v_at_m1():  # test_attention.cpp:162-170
    rng = np.random.default_rng(11)
    for _ in range(25):
        q, k = rand(rng, 9, 4), rand(rng, 9, 4)
        v = rand(rng, 9, 4, -3, 3)
        out = ops.cosine_attention_fused(q, k, v, 1.0, cfg(tile=5))
        assert np.abs(out).max() <= np.abs(v).max() + 1e-12


def test_masked_equals_real_rows_only():  # test_attention.cpp:212-251
    rng = np.random.default_rng(15)
    n_real, n_pad, d = 5, 3, 4
    qr, kr, vr = (rand(rng, n_real, d) for _ in range(3))
    junk = np.random.default_rng(99)
    q, k, v = (np.vstack([junk.uniform(-9, 9, (n_pad, d)), x]) for x in (qr, kr, vr))
    mask = RowMask.from_valid([0] * n_pad + [1] * n_real)
    full = ops.cosine_attention_fused(q, k, v, 1.0, cfg(tile=3), None, mask)
    sub = ops.cosine_attention_fused(qr, kr, vr, 1.0, cfg(tile=3))
    assert np.abs(full[n_pad:] - sub).max() < 1e-10


def test_zero_upstream_gradient():  # test_attention_grad.cpp:62-78
    rng = np.random.default_rng(100)
    q, k, v = (rand(rng, 4, 3) for _ in range(3))
    cache = AttentionCache()
    ops.attention_forward(q, k, v, 1.0, cfg(1e-6, 2), cache)
    g = ops.attention_backward(cache, np.zeros((4, 3)))
    assert not g.dq.any() and not g.dk.any() and not g.dv.any() and g.dm == 0.0


def test_dm_closed_form():  # test_attention_grad.cpp:107-123
    rng = np.random.default_rng(600)
    q = rand(rng, 4, 3, 0.1, 1.0)
    v = rand(rng, 4, 3, 0.1, 1.0)
    cache = AttentionCache()
    out = ops.attention_forward(q, q.copy(), v, 1.0, cfg(1e-9, 2), cache)
    g = ops.attention_backward(cache, out)
    assert abs(g.dm - (-np.log(4.0) * np.sum(out * out))) < 1e-8 and g.dm < 0


def _fd(f, x, step=1e-5):
    g = np.zeros_like(x)
    for i in np.ndindex(x.shape):
        s = x[i]
        x[i] = s + step
        up = f()
        x[i] = s - step
        dn = f()
        x[i] = s
        g[i] = (up - dn) / (2 * step)
    return g


def _rel(a, b):  # support/test_util.hpp:35-37
    return np.abs(a - b) / np.maximum(1.0, np.maximum(np.abs(a), np.abs(b)))


@pytest.mark.parametrize("seed,n,d,masked", [(401, 6, 4, False), (402, 9, 5, False), (800, 6, 3, True)])
def test_backward_matches_finite_differences(seed, n, d, masked):
    # test_attention_grad.cpp:90-93 (incl. dm), :153-189 (masked); acceptance C2
    rng = np.random.default_rng(seed)
    q, k, v, w = (rand(rng, n, d) for _ in range(4))
    m = np.array([0.5 + 0.5 * rng.uniform()])
    mask = None
    if masked:
        mask = RowMask.from_valid([0, 0] + [1] * (n - 2))
        w[:2] = 0.0
    c = cfg(1e-6, 3)
    f = lambda: float(np.sum(ops.cosine_attention_fused(q, k, v, m[0], c, None, mask) * w))  # noqa
    cache = AttentionCache()
    ops.cosine_attention_fused(q, k, v, m[0], c, cache, mask)
    g = ops.cosine_attention_backward(cache, w)
    worst = max(_rel(g.dq, _fd(f, q)).max(), _rel(g.dk, _fd(f, k)).max(),
                _rel(g.dv, _fd(f, v)).max(), _rel(np.array([g.dm]), _fd(f, m)).max())
    assert worst < 1e-4


def test_cache_fields_match_reference_cache():
    """The GPU forward fills AttentionCache like attention.cpp:308-322,390-393."""
    rng = np.random.default_rng(21)
    n, d = 20, 6
    q, k, v = (rand(rng, n, d) for _ in range(3))
    valid = (rng.random(n) < 0.5).astype(np.uint8)
    valid[3] = 1
    cache = AttentionCache()
    ops.cosine_attention_fused(q, k, v, 0.9, cfg(1e-6), cache, RowMask.from_valid(valid))
    r = oracle.fwd(q, k, v, valid, 0.9, 1e-6)
    np.testing.assert_allclose(cache.kv, r["S"], atol=1e-12)
    np.testing.assert_allclose(cache.norm_q[:, 0], r["norm_q"], rtol=1e-13)
    np.testing.assert_allclose(cache.norm_k[:, 0], r["norm_k"], rtol=1e-13)
    np.testing.assert_allclose(cache.qn, r["qn"], atol=1e-13)
    np.testing.assert_allclose(cache.kn, r["kn"], atol=1e-13)
    assert cache.true_n == int(valid.sum()) and cache.mechanism == "cosine"


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_golden_vectors_through_gpu(dtype):
    z = np.load(GOLDEN)
    names = sorted({k.split("/")[0] for k in z.files})
    for name in names:
        g = lambda key: z[name + "/" + key]  # noqa: E731
        n, d, m, eps = g("meta")
        valid = g("valid")
        mask = None if valid.size == 0 else RowMask.from_valid(valid)
        cache = AttentionCache()
        out = ops.cosine_attention_fused(g("q"), g("k"), g("v"), m, cfg(eps, dtype=dtype), cache,
                                         mask)
        grads = ops.cosine_attention_backward(cache, g("d_out"))
        tol = 1e-11 if dtype == "f64" else 1e-5
        # un-projected gradient magnitudes (the projection cancels for d_h <= 2)
        s = np.exp(-m * np.log(g("true_n")[0]))
        gq = np.abs(s * g("d_out") @ g("S").T / g("norm_q")[:, None]).max()
        dA = s * g("qn").T @ g("d_out")
        gk = np.abs(g("v") @ dA.T / g("norm_k")[:, None])
        gk = gk[valid != 0].max() if mask is not None else gk.max()
        floor = {"dq": gq, "dk": gk}
        for got, key in ((out, "out"), (grads.dq, "dq"), (grads.dk, "dk"), (grads.dv, "dv")):
            want = g(key)
            den = max(np.abs(want).max(), floor.get(key, 0.0) if d <= 2 else 0.0, 1e-300)
            err = np.abs(got - want).max() / den
            assert err <= tol, f"{name}/{key} ({dtype}): {err:.3e}"
        assert abs(grads.dm - g("dm")[0]) <= tol * max(1.0, abs(g("dm")[0])) * 10
        if mask is not None:
            assert np.all(grads.dk[valid == 0] == 0) and np.all(grads.dv[valid == 0] == 0)
