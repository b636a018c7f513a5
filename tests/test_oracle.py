"""Pins the CPU oracle (oracle/cosine_oracle.c) before anything trusts it.

* bit-exact against the reference itself (oracle/_ref, compiled from
  /root/reference sources) on random masked shapes;
* against the committed golden vectors (tests/golden/, made from the
  reference by make_golden.py);
* against the reference's own known-answer tests, re-expressed
  (test_attention.cpp, test_attention_grad.cpp, acceptance.cpp C1/C2).
"""
import os

import numpy as np
import pytest

import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "cosine_golden.npz")
needs_ref = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")


def golden_cases():
    z = np.load(GOLDEN)
    names = sorted({k.split("/")[0] for k in z.files})
    return z, names


def test_golden_file_present():
    z, names = golden_cases()
    assert len(names) >= 15


@pytest.mark.parametrize("name", golden_cases()[1])
def test_oracle_matches_golden(name):
    z = np.load(GOLDEN)
    g = lambda k: z[name + "/" + k]  # noqa: E731
    n, d, m, eps = g("meta")
    valid = g("valid")
    valid = None if valid.size == 0 else valid
    fw = oracle.fwd(g("q"), g("k"), g("v"), valid, m, eps)
    for key in ("out", "norm_q", "norm_k", "qn", "kn", "S"):
        np.testing.assert_array_equal(fw[key], g(key), err_msg=key)  # bit-exact
    out, dq, dk, dv, dm = oracle.fwd_bwd(g("q"), g("k"), g("v"), g("d_out"), valid, m, eps)
    np.testing.assert_array_equal(out, g("out"))
    np.testing.assert_array_equal(dq, g("dq"))
    np.testing.assert_array_equal(dk, g("dk"))
    np.testing.assert_array_equal(dv, g("dv"))
    assert dm == g("dm")[0]


@needs_ref
@pytest.mark.parametrize("seed", range(40))
def test_oracle_bit_exact_vs_reference(seed):
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(1, 129))
    d = int(rng.integers(1, 33))
    m = float(rng.uniform(0, 2))
    eps = float(10.0 ** rng.uniform(-12, -3))
    q, k, v, g = (rng.uniform(-2, 2, (n, d)) for _ in range(4))
    valid = None
    if seed % 3:
        valid = (rng.random(n) < 0.6).astype(np.uint8)
        valid[int(rng.integers(0, n))] = 1
    tile = int(rng.choice([1, 3, 32, n + 7]))
    ref = oracle.ref_fwd(q, k, v, valid, m, eps, tile)
    mine = oracle.fwd(q, k, v, valid, m, eps)
    for key in ("out", "norm_q", "norm_k", "qn", "kn", "S"):
        np.testing.assert_array_equal(mine[key], ref[key], err_msg=key)
    r = oracle.ref_fwd_bwd(q, k, v, g, valid, m, eps, tile)
    o = oracle.fwd_bwd(q, k, v, g, valid, m, eps)
    for a, b in zip(o[:4], r[:4]):
        np.testing.assert_array_equal(a, b)
    assert o[4] == r[4]


@needs_ref
def test_naive_route_matches_reference():
    rng = np.random.default_rng(5)
    for _ in range(20):
        n, d = int(rng.integers(1, 60)), int(rng.integers(1, 17))
        q, k, v = (rng.uniform(-2, 2, (n, d)) for _ in range(3))
        m = float(rng.uniform(0, 2))
        np.testing.assert_allclose(oracle.naive(q, k, v, m, 1e-9), oracle.ref_naive(q, k, v, m, 1e-9),
                                   rtol=0, atol=1e-13)


# ---- the reference's known-answer tests, on the oracle ----------------------

def test_kat_n1_q_equals_k_returns_v():  # test_attention.cpp:142-148
    rng = np.random.default_rng(9)
    q, v = rng.uniform(-1, 1, (1, 8)), rng.uniform(-1, 1, (1, 8))
    out = oracle.fwd(q, q, v, None, 1.3, 1e-12)["out"]
    assert np.abs(out - v).max() < 1e-10


def test_kat_orthogonal_gives_zero():  # test_attention.cpp:101-110
    q, k, v = np.zeros((2, 4)), np.zeros((2, 4)), np.full((2, 4), 5.0)
    q[0, 0], q[1, 1], k[0, 2], k[1, 3] = 1.0, 2.0, 3.0, -1.0
    assert np.abs(oracle.fwd(q, k, v, None, 1.0, 1e-12)["out"]).max() < 1e-12


def test_kat_2x2_hand_computation():  # test_attention.cpp:112-123
    q, v = np.eye(2), np.diag([2.0, 4.0])
    out = oracle.fwd(q, q, v, None, 1.0, 1e-13)["out"]
    np.testing.assert_allclose(out, np.diag([1.0, 2.0]), atol=1e-9)


def test_fused_equals_naive_200_instances():  # test_attention.cpp:125-140, acceptance C1
    rng = np.random.default_rng(8)
    worst = 0.0
    for it in range(200):
        n, d = int(rng.integers(1, 129)), int(rng.integers(1, 17))
        q, k, v = (rng.uniform(-2, 2, (n, d)) for _ in range(3))
        m = 0.25 * (it % 8)
        worst = max(worst, np.abs(oracle.fwd(q, k, v, None, m, 1e-9)["out"]
                                  - oracle.naive(q, k, v, m, 1e-9)).max())
    assert worst < 1e-10


def test_masked_equals_real_subset():  # test_attention.cpp:212-251
    rng = np.random.default_rng(15)
    n_real, n_pad, d = 5, 3, 4
    qr, kr, vr = (rng.uniform(-1, 1, (n_real, d)) for _ in range(3))
    q, k, v = (np.vstack([rng.uniform(-9, 9, (n_pad, d)), x]) for x in (qr, kr, vr))
    valid = np.r_[np.zeros(n_pad), np.ones(n_real)].astype(np.uint8)
    full = oracle.fwd(q, k, v, valid, 1.0, 1e-9)["out"]
    sub = oracle.fwd(qr, kr, vr, None, 1.0, 1e-9)["out"]
    assert np.abs(full[n_pad:] - sub).max() < 1e-10


def test_zero_upstream_gives_zero_grads():  # test_attention_grad.cpp:62-78
    rng = np.random.default_rng(100)
    q, k, v = (rng.uniform(-1, 1, (4, 3)) for _ in range(3))
    _, dq, dk, dv, dm = oracle.fwd_bwd(q, k, v, np.zeros((4, 3)), None, 1.0, 1e-6)
    assert not dq.any() and not dk.any() and not dv.any() and dm == 0.0


def test_dm_closed_form():  # test_attention_grad.cpp:107-123
    rng = np.random.default_rng(600)
    q = rng.uniform(0.1, 1.0, (4, 3))
    v = rng.uniform(0.1, 1.0, (4, 3))
    out = oracle.fwd(q, q, v, None, 1.0, 1e-9)["out"]
    dm = oracle.fwd_bwd(q, q, v, out, None, 1.0, 1e-9)[4]
    assert abs(dm - (-np.log(4.0) * np.sum(out * out))) < 1e-8 and dm < 0


def _fd(f, x, step=1e-5):  # support/oracles.hpp:63-87
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
def test_gradients_match_finite_differences(seed, n, d, masked):
    # test_attention_grad.cpp:90-93 (incl. dm) and :153-189 (masked)
    rng = np.random.default_rng(seed)
    q, k, v, w = (rng.uniform(-1, 1, (n, d)) for _ in range(4))
    m = np.array([0.5 + 0.5 * rng.uniform()])
    valid = None
    if masked:
        valid = np.ones(n, np.uint8)
        valid[:2] = 0
        w[:2] = 0.0
    f = lambda: float(np.sum(oracle.fwd(q, k, v, valid, m[0], 1e-6)["out"] * w))  # noqa: E731
    _, dq, dk, dv, dm = oracle.fwd_bwd(q, k, v, w, valid, m[0], 1e-6)
    worst = max(_rel(dq, _fd(f, q)).max(), _rel(dk, _fd(f, k)).max(), _rel(dv, _fd(f, v)).max())
    worst = max(worst, _rel(np.array([dm]), _fd(f, m)).max())
    assert worst < 1e-4


@needs_ref
def test_reference_error_codes():
    # check_qkv: true_count == 0 -> UsageError (code 2); missing cache -> UsageError
    q = np.ones((3, 2))
    with pytest.raises(oracle.OracleError):
        oracle.ref_fwd(q, q, q, np.zeros(3, np.uint8))
    assert oracle.ref_error_code("cosref_bwd_without_cache", 2, 2) == 2
