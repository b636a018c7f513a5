"""GPU tests of the C-ABI's edge contracts: host entry points on dense layouts
whose batch is not the outermost dimension, outputs allocated for a gapped
(fused-projection) q, per-stream workspaces (two streams of one host thread,
both asking for the in-kernel dm total), and the device-resident host cache
(cotten_*_host_cached: bit-identical to the uncached pair, backward on another
thread, pooled buffers, the missing-cache UsageError of attention.cpp:398-400)."""
import ctypes

import numpy as np
import pytest

import oracle
from paper_2602_06935_b200 import _lib, inputs, ops

pytestmark = pytest.mark.gpu


def _torch():
    import torch
    return torch


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr())


@pytest.mark.parametrize("order", ["nbhd", "hbnd"])
def test_host_entry_non_batch_major_dense_layout(order):
    """cotten_fwd_host / cotten_bwd_host with a gap-free layout whose
    outermost dimension is N or H: the whole span is staged (one slice), and
    the results equal the contiguous device call."""
    torch = _torch()
    B, H, N, D = 64, 2, 200, 32
    h = inputs.make_host(B, H, N, D, seed=77)
    valid = inputs.left_padded_mask(B, N, 77)
    perm = {"nbhd": (2, 0, 1, 3), "hbnd": (1, 0, 2, 3)}[order]
    host = {}
    for n, x in h.items():  # storage in `order`, viewed as [B, H, N, D]
        st = torch.from_numpy(np.ascontiguousarray(x.transpose(perm))).pin_memory()
        inv = np.argsort(perm)
        host[n] = st.permute(*inv)
    strides = host["q"].stride()
    desc = _lib.make_desc(B, H, N, D, "f32", 1e-6, strides[:3])
    outs = {}
    for n in ("out", "dq", "dk", "dv"):
        st = torch.empty([(B, H, N, D)[i] for i in perm], dtype=torch.float32).pin_memory()
        outs[n] = st.permute(*np.argsort(perm))
    S = torch.empty(B * H, D, D).pin_memory()
    dm_total = torch.zeros(1, dtype=torch.float64).pin_memory()
    vm = torch.from_numpy(valid).pin_memory()
    lib = _lib.load()
    _lib.check(lib.cotten_fwd_host(ctypes.byref(desc), _ptr(host["q"]), _ptr(host["k"]),
                                   _ptr(host["v"]), _ptr(vm), 1.0, _ptr(outs["out"]), _ptr(S), None))
    _lib.check(lib.cotten_bwd_host(ctypes.byref(desc), _ptr(host["q"]), _ptr(host["k"]),
                                   _ptr(host["v"]), _ptr(vm), 1.0, _ptr(host["d_out"]), _ptr(S),
                                   _ptr(outs["dq"]), _ptr(outs["dk"]), _ptr(outs["dv"]), None,
                                   _ptr(dm_total)))
    ref = oracle.batched_f32(h["q"], h["k"], h["v"], h["d_out"], valid, 1.0, 1e-6)
    for name, want in zip(("out", "dq", "dk", "dv"), ref[:4]):
        got = outs[name].contiguous().double().numpy().reshape(B * H, -1)
        w = want.reshape(B * H, -1)
        err = float((np.abs(got - w).max(1) / np.abs(w).max(1)).max())
        assert err <= 1e-5, (name, err)
    assert dm_total.item() == pytest.approx(ref[4].sum(), rel=1e-5)


@pytest.mark.parametrize("D", [32, 64])
def test_outputs_for_gapped_q_keep_its_strides(D):
    """q, k, v as slices of one fused [B, N, 3*H*D] projection output: the
    outputs forward()/backward() allocate get q's strides (empty_like would
    return a dense tensor 3x too small for writes at q's strides)."""
    torch = _torch()
    B, H, N = 16, 2, 200
    x = torch.rand(B, N, 3 * H * D, device="cuda") * 2 - 1
    q, k, v = (x[..., i * H * D:(i + 1) * H * D].view(B, N, H, D).transpose(1, 2) for i in range(3))
    g = torch.rand(B, N, H * D, device="cuda").view(B, N, H, D).transpose(1, 2) * 2 - 1
    g = torch.empty_strided(q.shape, q.stride(), device="cuda").copy_(g)
    guard = torch.full((4 << 20,), 7.0, device="cuda")  # a neighbour allocation that must survive
    S = torch.empty(B * H, D, D, device="cuda")
    out = ops.forward(q, k, v, None, 1.0, saved_S=S)
    dq, dk, dv = ops.backward(q, k, v, None, 1.0, g, S)
    torch.cuda.synchronize()
    assert out.stride() == q.stride() and dq.stride() == q.stride()
    assert bool((guard == 7.0).all())
    qc, kc, vc, gc = (t.contiguous() for t in (q, k, v, g))
    out2 = ops.forward(qc, kc, vc, None, 1.0, saved_S=S)
    dq2, dk2, dv2 = ops.backward(qc, kc, vc, None, 1.0, gc, S)
    for a, b in ((out, out2), (dq, dq2), (dk, dk2), (dv, dv2)):
        assert torch.equal(a.contiguous(), b)


def test_two_streams_one_thread_dm_total():
    """Two concurrent cotten_bwd(..., dm_total) calls from one host thread on
    two streams: each stream has its own CTA-completion counter and dm
    scratch, so both totals equal their single-stream values (repeatedly)."""
    torch = _torch()
    B, H, N, D = 512, 2, 200, 32
    sets = []
    for seed in (5, 6):
        t = inputs.make_device(B, H, N, D, seed=seed)
        t["valid"] = torch.from_numpy(inputs.left_padded_mask(B, N, seed)).cuda()
        t["S"] = torch.empty(B * H, D, D, device="cuda")
        ops.forward(t["q"], t["k"], t["v"], t["valid"], 1.0, saved_S=t["S"])
        t["ref"] = torch.empty(1, dtype=torch.float64, device="cuda")
        ops.backward(t["q"], t["k"], t["v"], t["valid"], 1.0, t["d_out"], t["S"], dm_total=t["ref"])
        sets.append(t)
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    for s, t in zip(streams, sets):  # first use of each stream: workspace allocation
        ops.backward(t["q"], t["k"], t["v"], t["valid"], 1.0, t["d_out"], t["S"],
                     dm_total=torch.empty(1, dtype=torch.float64, device="cuda"), stream=s)
    torch.cuda.synchronize()
    for rep in range(20):
        tots = [torch.empty(1, dtype=torch.float64, device="cuda") for _ in sets]
        for s, t, tot in zip(streams, sets, tots):
            s.wait_stream(torch.cuda.current_stream())
            ops.backward(t["q"], t["k"], t["v"], t["valid"], 1.0, t["d_out"], t["S"],
                         dm_total=tot, stream=s)
        torch.cuda.synchronize()
        for t, tot in zip(sets, tots):
            assert tot.item() == t["ref"].item(), rep


def _host_inputs(B, H, N, D, seed, dtype="f32"):
    torch = _torch()
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    h = inputs.make_host(B, H, N, D, seed=seed)
    t = {n: torch.from_numpy(x).to(tdt).contiguous() for n, x in h.items()}
    t["valid"] = torch.from_numpy(inputs.left_padded_mask(B, N, seed)).contiguous()
    return t


@pytest.mark.parametrize("D,dtype,N", [(32, "f32", 200), (64, "f32", 300), (32, "bf16", 256),
                                       (32, "f32", 50), (128, "f32", 300), (128, "bf16", 256)])
def test_cached_host_pair_equals_uncached_host_pair(D, dtype, N):
    """cotten_fwd_host_cached / cotten_bwd_host_cached (the AttentionCache kept on
    the device) give bit-identical outputs to cotten_fwd_host / cotten_bwd_host."""
    torch = _torch()
    lib = _lib.load()
    B, H = 37, 2
    t = _host_inputs(B, H, N, D, seed=D + N, dtype=dtype)
    desc = _lib.make_desc(B, H, N, D, dtype, 1e-6)
    z = lambda: torch.empty_like(t["q"])  # noqa: E731
    o1, dq1, dk1, dv1 = z(), z(), z(), z()
    S = torch.empty(B * H, D, D)
    dm1 = torch.zeros(1, dtype=torch.float64)
    _lib.check(lib.cotten_fwd_host(ctypes.byref(desc), _ptr(t["q"]), _ptr(t["k"]), _ptr(t["v"]),
                                   _ptr(t["valid"]), 0.75, _ptr(o1), _ptr(S), None))
    _lib.check(lib.cotten_bwd_host(ctypes.byref(desc), _ptr(t["q"]), _ptr(t["k"]), _ptr(t["v"]),
                                   _ptr(t["valid"]), 0.75, _ptr(t["d_out"]), _ptr(S), _ptr(dq1),
                                   _ptr(dk1), _ptr(dv1), None, _ptr(dm1)))
    o2, dq2, dk2, dv2 = z(), z(), z(), z()
    dm2 = torch.zeros(1, dtype=torch.float64)
    dmu = torch.zeros(B * H, dtype=torch.float64)
    c = ctypes.c_void_p()
    _lib.check(lib.cotten_fwd_host_cached(ctypes.byref(desc), _ptr(t["q"]), _ptr(t["k"]),
                                          _ptr(t["v"]), _ptr(t["valid"]), 0.75, _ptr(o2), None,
                                          ctypes.byref(c)))
    assert c.value
    _lib.check(lib.cotten_bwd_host_cached(c, _ptr(t["d_out"]), _ptr(dq2), _ptr(dk2), _ptr(dv2),
                                          _ptr(dmu), _ptr(dm2)))
    _lib.check(lib.cotten_host_cache_free(c))
    for a, b in ((o1, o2), (dq1, dq2), (dk1, dk2), (dv1, dv2), (dm1, dm2)):
        assert torch.equal(a, b)
    assert float(dm2) == pytest.approx(float(dmu.sum()), rel=1e-12, abs=1e-12)


def test_cached_backward_on_another_thread_and_pool_reuse():
    import threading
    torch = _torch()
    lib = _lib.load()
    B, H, N, D = 20, 2, 200, 32
    t = _host_inputs(B, H, N, D, seed=3)
    desc = _lib.make_desc(B, H, N, D, "f32", 1e-6)
    outs = []
    for rep in range(3):  # freed caches' device buffers are reused by the next forward
        c = ctypes.c_void_p()
        o = torch.empty_like(t["q"])
        _lib.check(lib.cotten_fwd_host_cached(ctypes.byref(desc), _ptr(t["q"]), _ptr(t["k"]),
                                              _ptr(t["v"]), _ptr(t["valid"]), 1.0, _ptr(o), None,
                                              ctypes.byref(c)))
        g = [torch.empty_like(t["q"]) for _ in range(3)]
        rc = []
        th = threading.Thread(target=lambda: rc.append(lib.cotten_bwd_host_cached(
            c, _ptr(t["d_out"]), _ptr(g[0]), _ptr(g[1]), _ptr(g[2]), None, None)))
        th.start()
        th.join()
        assert rc == [0]
        _lib.check(lib.cotten_host_cache_free(c))
        outs.append((o, *g))
    for a, b in zip(outs[0], outs[2]):
        assert torch.equal(a, b)
    ref = oracle.batched_f32(t["q"].numpy(), t["k"].numpy(), t["v"].numpy(), t["d_out"].numpy(),
                             t["valid"].numpy(), 1.0, 1e-6)
    for got, want in zip(outs[0], ref[:4]):
        g = got.double().numpy().reshape(B * H, -1)
        w = want.reshape(B * H, -1)
        assert float((np.abs(g - w).max(1) / np.abs(w).max(1)).max()) <= 1e-5


def test_many_host_threads_through_the_gate():
    """12 threads (more than the default 8 concurrent host calls the gate
    admits) each run cached fwd + bwd on their own batch slice, 3 times; every
    slice equals the same call made alone, and nothing deadlocks."""
    import threading
    torch = _torch()
    lib = _lib.load()
    B, H, N, D, W = 48, 2, 200, 32, 12
    t = _host_inputs(B, H, N, D, seed=9)
    per = B // W
    es = 4

    def call(b0, outs):
        dsc = _lib.make_desc(per, H, N, D, "f32", 1e-6)
        off = b0 * H * N * D * es
        q = lambda x: ctypes.c_void_p(x.data_ptr() + off)  # noqa: E731
        c = ctypes.c_void_p()
        rc = lib.cotten_fwd_host_cached(ctypes.byref(dsc), q(t["q"]), q(t["k"]), q(t["v"]),
                                        ctypes.c_void_p(t["valid"].data_ptr() + b0 * N), 1.0,
                                        q(outs[0]), None, ctypes.byref(c))
        if rc == 0:
            rc = lib.cotten_bwd_host_cached(c, q(t["d_out"]), q(outs[1]), q(outs[2]), q(outs[3]),
                                            None, None)
            lib.cotten_host_cache_free(c)
        return rc

    alone = [torch.empty_like(t["q"]) for _ in range(4)]
    for w in range(W):
        assert call(w * per, alone) == 0
    for _ in range(3):
        got = [torch.full_like(t["q"], float("nan")) for _ in range(4)]
        rcs = [None] * W

        def worker(w):
            rcs[w] = call(w * per, got)
        ths = [threading.Thread(target=worker, args=(w,)) for w in range(W)]
        for th in ths:
            th.start()
        for th in ths:
            th.join(timeout=120)
        assert not any(th.is_alive() for th in ths)
        assert rcs == [0] * W
        for a, b in zip(alone, got):
            assert torch.equal(a, b)


def test_cached_backward_without_cache_is_usage_error():
    lib = _lib.load()
    rc = lib.cotten_bwd_host_cached(None, None, None, None, None, None, None)
    assert rc == _lib.COTTEN_ERR_USAGE
    assert b"missing cache" in lib.cotten_last_error()
