"""GPU tests of the C-ABI's edge contracts: host entry points on dense layouts
whose batch is not the outermost dimension, outputs allocated for a gapped
(fused-projection) q, and per-stream workspaces (two streams of one host
thread, both asking for the in-kernel dm total)."""
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
