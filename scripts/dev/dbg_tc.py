"""Bring-up probe for the tcgen05 kernels: one tiny unit, prints S / O / grads vs numpy."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2602_06935_b200 import ops, _lib

torch.manual_seed(0)
B, H, N, D = int(sys.argv[1]) if len(sys.argv) > 1 else 1, 1, int(sys.argv[2]) if len(sys.argv) > 2 else 128, 32
q, k, v, g = (torch.rand(B, H, N, D, device="cuda") * 2 - 1 for _ in range(4))
eps = 1e-6
def ref(q, k, v, g):
    q, k, v, g = (x.double().cpu().numpy() for x in (q, k, v, g))
    qn = q / np.sqrt((q * q).sum(-1, keepdims=True) + eps)
    kn = k / np.sqrt((k * k).sum(-1, keepdims=True) + eps)
    S = np.einsum("bhna,bhnc->bhac", kn, v)
    s = N ** -1.0
    O = s * np.einsum("bhna,bhac->bhnc", qn, S)
    G = np.einsum("bhna,bhnc->bhac", qn, g)
    return S, O, G
S_ref, O_ref, G_ref = ref(q, k, v, g)
for flags in (_lib.FLAG_FP32_PIPE, 0):
    S = torch.zeros(B * H, D, D, device="cuda")
    out = torch.zeros_like(q)
    ops.forward(q, k, v, None, 1.0, eps, out=out, saved_S=S, flags=flags)
    torch.cuda.synchronize()
    Sg = S.double().cpu().numpy().reshape(B, H, D, D)
    Og = out.double().cpu().numpy()
    print("flags", flags)
    print("  S err", np.abs(Sg - S_ref).max(), "S max", np.abs(S_ref).max(), "S got max", np.abs(Sg).max())
    print("  O err", np.abs(Og - O_ref).max(), "O max", np.abs(O_ref).max(), "O got max", np.abs(Og).max())
    print("  S[0,0,:4,:4] got\n", Sg[0, 0, :4, :4], "\n  ref\n", S_ref[0, 0, :4, :4])
    print("  O[0,0,:3,:6] got\n", Og[0, 0, :3, :6], "\n  ref\n", O_ref[0, 0, :3, :6])
    dq, dk, dv = ops.backward(q, k, v, None, 1.0, g, S, eps=eps, flags=flags)
    torch.cuda.synchronize()
    if flags == _lib.FLAG_FP32_PIPE:
        base = [x.double().cpu().numpy() for x in (dq, dk, dv)]
    else:
        for n, x, y in zip(("dq", "dk", "dv"), (dq, dk, dv), base):
            x = x.double().cpu().numpy()
            print("  ", n, "err vs fp32pipe", np.abs(x - y).max(), "max", np.abs(y).max(), "got max", np.abs(x).max())
            print("     got", x[0, 0, 0, :5], "\n     ref", y[0, 0, 0, :5])
