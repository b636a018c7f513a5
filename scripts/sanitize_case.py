"""One small multi-unit fwd+bwd of a chosen kernel path, for compute-sanitizer
(memcheck / racecheck / synccheck): python scripts/sanitize_case.py <path>
with path in tc | tclong | tcf64 | tcflong | tcfmerge | tcb64 | tcbpair |
tcblong | tch | tchlong | tcg | tcglong | d32 | rt64 | rt128 | rtbf16 | generic.  Exits non-zero on a
parity failure vs the oracle (so a sanitizer run also checks the values)."""
import sys

import numpy as np

sys.path.insert(0, ".")
import oracle  # noqa: E402
import torch  # noqa: E402
from paper_2602_06935_b200 import _lib, inputs, ops  # noqa: E402

path = sys.argv[1]
FP = _lib.FLAG_FP32_PIPE
B, H, N, D, dt, flags = {
    "tc": (160, 2, 200, 32, torch.float32, 0),        # 320 units on 148 CTAs, 2 chunks/unit
    "tclong": (2, 2, 700, 32, torch.float32, 0),      # 6 chunks, flush of the running sum
    "tcf64": (160, 2, 300, 64, torch.float32, 0),     # fp32 d_h 64 three-part kernels, 5 chunks/unit
    "tcflong": (2, 2, 700, 64, torch.float32, 0),     # 11 chunks, flush every 8
    "tcfmerge": (320, 2, 50, 32, torch.float32, 0),   # head pairs merged, 320 pairs on 148 CTAs
    "tcb64": (160, 2, 300, 64, torch.bfloat16, 0),    # bf16 d_h 64
    "tcbpair": (160, 2, 300, 32, torch.bfloat16, 0),  # bf16 d_h 32 as paired rows
    "tcblong": (2, 2, 1100, 64, torch.bfloat16, 0),   # 9 chunks, flush every 4
    "d32": (160, 2, 50, 32, torch.float32, FP),
    "rt64": (20, 2, 300, 64, torch.float32, FP),
    "rt128": (8, 2, 300, 128, torch.float32, FP),
    "tch": (160, 2, 300, 128, torch.bfloat16, 0),     # bf16 d_h 128, 5 chunks/unit, >= 2 units/CTA
    "tchlong": (2, 2, 700, 128, torch.bfloat16, 0),   # 11 chunks, TMEM running-sum flush
    "tcg": (160, 2, 300, 128, torch.float32, 0),      # fp32 d_h 128, 10 items/pass, >= 2 units/CTA
    "tcglong": (2, 2, 700, 128, torch.float32, 0),    # 22 items, TMEM running-sum flush
    "tchsmall": (2, 2, 200, 128, torch.bfloat16, 0),  # racecheck-sized
    "tcgsmall": (2, 2, 200, 128, torch.float32, 0),
    "rtbf16": (20, 2, 301, 32, torch.bfloat16, 0),    # odd N: register-tiled
    "generic": (6, 2, 70, 24, torch.float32, 0),
}[path]
h = inputs.make_host(B, H, N, D, seed=1)
valid = inputs.left_padded_mask(B, N, 1)
t = {n: torch.from_numpy(x).cuda().to(dt) for n, x in h.items()}
vm = torch.from_numpy(valid).cuda()
S = torch.empty(B * H, D, D, device="cuda")
out = ops.forward(t["q"], t["k"], t["v"], vm, 1.0, saved_S=S, flags=flags)
dmt = torch.empty(1, dtype=torch.float64, device="cuda")
dq, dk, dv = ops.backward(t["q"], t["k"], t["v"], vm, 1.0, t["d_out"], S, dm_total=dmt, flags=flags)
torch.cuda.synchronize()
x = {n: v.float().cpu().numpy() for n, v in t.items()}
ref = oracle.batched_f32(x["q"], x["k"], x["v"], x["d_out"], valid, 1.0, 1e-6)
tol = 1e-2 if dt == torch.bfloat16 else 1e-5
for name, got, want in zip(("out", "dq", "dk", "dv"), (out, dq, dk, dv), ref[:4]):
    g = got.double().cpu().numpy().reshape(B * H, -1)
    w = want.reshape(B * H, -1)
    err = float((np.abs(g - w).max(1) / np.abs(w).max(1)).max())
    assert err <= tol, (path, name, err)
print(f"sanitize_case {path}: B={B} H={H} N={N} D={D} parity ok")
