"""Normwise error of each d_h=32 path vs the float64 oracle, per N (diagnostic)."""
import sys
import numpy as np
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from test_gpu_parity import run_gpu, oracle_for, normwise  # noqa: E402
from paper_2602_06935_b200 import _lib, inputs  # noqa: E402

for N in (1, 2, 50, 65, 128, 200, 256, 513, 2048, 4096, 16384):
    B, H, D = 8, 2, 32
    h = inputs.make_host(B, H, N, D, seed=N)
    valid = inputs.left_padded_mask(B, N, N)
    line = [f"N={N:5d}"]
    for name, flags in (("tc", 0), ("fp32", _lib.FLAG_FP32_PIPE)):
        res = run_gpu(h, valid, 0.75, 1e-6, "f32", flags)
        ref = oracle_for(res["inputs"], valid, 0.75, 1e-6)
        errs = [normwise(res[k], w) for k, w in zip(("out", "dq", "dk", "dv"), ref[:4])]
        dm = np.abs(res["dm_unit"] - ref[4]).max() / np.abs(ref[4]).max()
        line.append(f"{name}: " + " ".join(f"{e:.1e}" for e in errs + [dm]))
    print("  ".join(line), flush=True)
