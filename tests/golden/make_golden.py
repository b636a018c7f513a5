"""Generate tests/golden/cosine_golden.npz from the REFERENCE ITSELF.

Runs the unmodified reference operator (compiled from /root/reference by
oracle/Makefile into oracle/_ref/libcosrec_ref.so) on seeded float32-rounded
inputs and stores inputs + every output of
cosine_attention_fused(..., &cache, &mask) / cosine_attention_backward.
Run here (the GPU box has no /root/reference):

    make -C oracle && python tests/golden/make_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cosine_golden.npz")

# (name, n, d, m, eps, mask kind, seed)
CASES = [
    ("n1_d6", 1, 6, 0.7, 1e-12, "none", 7),
    ("n2_d2", 2, 2, 1.0, 1e-13, "none", 1),
    ("n5_d3_lead_pad", 5, 3, 1.0, 1e-9, "lead2", 2),
    ("n6_d3_masked_fd", 6, 3, 1.0, 1e-6, "lead2", 800),
    ("n7_d5_m0", 7, 5, 0.0, 1e-9, "none", 3),
    ("n9_d4_trail_pad", 9, 4, 1.25, 1e-6, "trail3", 4),
    ("n13_d16_random", 13, 16, 0.5, 1e-6, "random", 5),
    ("n33_d1", 33, 1, 1.5, 1e-6, "random", 6),
    ("n64_d8_single_valid", 64, 8, 1.0, 1e-6, "single", 8),
    ("n128_d16", 128, 16, 1.75, 1e-9, "left", 9),
    ("beauty_n50_d32", 50, 32, 1.0, 1e-6, "left", 42),
    ("ml1m_n200_d32", 200, 32, 1.0, 1e-6, "left", 0),
    ("ml1m_n200_d32_m075_allvalid", 200, 32, 0.75, 1e-6, "none", 123),
    ("n64_d64", 64, 64, 1.0, 1e-6, "random", 11),
    ("n24_d128", 24, 128, 1.0, 1e-6, "left", 12),
]


def mask_for(kind, n, rng):
    if kind == "none":
        return None
    v = np.zeros(n, np.uint8)
    if kind == "lead2":
        v[2:] = 1
    elif kind == "trail3":
        v[: n - 3] = 1
    elif kind == "left":
        L = int(rng.integers(1, n + 1))
        v[n - L:] = 1
    elif kind == "random":
        v = (rng.random(n) < 0.6).astype(np.uint8)
        v[int(rng.integers(0, n))] = 1
    elif kind == "single":
        v[int(rng.integers(0, n))] = 1
    return v


def main():
    store = {}
    for name, n, d, m, eps, kind, seed in CASES:
        rng = np.random.default_rng(seed)
        q, k, v, g = (rng.uniform(-1, 1, (n, d)).astype(np.float32) for _ in range(4))
        valid = mask_for(kind, n, rng)
        if valid is not None:  # junk (incl. NaN) in padded K rows must never be read
            k[valid == 0] = np.float32(np.nan)
        fw = oracle.ref_fwd(q, k, v, valid, m, eps)
        kk = k.copy()
        out, dq, dk, dv, dm = oracle.ref_fwd_bwd(q, kk, v, g, valid, m, eps)
        assert np.array_equal(out, fw["out"], equal_nan=True)
        p = name + "/"
        store[p + "q"], store[p + "k"], store[p + "v"], store[p + "d_out"] = q, k, v, g
        store[p + "valid"] = valid if valid is not None else np.ones(0, np.uint8)
        store[p + "meta"] = np.array([n, d, m, eps], np.float64)
        for key in ("out", "norm_q", "norm_k", "qn", "kn", "S"):
            store[p + key] = fw[key]
        store[p + "true_n"] = np.array([fw["true_n"]], np.int64)
        store[p + "dq"], store[p + "dk"], store[p + "dv"] = dq, dk, dv
        store[p + "dm"] = np.array([dm])
    np.savez_compressed(OUT, **store)
    print(f"wrote {OUT}: {len(CASES)} cases, {os.path.getsize(OUT)} bytes")


if __name__ == "__main__":
    main()
