"""Synthetic inputs for the cosine-attention path.

Seeding follows the reference bench recipe: a stream seed
``mix_seed(seed, N, D)`` (rng.hpp:9-21, bench.cpp:50) and U(-1, 1) values
(bench.cpp:21-26).  The stream itself is numpy's PCG64 (host) or torch's
Philox (device) instead of std::mt19937_64, so the values differ from the
reference bench's while keeping its distribution and per-shape seeding.
Masks are left-padded like data.cpp:193-199: sequence b keeps its last L_b
rows, L_b ~ U{1..N}.
"""
from __future__ import annotations

import numpy as np

_M64 = (1 << 64) - 1


def splitmix64(x: int) -> int:
    """rng.hpp:9-14"""
    x = (x + 0x9E3779B97F4A7C15) & _M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _M64
    return x ^ (x >> 31)


def mix_seed(a: int, b: int, c: int = 0) -> int:
    """rng.hpp:19-21"""
    return splitmix64(splitmix64(splitmix64(a) ^ b) ^ c)


def lengths(B: int, N: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(mix_seed(seed, N, 0xA5A5))
    return rng.integers(1, N + 1, size=B)


def left_padded_mask(B: int, N: int, seed: int) -> np.ndarray:
    """uint8 [B, N]: valid[b, i] = i >= N - L_b (data.cpp:193-199)."""
    L = lengths(B, N, seed)
    return (np.arange(N)[None, :] >= (N - L)[:, None]).astype(np.uint8)


def random_mask(B: int, N: int, seed: int, p: float = 0.5) -> np.ndarray:
    """Arbitrary valid patterns (the op allows any), at least one valid row."""
    rng = np.random.default_rng(mix_seed(seed, N, 0x5A5A))
    m = (rng.random((B, N)) < p).astype(np.uint8)
    m[np.arange(B), rng.integers(0, N, size=B)] = 1
    return m


def make_host(B, H, N, D, seed=0, with_grad=True, dtype=np.float32):
    """Q, K, V (and dO) as [B, H, N, D] U(-1,1) arrays."""
    rng = np.random.default_rng(mix_seed(seed, N, D))
    names = ("q", "k", "v", "d_out") if with_grad else ("q", "k", "v")
    return {n: rng.uniform(-1.0, 1.0, size=(B, H, N, D)).astype(dtype) for n in names}


def make_device(B, H, N, D, seed=0, with_grad=True, dtype=None, device="cuda"):
    """Same distribution generated on the device (torch Philox), for sizes
    where host generation would dominate (ML-20M: 3.4 GB per tensor)."""
    import torch
    dtype = torch.float32 if dtype is None else dtype
    g = torch.Generator(device=device)
    g.manual_seed(mix_seed(seed, N, D) & ((1 << 63) - 1))
    names = ("q", "k", "v", "d_out") if with_grad else ("q", "k", "v")
    out = {}
    for n in names:
        t = torch.empty((B, H, N, D), dtype=torch.float32, device=device)
        t.uniform_(-1.0, 1.0, generator=g)
        out[n] = t.to(dtype) if dtype != torch.float32 else t
    return out
