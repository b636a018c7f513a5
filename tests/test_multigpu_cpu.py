"""The N>1 path on CPU (gloo, world_size 2): bench.py's contiguous batch
sharding covers every sequence exactly once with no data-path collective, and
the one real exchange of the training step — the all-reduce of the learnable
exponent's gradient dm (summed over heads, attention.cpp:555, and sequences,
encoder.cpp:375) — reproduces the single-process total."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bench
import oracle
from paper_2602_06935_b200 import inputs


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, B, H, N, D, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = bench.shard(B, rank, world)
    h = inputs.make_host(B, H, N, D, seed=3)
    valid = inputs.left_padded_mask(B, N, 3)
    sl = slice(lo, hi)
    _, _, _, _, dm_unit = oracle.batched_f32(h["q"][sl], h["k"][sl], h["v"][sl], h["d_out"][sl],
                                             valid[sl], 1.0, 1e-6)
    dm = torch.tensor([dm_unit.sum()], dtype=torch.float64)
    dist.all_reduce(dm)  # the only collective: dm (and, in training, weight gradients)
    cover = torch.zeros(B, dtype=torch.int64)
    cover[lo:hi] = 1
    dist.all_reduce(cover)
    if rank == 0:
        out.put((float(dm.item()), cover.numpy().tolist()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("B", [7, 16])
def test_sharded_dm_allreduce_matches_single_process(B):
    H, N, D = 2, 20, 8
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, B, H, N, D, q)) for r in range(2)]
    for p in procs:
        p.start()
    dm_total, cover = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    h = inputs.make_host(B, H, N, D, seed=3)
    valid = inputs.left_padded_mask(B, N, 3)
    full = oracle.batched_f32(h["q"], h["k"], h["v"], h["d_out"], valid, 1.0, 1e-6)[4].sum()
    assert cover == [1] * B
    assert dm_total == pytest.approx(full, rel=1e-12, abs=1e-12)


@pytest.mark.parametrize("total,world", [(65536, 8), (65536, 3), (256, 2), (5, 8)])
def test_shard_partition(total, world):
    spans = [bench.shard(total, r, world) for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == total
    for (a, b), (c, d) in zip(spans, spans[1:]):
        assert b == c and b >= a
    sizes = [b - a for a, b in spans]
    assert max(sizes) - min(sizes) <= 1
