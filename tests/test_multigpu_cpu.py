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


def _bench_line(*argv):
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), *argv], cwd=root,
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]  # exactly one JSON line (rank 0)
    return json.loads(lines[0])


@pytest.mark.parametrize("workload,strong", [("ml20m", True), ("ml1m", False)])
def test_bench_launcher_spawns_ranks(workload, strong):
    """`bench.py --gpus 2` outside torchrun re-executes itself under
    torch.distributed.run with 2 ranks (gloo here): the line reports n_gpus 2,
    the right global batch and shards that tile the batch."""
    res = _bench_line("--gpus", "2", "--plan", "--workload", workload)
    total_b = bench.WORKLOADS[workload][0]
    assert res["n_gpus"] == 2
    assert res["config"]["global_batch"] == (total_b if strong else 2 * total_b)
    assert res["config"]["parallelism"].startswith("dp2")
    if strong:
        assert res["shards"] == [[0, total_b // 2], [total_b // 2, total_b]]
    else:
        assert res["shards"] == [[0, total_b], [0, total_b]]


@pytest.mark.skipif(not oracle.ref_available(release=True), reason="oracle/_ref not built")
def test_reference_arm_two_ranks_same_config():
    """The reference arm under the launcher: rank 0 alone runs and prints, with
    the config dict the GPU arm emits (workload_config)."""
    res = _bench_line("--gpus", "2", "--impl", "reference", "--steps", "1", "--warmup", "0",
                      "--workload", "beauty")
    assert res["impl"] == "reference" and res["n_gpus"] == 2
    assert res["config"] == bench.workload_config("beauty", 2)
    assert res["cpu_baseline"]["kind"] == "reference" and res["value"] > 0


@pytest.mark.skipif(not oracle.ref_available(release=True), reason="oracle/_ref not built")
def test_reference_arm_never_maps_the_product_library():
    """--impl reference must not import the product package: after a full
    reference-arm run, libcotten.so is absent from the process's mappings."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import sys, argparse; sys.argv=['bench.py']; import bench; "
            "a=argparse.Namespace(workload='beauty', steps=1, warmup=0); "
            "r=bench.run_reference(a, 1, 0); assert r['value'] > 0; "
            "maps=open('/proc/self/maps').read(); "
            "assert 'libcotten' not in maps, 'product library mapped'; "
            "assert 'paper_2602_06935_b200' not in sys.modules; print('clean')")
    r = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0 and "clean" in r.stdout, r.stderr[-2000:]
