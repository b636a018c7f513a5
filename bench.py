#!/usr/bin/env python
"""Benchmark of the cosine-attention hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload ml1m|beauty|ml20m]

A step is one training pass of the op over one batch: for BASELINE config #2
(the default "ml1m" workload: 2 Cotten layers, B=256, N=200, model d=64 with
H=2 heads, so d_h=32, fp32, left-padded mask) that is the forward of layer 0
and 1, then the backward of layer 1 and 0 (each layer has its own Q/K/V/dO),
plus, at N>1, the NCCL all-reduce of the learnable-exponent gradients dm (the
op's only parameter gradient).  Per-GPU batch is fixed (weak scaling) except
for ml20m, whose 65536-sequence batch is split across ranks (strong).

Timing: W untimed warm-up steps, then exactly K steps; every step is bracketed
by CUDA events on the launching stream, L2 is flushed (256 MiB write) between
steps outside the events, barrier + synchronize on both sides, max over ranks.
`value` = sequences/s of the whole job; `e2e` = the same metric through the
reference-facing host entry points (cotten_fwd_host / cotten_bwd_host) with
pinned host buffers, copies inside the timed region; `roofline` = the
dominant kernel's algorithmic bytes per launch over its average event time.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "cosine-attn fwd+bwd seqs/sec @N=200,d=64; % of HBM roofline; vs CPU ref"
WORKLOADS = {
    # name: (per-GPU batch or total batch, N, H, d_h, layers, strong_scaling, description)
    "ml1m": (256, 200, 2, 32, 2, False,
             "BASELINE config #2 at op level: 2 Cotten layers x cosine-attn fwd+bwd, ML-1M shape "
             "(B=256, N=200, d=64 -> H=2 x d_h=32), fp32, left-padded mask"),
    "beauty": (8192, 50, 2, 32, 1, False,
               "BASELINE config #3: cosine-attn fwd+bwd, Beauty/Steam shape (B=8192, N=50, H=2, "
               "d_h=32), fp32, left-padded mask"),
    "ml20m": (65536, 200, 2, 32, 1, True,
              "BASELINE config #4: cosine-attn fwd+bwd, ML-20M shape (B=65536 split across GPUs, "
              "N=200, H=2, d_h=32), fp32, left-padded mask"),
    # BASELINE config #5 (long-sequence sweep) points; ~0.5-1 G rows of work each
    "long4k": (1024, 4096, 2, 32, 1, True,
               "BASELINE config #5 point: cosine-attn fwd+bwd, N=4096, H=2, d_h=32, B=1024, fp32, "
               "left-padded mask"),
    "long16k": (256, 16384, 2, 32, 1, True,
                "BASELINE config #5 point: cosine-attn fwd+bwd, N=16384, H=2, d_h=32, B=256, fp32, "
                "left-padded mask"),
    "long4k_d64": (512, 4096, 1, 64, 1, True,
                   "BASELINE config #5 point: cosine-attn fwd+bwd, N=4096, H=1, d_h=64, B=512, fp32 "
                   "(register-tiled FP32-pipe kernels), left-padded mask"),
    "long4k_d128": (256, 4096, 1, 128, 1, True,
                    "BASELINE config #5 point: cosine-attn fwd+bwd, N=4096, H=1, d_h=128, B=256, fp32 "
                    "(register-tiled FP32-pipe kernels), left-padded mask"),
}
# bf16 in HBM (fp32 arithmetic) points of config #5: the same shapes, half the bytes
for _name in ("long4k", "long4k_d64", "long4k_d128"):
    _w = WORKLOADS[_name]
    WORKLOADS[_name + "_bf16"] = _w[:6] + (_w[6].replace("fp32", "bf16 in HBM (fp32 arithmetic)"),)
WORKLOAD_DTYPE = {n: "bf16" for n in WORKLOADS if n.endswith("_bf16")}
L2_FLUSH_BYTES = 256 << 20


def algorithmic_bytes(B, H, N, D, elt=4):
    """fwd reads Q,K,V and writes O (4·N·D·s per unit) + N mask
    bytes per sequence; bwd reads Q,K,V,dO and writes dQ,dK,dV (7·N·D·s) + mask."""
    fwd = B * H * 4 * N * D * elt + B * N
    bwd = B * H * 7 * N * D * elt + B * N
    return fwd, bwd


FP32_PEAK_FLOPS = 148 * 128 * 2 * 1.965e9


def pipe_flops(B, H, N, D):
    """SURVEY §8d flops per launch: fwd 4·N·d² + 7·N·d, bwd 8·N·d² + 12·N·d per unit."""
    return B * H * (4 * N * D * D + 7 * N * D), B * H * (8 * N * D * D + 12 * N * D)


def kernel_path(path, N, D, dname="f32"):
    """The kernels the library picks for this shape (cotten_capi.cu launch_*_t)."""
    if dname == "bf16" and D == 32:
        return "fp32-rt register-tiled FP32 pipe (kernels_rt.cuh)"
    if D == 32 and path == "tcgen05" and N > 64:
        return "tcgen05 (kernels_tc.cuh)"
    if D == 32:
        return "fp32pipe (kernels_d32.cuh)"
    if D in (64, 128):
        return "fp32-rt register-tiled FP32 pipe (kernels_rt.cuh)"
    return "generic (kernels_generic.cuh)"


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled while the timed region runs."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q,
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.thread is not None:
            self.thread.join(timeout=5)
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if r[3 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def dist_setup(want_gpus):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if torch.cuda.is_available():
            torch.cuda.set_device(local)
        dist.init_process_group("nccl" if torch.cuda.is_available() else "gloo")
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return world, rank, local


def shard(total, rank, world):
    """Contiguous batch shard [lo, hi) of rank: no collective."""
    per, rem = divmod(total, world)
    lo = rank * per + min(rank, rem)
    return lo, lo + per + (1 if rank < rem else 0)


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


# ---------------------------------------------------------------------------

def run_ours(args, world, rank, local):
    import torch
    from paper_2602_06935_b200 import _lib, inputs, ops

    total_b, N, H, D, layers, strong, desc = WORKLOADS[args.workload]
    dname = WORKLOAD_DTYPE.get(args.workload, "f32")
    tdtype = torch.bfloat16 if dname == "bf16" else torch.float32
    lo, hi = shard(total_b, rank, world) if strong else (0, total_b)
    B = hi - lo
    global_b = total_b if strong else total_b * world
    dev = torch.device("cuda", torch.cuda.current_device())
    stream = torch.cuda.current_stream()

    # Inputs resident in HBM before the timed region (distinct per layer / rank).
    L = []
    for layer in range(layers):
        t = inputs.make_device(B, H, N, D, seed=1000 * layer + rank, dtype=tdtype, device=dev)
        valid = torch.from_numpy(inputs.left_padded_mask(B, N, 1000 * layer + rank)).to(dev)
        t.update(valid=valid,
                 out=torch.empty_like(t["q"]), S=torch.empty(B * H, D, D, device=dev),
                 dq=torch.empty_like(t["q"]), dk=torch.empty_like(t["q"]),
                 dv=torch.empty_like(t["q"]),
                 dm_unit=torch.empty(B * H, dtype=torch.float64, device=dev))
        L.append(t)
    dm_tot = torch.zeros(layers, dtype=torch.float64, device=dev)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    m = 1.0
    flags = _lib.FLAG_FP32_PIPE if args.path == "fp32pipe" else 0

    launches = [0]

    def fwd(t):
        ops.forward(t["q"], t["k"], t["v"], t["valid"], m, out=t["out"], saved_S=t["S"],
                    stream=stream, flags=flags)
        launches[0] += _lib.launches()

    def bwd(t, i):
        ops.backward(t["q"], t["k"], t["v"], t["valid"], m, t["d_out"], t["S"], t["dq"],
                     t["dk"], t["dv"], t["dm_unit"], dm_tot[i:i + 1], stream=stream, flags=flags)
        launches[0] += _lib.launches()

    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    n_marks = 2 * layers + 1
    args.no_graph = args.graph == "off"

    def step(marks=None):
        if marks is not None:
            marks[0].record(stream)
        for i in range(layers):
            fwd(L[i])
            if marks is not None:
                marks[1 + i].record(stream)
        for j, i in enumerate(reversed(range(layers))):
            bwd(L[i], i)
            if marks is not None:
                marks[1 + layers + j].record(stream)
        if world > 1:  # the op's parameter-gradient exchange (dm per layer)
            import torch.distributed as dist
            dist.all_reduce(dm_tot)

    for _ in range(max(args.warmup, 3) if args.warmup >= 0 else 3):
        step()
    torch.cuda.synchronize()
    # graphs only where host launch overhead paces the step (short steps); long
    # steps measured ~4 % faster issued eagerly (ML-20M), so they stay eager
    w0, w1 = ev(), ev()
    w0.record(stream)
    step()
    w1.record(stream)
    torch.cuda.synchronize()
    eager_step_ms = w0.elapsed_time(w1)
    if args.graph == "on" or (args.graph == "auto" and eager_step_ms < 2.0):
        args.no_graph = False
    else:
        args.no_graph = True

    if not args.no_graph:
        # One CUDA graph per op call (the tensor maps, scale constants and
        # launch geometry are baked in at capture): a replay is a single
        # cudaGraphLaunch, so the host no longer paces small batches.  Warm-up
        # above already allocated every workspace the calls need.
        graphs = {}
        counts = {}
        cap = torch.cuda.Stream()
        cap.wait_stream(stream)
        for i in range(layers):
            for kind in ("fwd", "bwd"):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=cap):
                    s_cap = torch.cuda.current_stream()
                    if kind == "fwd":
                        ops.forward(L[i]["q"], L[i]["k"], L[i]["v"], L[i]["valid"], m,
                                    out=L[i]["out"], saved_S=L[i]["S"], stream=s_cap, flags=flags)
                    else:
                        t = L[i]
                        ops.backward(t["q"], t["k"], t["v"], t["valid"], m, t["d_out"], t["S"],
                                     t["dq"], t["dk"], t["dv"], t["dm_unit"], dm_tot[i:i + 1],
                                     stream=s_cap, flags=flags)
                    counts[(kind, i)] = _lib.launches()
                graphs[(kind, i)] = g
        stream.wait_stream(cap)
        torch.cuda.synchronize()

        fwd_eager, bwd_eager = fwd, bwd

        def fwd(t, _i=None):  # noqa: F811
            i = next(k for k in range(layers) if L[k] is t)
            graphs[("fwd", i)].replay()
            launches[0] += counts[("fwd", i)]

        def bwd(t, i):  # noqa: F811
            graphs[("bwd", i)].replay()
            launches[0] += counts[("bwd", i)]

        step_launches = sum(counts.values())
        # The whole step as one graph too: inside a graph the kernels'
        # programmatic-dependent-launch attribute becomes a programmatic edge,
        # so each kernel's prologue overlaps the previous kernel's tail, which
        # separate graph launches cannot do.
        gstep = None
        if args.graph_scope == "step":
            gstep = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gstep, stream=cap):
                s_cap = torch.cuda.current_stream()
                for i in range(layers):
                    t = L[i]
                    ops.forward(t["q"], t["k"], t["v"], t["valid"], m, out=t["out"], saved_S=t["S"],
                                stream=s_cap, flags=flags)
                for i in reversed(range(layers)):
                    t = L[i]
                    ops.backward(t["q"], t["k"], t["v"], t["valid"], m, t["d_out"], t["S"], t["dq"],
                                 t["dk"], t["dv"], t["dm_unit"], dm_tot[i:i + 1], stream=s_cap,
                                 flags=flags)
        stream.wait_stream(cap)
        torch.cuda.synchronize()
        for _ in range(2):
            step()
        torch.cuda.synchronize()

    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.25)
    all_marks = [[ev() for _ in range(n_marks)] for _ in range(args.steps)]
    if not args.no_graph:
        # per-op kernel times (roofline fields) from a separately marked pass
        for s_ in range(args.steps):
            flush.zero_()
            step(all_marks[s_])
        torch.cuda.synchronize()
        step_marks = [(ev(), ev()) for _ in range(args.steps)]
    barrier(world)
    torch.cuda.synchronize()
    launches[0] = 0
    for s_ in range(args.steps):
        flush.zero_()  # L2 flush between timed steps, outside the events
        if args.no_graph:
            step(all_marks[s_])
        else:
            # the step's per-op graphs back to back, events at the step boundaries only
            step_marks[s_][0].record(stream)
            if gstep is not None:
                gstep.replay()
            else:
                for i in range(layers):
                    graphs[("fwd", i)].replay()
                for i in reversed(range(layers)):
                    graphs[("bwd", i)].replay()
            launches[0] += step_launches
            if world > 1:
                import torch.distributed as dist
                dist.all_reduce(dm_tot)
            step_marks[s_][1].record(stream)
    torch.cuda.synchronize()
    barrier(world)
    gpu_launches = launches[0]
    graph_check = None
    if not args.no_graph:
        # the graphs' outputs of the last timed step == a plain eager step's (same inputs)
        names = ("out", "dq", "dk", "dv")
        snap = [L[i][n].clone() for i in range(layers) for n in names]
        snap_dm = dm_tot.clone()
        for i in range(layers):
            fwd_eager(L[i])
        for i in reversed(range(layers)):
            bwd_eager(L[i], i)
        torch.cuda.synchronize()
        graph_check = all(torch.equal(a, L[i][n]) for a, (i, n) in
                          zip(snap, [(i, n) for i in range(layers) for n in names]))
        graph_check = bool(graph_check and (world > 1 or torch.equal(snap_dm, dm_tot)))
    # keep the GPU busy a little longer so the sampler sees the load
    extra_t0 = time.time()
    while time.time() - extra_t0 < 1.0:
        flush.zero_()
        step()
    torch.cuda.synchronize()
    clocks = sampler.stop()

    if args.no_graph:
        step_ms = [m_[0].elapsed_time(m_[-1]) for m_ in all_marks]
    else:
        step_ms = [a.elapsed_time(b) for a, b in step_marks]
    fwd_ms = [m_[i].elapsed_time(m_[i + 1]) for m_ in all_marks for i in range(layers)]
    bwd_ms = [m_[layers + i].elapsed_time(m_[layers + i + 1]) for m_ in all_marks
              for i in range(layers)]
    total_ms = max_over_ranks(sum(step_ms), world)
    ms_per_step = total_ms / args.steps
    value = global_b * args.steps / (total_ms / 1e3)

    fwd_bytes, bwd_bytes = algorithmic_bytes(B, H, N, D, elt=2 if dname == "bf16" else 4)
    peak, peak_src = load_peaks()
    fwd_avg = statistics.mean(fwd_ms) / 1e3
    bwd_avg = statistics.mean(bwd_ms) / 1e3
    bwd_gbs = bwd_bytes / bwd_avg / 1e9
    fwd_gbs = fwd_bytes / fwd_avg / 1e9
    step_gbs = layers * (fwd_bytes + bwd_bytes) / (ms_per_step / 1e3) / 1e9

    res = {
        "metric": METRIC, "value": value, "unit": "seq/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong" if strong else "weak", "vs_baseline": None, "dtype": dname,
        "data": "synthetic U(-1,1) (mix_seed per shape, bench.cpp:21-26,50), left-padded masks",
        "config": {"workload": desc, "name": args.workload, "global_batch": global_b,
                   "batch_per_gpu": B, "seq_len": N, "heads": H, "head_dim": D, "model_dim": H * D,
                   "layers": layers, "parallelism": f"dp{world} (batch x head shards)",
                   "kernel_path": kernel_path(args.path, N, D, dname),
                   "launch": "eager" if args.no_graph else (
                       ("one CUDA graph per step (the 2 x layers op calls; programmatic-dependent-launch "
                        "edges between the kernels)" if args.graph_scope == "step" else
                        "one CUDA graph per op call, replayed back to back")
                       + " (events at step boundaries); per-op kernel times from a separately marked "
                         "pass of per-op graphs"),
                   "l2": "flushed between timed steps (256 MiB write), outside the events"},
        "roofline": {"bound": "hbm", "kernel": "cos_bwd (backward, dominant)",
                     "achieved": bwd_gbs, "peak": peak, "unit": "GB/s", "frac": bwd_gbs / peak,
                     "traffic": None, "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": bwd_bytes,
                     "avg_launch_us": bwd_avg * 1e6},
        "kernels": {"fwd_us": fwd_avg * 1e6, "fwd_GBps": fwd_gbs, "fwd_frac": fwd_gbs / peak,
                    "bwd_us": bwd_avg * 1e6, "bwd_GBps": bwd_gbs, "bwd_frac": bwd_gbs / peak,
                    "step_GBps": step_gbs, "step_frac": step_gbs / peak},
        "gpu_launches": gpu_launches,
        "graph_outputs_equal_eager": graph_check,
        "clocks": clocks,
    }
    if D != 32 or dname == "bf16":  # FP32-pipe kernels: compute at peak bounds them, not HBM (north star: max of both)
        ff, fb = pipe_flops(B, H, N, D)
        t_f = max(ff / FP32_PEAK_FLOPS, fwd_bytes / (peak * 1e9))
        t_b = max(fb / FP32_PEAK_FLOPS, bwd_bytes / (peak * 1e9))
        res["roofline_max"] = {
            "model": "max(compute-at-peak, bytes-at-HBM) per launch; FP32 pipe peak = 148 SM x 128 FFMA "
                     "x 2 x 1.965 GHz (derived, no measured FP32 peak in MEASURED_PEAKS.json)",
            "pipe": "fp32", "peak_tflops": FP32_PEAK_FLOPS / 1e12,
            "fwd_bound": "fp32" if ff / FP32_PEAK_FLOPS > fwd_bytes / (peak * 1e9) else "hbm",
            "bwd_bound": "fp32" if fb / FP32_PEAK_FLOPS > bwd_bytes / (peak * 1e9) else "hbm",
            "fwd_tflops": ff / fwd_avg / 1e12, "bwd_tflops": fb / bwd_avg / 1e12,
            "fwd_frac": t_f / fwd_avg, "bwd_frac": t_b / bwd_avg,
            "step_frac": layers * (t_f + t_b) / (ms_per_step / 1e3)}
    traffic = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(traffic):
        try:
            with open(traffic) as f:
                tr = json.load(f).get(args.workload)
            if tr:
                res["roofline"]["traffic"] = tr.get("bwd")
                res["roofline"]["traffic_source"] = "profiles/traffic.json (ncu, per launch)"
        except Exception:
            pass

    if not args.no_e2e and dname == "bf16":
        res["e2e"] = {"value": None, "note": "bf16 points are device-resident kernel measurements only"}
    elif not args.no_e2e:
        res["e2e"] = run_e2e(args, world, B, N, H, D, layers, global_b)
    if rank == 0 and world == 1 and not args.no_cpu and dname == "f32":
        res["cpu_baseline"] = run_cpu_baseline(args, N, H, D, layers, B)
    return res


def run_e2e(args, world, B, N, H, D, layers, global_b):
    """Same metric through the reference-facing host entry points
    (cotten_fwd_host / cotten_bwd_host: the calls under cosine_attention_fused /
    cosine_attention_backward), pinned host buffers, copies inside the timing."""
    import torch
    from paper_2602_06935_b200 import inputs
    from paper_2602_06935_b200 import _lib
    import ctypes

    lib = _lib.load()
    desc = _lib.make_desc(B, H, N, D, "f32", 1e-6)
    p = lambda a: ctypes.c_void_p(a.ctypes.data)  # noqa: E731

    def pinned(shape, dtype=torch.float32):
        return torch.empty(shape, dtype=dtype, pin_memory=True).numpy()

    Ls = []
    for layer in range(layers):
        h = inputs.make_host(B, H, N, D, seed=7 + layer)
        t = {}
        for n, x in h.items():
            t[n] = pinned(x.shape)
            t[n][...] = x
        t["valid"] = pinned((B, N), torch.uint8)
        t["valid"][...] = inputs.left_padded_mask(B, N, 7 + layer)
        for n in ("out", "dq", "dk", "dv"):
            t[n] = pinned((B, H, N, D))
        t["S"] = pinned((B * H, D, D))
        t["dm"] = pinned((1,), torch.float64)
        Ls.append(t)

    def step():
        for t in Ls:
            _lib.check(lib.cotten_fwd_host(ctypes.byref(desc), p(t["q"]), p(t["k"]), p(t["v"]),
                                           p(t["valid"]), 1.0, p(t["out"]), p(t["S"]), None))
        for t in reversed(Ls):
            _lib.check(lib.cotten_bwd_host(ctypes.byref(desc), p(t["q"]), p(t["k"]), p(t["v"]),
                                           p(t["valid"]), 1.0, p(t["d_out"]), p(t["S"]),
                                           p(t["dq"]), p(t["dk"]), p(t["dv"]), None, p(t["dm"])))

    for _ in range(max(args.warmup, 3)):
        step()
    barrier(world)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    el = max_over_ranks(time.perf_counter() - t0, world)
    tb = B * H * N * D * 4
    h2d = layers * (3 * tb + B * N) + layers * (4 * tb + B * N + B * H * D * D * 4)
    d2h = layers * (tb + B * H * D * D * 4) + layers * (3 * tb + 8)
    return {"value": global_b * args.steps / el, "unit": "seq/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h,
            "path": "cotten_fwd_host + cotten_bwd_host per layer (pinned host buffers)"}


def run_cpu_baseline(args, N, H, D, layers, B, budget_s=None):
    """The reference operator (oracle/_ref, compiled from /root/reference
    sources) on this host's cores: the same per-layer fwd(+cache)+bwd calls
    per (seq, head) on a persistent pool, on the same shape."""
    import oracle
    from paper_2602_06935_b200 import inputs
    budget_s = args.cpu_seconds if budget_s is None else budget_s
    threads = os.cpu_count() or 1
    if not oracle.ref_available():
        return {"value": None, "unit": "seq/s", "cores": threads, "kind": "reference",
                "sample": "unavailable: oracle/_ref/libcosrec_ref.so not built"}
    Bs = min(B, 256)
    per_layer = []
    for layer in range(layers):
        h = inputs.make_host(Bs, H, N, D, seed=7 + layer)
        valid = inputs.left_padded_mask(Bs, N, 7 + layer)
        outs = tuple(np.empty(h["q"].shape, np.float32) for _ in range(4)) + (np.zeros(Bs * H),)
        per_layer.append((h, valid, outs))

    def one():
        for h, valid, outs in per_layer:
            oracle.ref_batched_f32(h["q"], h["k"], h["v"], h["d_out"], valid, 1.0, 1e-6,
                                   threads, outs)

    one()  # warm-up (pool spawn, first touch)
    times = []
    t_start = time.perf_counter()
    while time.perf_counter() - t_start < budget_s or len(times) < 3:
        t0 = time.perf_counter()
        one()
        times.append(time.perf_counter() - t0)
    med = statistics.median(times)
    cpu = ""
    try:
        with open("/proc/cpuinfo") as f:
            cpu = next(l.split(":", 1)[1].strip() for l in f if l.startswith("model name"))
    except Exception:
        pass
    return {"value": Bs / med, "unit": "seq/s", "cores": threads, "kind": "reference",
            "sample": f"{Bs} sequences x {layers} layer(s) of cosine_attention_fused(+cache,+mask)"
                      f" + cosine_attention_backward per (seq, head), median of {len(times)} reps"
                      f" over {time.perf_counter() - t_start:.1f}s, {threads} threads, {cpu}"}


def run_reference(args, world, rank):
    """--impl reference: the reference's own CPU operator on this host."""
    if rank != 0:
        return None
    total_b, N, H, D, layers, strong, desc = WORKLOADS[args.workload]
    import oracle
    from paper_2602_06935_b200 import inputs
    threads = os.cpu_count() or 1
    Bs = min(total_b, 256)
    data = []
    for layer in range(layers):
        h = inputs.make_host(Bs, H, N, D, seed=7 + layer)
        valid = inputs.left_padded_mask(Bs, N, 7 + layer)
        outs = tuple(np.empty(h["q"].shape, np.float32) for _ in range(4)) + (np.zeros(Bs * H),)
        data.append((h, valid, outs))

    def step():
        for h, valid, outs in data:
            oracle.ref_batched_f32(h["q"], h["k"], h["v"], h["d_out"], valid, 1.0, 1e-6,
                                   threads, outs)

    for _ in range(max(args.warmup, 1)):
        step()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        step()
        times.append(time.perf_counter() - t0)
    total = sum(times)
    value = Bs * args.steps / total
    sample = (f"{Bs}-sequence sample of the {total_b}-sequence batch per step" if Bs < total_b
              else f"full {Bs}-sequence batch per step") + \
        f", {layers} layer(s), reference operator (oracle/_ref), {threads} threads"
    return {"metric": METRIC, "value": value, "unit": "seq/s", "impl": "reference",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": total / args.steps * 1e3 * (total_b / Bs if strong else 1.0),
            "higher_is_better": True, "scaling": "strong" if strong else "weak",
            "vs_baseline": None, "dtype": "f64 (reference arithmetic; f32 inputs)",
            "data": "synthetic", "config": {"workload": desc, "name": args.workload,
                                            "global_batch": total_b, "seq_len": N, "heads": H,
                                            "head_dim": D, "layers": layers},
            "cpu_baseline": {"value": value, "unit": "seq/s", "cores": threads,
                             "kind": "reference", "sample": sample},
            "e2e": {"value": value, "unit": "seq/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="ml1m", choices=sorted(WORKLOADS))
    ap.add_argument("--graph-scope", default="step", choices=["step", "op"],
                    help="graph mode: one graph for the whole step (default) or one per op call")
    ap.add_argument("--path", default="tcgen05", choices=["tcgen05", "fp32pipe"],
                    help="d_h=32 kernels: tcgen05 3xTF32 (default) or the FP32-pipe variant")
    ap.add_argument("--graph", default="auto", choices=["auto", "on", "off"],
                    help="replay captured CUDA graphs of the op calls (auto: when the eager step < 2 ms)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-steady", action="store_true",
                    help="skip the ML-20M steady-state block appended to the default (ml1m) line")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    args = ap.parse_args()

    world, rank, local = dist_setup(args.gpus)
    if args.impl == "reference":
        res = run_reference(args, world, rank)
    else:
        res = run_ours(args, world, rank, local)
        if (world == 1 and args.workload == "ml1m" and not args.no_steady and res is not None):
            # The default workload (config #2, B=256: 512 units on 148 SMs) is
            # latency-bound; report the same op at the ML-20M batch (config #4)
            # beside it as the kernels' steady-state roofline figure.
            import copy
            import torch
            torch.cuda.empty_cache()
            a2 = copy.copy(args)
            a2.workload, a2.steps, a2.warmup, a2.no_e2e, a2.no_cpu = "ml20m", 5, 3, True, True
            r2 = run_ours(a2, world, rank, local)
            res["steady_state"] = {
                "workload": r2["config"]["workload"], "value": r2["value"], "unit": "seq/s",
                "ms_per_step": r2["ms_per_step"], "launch": r2["config"]["launch"],
                "step_frac_of_hbm": r2["kernels"]["step_frac"],
                "fwd_frac": r2["kernels"]["fwd_frac"], "bwd_frac": r2["kernels"]["bwd_frac"],
                "roofline": r2["roofline"], "clocks": r2["clocks"]}
            torch.cuda.empty_cache()
    if rank == 0 and res is not None:
        print(json.dumps(res), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
