"""Summarise tcgen05 phase traces ($COTTEN_TRACE_DIR/{fwd,bwd}.bin, trace builds)."""
import sys
import numpy as np

K = 64
for tag in ("fwd", "bwd"):
    try:
        a = np.fromfile(f"{sys.argv[1]}/{tag}.bin", dtype=np.int64)
    except FileNotFoundError:
        continue
    a = a.reshape(-1, 3, K, 8).astype(np.float64)
    sp, ep, mm = a[:, 0], a[:, 1], a[:, 2]
    ok = (sp[..., 2] > 0) & (ep[..., 4] > 0) & (mm[..., 2] > 0)
    print(f"{tag}: items traced {int(ok.sum())}")
    def stat(name, v):
        print(f"  {name:34s} mean {v.mean():7.0f}  median {np.median(v):7.0f}  p90 {np.percentile(v, 90):7.0f}")
    stat("splitter: wait stage + lo buffer", (sp[..., 1] - sp[..., 0])[ok])
    stat("splitter: split", (sp[..., 2] - sp[..., 1])[ok])
    okn = ok[:, 1:] & ok[:, :-1]
    stat("splitter: period", (sp[:, 1:, 0] - sp[:, :-1, 0])[okn])
    stat("mma: split published -> start", (mm[..., 1] - sp[..., 2])[ok])
    stat("mma: issue", (mm[..., 2] - mm[..., 1])[ok])
    stat("mma issued -> epiloguer sees done", (ep[..., 3] - mm[..., 2])[ok])
    stat("epiloguer: compute+stage", (ep[..., 5] - ep[..., 3])[ok])
    stat("epiloguer: staged arrive", (ep[..., 4] - ep[..., 5])[ok])
    stat("epiloguer: idle before next done", (ep[:, 1:, 3] - ep[:, :-1, 4])[okn])
    stat("epiloguer: period", (ep[:, 1:, 3] - ep[:, :-1, 3])[okn])
    if tag == "bwd":
        for kind in (0, 1):
            sel = [it for it in range(K) if it % 4 == kind]
            g = lambda x: np.concatenate([x[:, it][ok[:, it]] for it in sel]).mean()  # noqa: E731
            print(f"  bwd p1 kind {kind} split phases: load+norm+split {g(sp[..., 3] - sp[..., 1]):5.0f}"
                  f"  Q stores+unswap+tmem {g(sp[..., 4] - sp[..., 3]):5.0f}  dO load/split/stores+unswap {g(sp[..., 5] - sp[..., 4]):5.0f}"
                  f"  dO tmem+S-op+wait {g(sp[..., 6] - sp[..., 5]):5.0f}  fence+arrive {g(sp[..., 2] - sp[..., 6]):5.0f}")
    for kind in range(4):
        sel = [it for it in range(K) if it % 4 == kind]
        f = lambda x: np.concatenate([x[:, it][ok[:, it]] for it in sel]).mean()  # noqa: E731
        print(f"  kind {kind} (it%4): split {f(sp[..., 2] - sp[..., 1]):6.0f}  mma {f(mm[..., 2] - mm[..., 1]):6.0f}"
              f"  epi {f(ep[..., 5] - ep[..., 3]):6.0f}  epi-staged {f(ep[..., 4] - ep[..., 5]):6.0f}")

# CTA timelines (globaltimer ns): entry, setup done, last item done, exit
for tag in ("fwd", "bwd"):
    try:
        a = np.fromfile(f"{sys.argv[1]}/{tag}.bin", dtype=np.int64).reshape(-1, 3, K, 8)
    except FileNotFoundError:
        continue
    c = a[:, 2, K - 1, 4:8].astype(np.float64)
    c = c[c[:, 0] > 0]
    t0 = c[:, 0].min()
    c = (c - t0) / 1e3  # us
    print(f"{tag} CTA timeline (us from the first CTA entry): entry max {c[:, 0].max():.2f}  setup done mean {c[:, 1].mean():.2f}"
          f"  last item done mean {c[:, 2].mean():.2f} max {c[:, 2].max():.2f}  exit max {c[:, 3].max():.2f}")

# Item timeline of the slowest CTA (clock64 cycles from its first splitter stamp, in us at 1.965 GHz)
for tag in ("fwd", "bwd"):
    try:
        a = np.fromfile(f"{sys.argv[1]}/{tag}.bin", dtype=np.int64).reshape(-1, 3, K, 8)
    except FileNotFoundError:
        continue
    c = a[:, 2, K - 1, 4:8].astype(np.float64)
    live = np.where(c[:, 0] > 0)[0]
    slow = live[np.argmax(c[live, 2])]
    sp, ep, mm = (a[slow, i].astype(np.float64) for i in range(3))
    n = int(((sp[:, 0] > 0) & (sp[:, 2] > 0)).sum())
    t0 = sp[0, 0]
    us = lambda x: (x - t0) / 1965.0  # noqa: E731
    print(f"{tag}: slowest CTA {slow}, {n} items (us): split start / published | mma start / issued | epi sees done / staged")
    for it in range(min(n, 24)):
        print(f"  it {it:2d}: {us(sp[it, 1]):6.2f} {us(sp[it, 2]):6.2f} | {us(mm[it, 1]):6.2f} {us(mm[it, 2]):6.2f} | "
              f"{us(ep[it, 3]):6.2f} {us(ep[it, 4]):6.2f}")

# Start-up stamps (globaltimer, us from the first CTA entry): mask warp start, flags
# published, producer's first TMA issued, splitter past fl_full, item 0 landed
for tag in ("fwd", "bwd"):
    try:
        a = np.fromfile(f"{sys.argv[1]}/{tag}.bin", dtype=np.int64).reshape(-1, 3, K, 8)
    except FileNotFoundError:
        continue
    c = a[:, 2, K - 1, 4:8].astype(np.float64)
    t = a[:, 2, K - 2, 0:5].astype(np.float64)
    live = (c[:, 0] > 0) & (t[:, 0] > 0)
    if not live.any():
        continue
    t0 = c[live, 0].min()
    t = (t[live] - t0) / 1e3
    names = ("mask start", "flags published", "first TMA issued", "splitter past flags", "item 0 landed")
    print(f"{tag} start-up (us): " + "  ".join(f"{n} {t[:, i].mean():.2f}/{t[:, i].max():.2f}" for i, n in enumerate(names)))
