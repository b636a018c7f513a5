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
    w = a[:, :2, :, :5]
    ok = (w[..., 4] > 0) & (w[..., 0] > 0)
    d = np.diff(w, axis=-1)
    gap = w[:, :, 1:, 0] - w[:, :, :-1, 4]
    okg = ok[:, :, 1:] & ok[:, :, :-1]
    print(f"{tag}: items traced {int(ok.sum())}")
    for i, n in enumerate(["tma_wait", "split", "mma_wait", "epilogue"]):
        v = d[..., i][ok]
        print(f"  {n:9s} mean {v.mean():8.0f} cyc  median {np.median(v):8.0f}  p90 {np.percentile(v, 90):8.0f}")
    print(f"  {'gap':9s} mean {gap[okg].mean():8.0f} cyc")
    w5 = a[:, :2, :, 5]
    ok5 = ok & (w5 > 0)
    print(f"  epi before barrier->store {(w5 - w[..., 3])[ok5].mean():8.0f}   store issue {(w[..., 4] - w5)[ok5].mean():8.0f}")
    per_item = (w[:, :, 1:, 0] - w[:, :, :-1, 0])[okg]
    print(f"  item period per group: mean {per_item.mean():.0f} cyc")
    # MMA thread: global item it -> group it&1, group-local index it>>1
    m = a[:, 2, :, :3]
    okm = m[..., 2] > 0
    print(f"  mma: wait for split mean {(m[..., 1] - m[..., 0])[okm].mean():.0f}  issue mean {(m[..., 2] - m[..., 1])[okm].mean():.0f}")
    # latency from worker 'split published' to MMA thread 'got split', and MMA issue end -> worker sees done
    lat1, lat2 = [], []
    for it in range(K):
        g, k = it & 1, it >> 1
        okk = okm[:, it] & ok[:, g, k]
        lat1.append((m[:, it, 1] - w[:, g, k, 2])[okk])
        lat2.append((w[:, g, k, 3] - m[:, it, 2])[okk])
    lat1, lat2 = np.concatenate(lat1), np.concatenate(lat2)
    print(f"  split published -> MMA thread starts: mean {lat1.mean():.0f}  median {np.median(lat1):.0f}")
    print(f"  MMA issued -> worker sees done:      mean {lat2.mean():.0f}  median {np.median(lat2):.0f}")
    for kind in range(4):
        # items by pass/chunk pattern for C=2: it%4 = 0:p1c0 1:p1c1 2:p2c0 3:p2c1
        sel = [it for it in range(K) if it % 4 == kind]
        v = np.concatenate([(w[:, it & 1, it >> 1, 3] - m[:, it, 2])[okm[:, it] & ok[:, it & 1, it >> 1]] for it in sel])
        sp = np.concatenate([d[:, it & 1, it >> 1, 1][ok[:, it & 1, it >> 1]] for it in sel])
        ep = np.concatenate([d[:, it & 1, it >> 1, 3][ok[:, it & 1, it >> 1]] for it in sel])
        iss = np.concatenate([(m[:, it, 2] - m[:, it, 1])[okm[:, it]] for it in sel])
        print(f"  item kind {kind} (it%4): split {sp.mean():6.0f}  issue {iss.mean():6.0f}  exec {v.mean():6.0f}  epi {ep.mean():6.0f}")
