"""Summarise bf16 tcgen05 per-item traces ($COTTEN_TRACE_DIR/tcb_{fwd,bwd}.bin,
-DCOTTEN_TCB_TRACE=1 builds): [cta][item][8] clock64 stamps, see kernels_tcb.cuh."""
import sys
import numpy as np

K = 64
names = ["split wait raw", "raw landed", "split published", "mma sees split", "mma issued",
         "epi sees done", "epi staged", "slot freed"]
for tag in ("tcb_fwd", "tcb_bwd", "tcg_bwd"):
    try:
        a = np.fromfile(f"{sys.argv[1]}/{tag}.bin", dtype=np.int64).reshape(-1, K, 8).astype(np.float64)
    except FileNotFoundError:
        continue
    ok = np.all(a > 0, axis=2)
    ok[:, :8] = False  # skip the ramp
    print(f"{tag}: items {int(ok.sum())}")
    d = lambda i, j: (a[..., j] - a[..., i])[ok]  # noqa: E731
    for i, j, n in [(0, 1, "splitter wait raw"), (1, 2, "split work"), (2, 3, "split->mma"),
                    (3, 4, "mma issue"), (4, 5, "mma issued->epi sees done"), (5, 6, "epilogue work"),
                    (6, 7, "staged->slot freed (store)"), (1, 7, "raw landed->slot freed")]:
        v = d(i, j)
        print(f"  {n:30s} mean {v.mean():7.0f} median {np.median(v):7.0f} p90 {np.percentile(v, 90):7.0f}")
    okn = ok[:, 1:] & ok[:, :-1]
    for k, n in [(0, "splitter"), (3, "mma"), (5, "epiloguer"), (7, "store")]:
        v = (a[:, 1:, k] - a[:, :-1, k])[okn]
        print(f"  period {n:22s} mean {v.mean():7.0f} median {np.median(v):7.0f}")
