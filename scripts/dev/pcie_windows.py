"""Pinned h2d / d2h bandwidth in repeated windows (is the PCIe path itself noisy on
this box?): 15 windows of 8 x 64 MB each way, duplex on two streams."""
import time
import torch
n = 64 << 20
h = torch.empty(n, dtype=torch.uint8).pin_memory(); h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda"); d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for w in range(15):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(8):
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    print("window %2d: %.1f GB/s each way" % (w, 8 * n / el / 1e9))
