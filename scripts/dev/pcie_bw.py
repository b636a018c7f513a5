"""Pinned h2d / d2h / duplex copy bandwidth on this box (the e2e bound)."""
import torch
n = 64 << 20
h = torch.empty(n, dtype=torch.uint8).pin_memory(); h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda"); d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(f, reps=10):
    for _ in range(2): f()
    torch.cuda.synchronize(); a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); [f() for _ in range(reps)]; b.record(); torch.cuda.synchronize(); return a.elapsed_time(b) / reps / 1e3
th = t(lambda: d.copy_(h, non_blocking=True)); td = t(lambda: h2.copy_(d2, non_blocking=True))
def duplex():
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
tb = t(duplex)
print("h2d %.1f GB/s  d2h %.1f GB/s  duplex %.1f GB/s each way" % (n / th / 1e9, n / td / 1e9, n / tb / 1e9))
