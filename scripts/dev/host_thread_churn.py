"""Host entry points called from a new thread for every step (the reference's
short-lived parallel_chunks workers) against one persistent thread: ML-1M shape,
2 layers, cached fwd/bwd pair per layer, pinned buffers; seq/s per 20-step window."""
import ctypes
import sys
import threading
import time

import torch

sys.path.insert(0, ".")
from paper_2602_06935_b200 import _lib, inputs  # noqa: E402

B, H, N, D, layers = 256, 2, 200, 32, 2
lib = _lib.load()
desc = _lib.make_desc(B, H, N, D, "f32", 1e-6)
Ls = []
for layer in range(layers):
    h = inputs.make_host(B, H, N, D, seed=7 + layer)
    t = {n: torch.from_numpy(x).pin_memory() for n, x in h.items()}
    t["valid"] = torch.from_numpy(inputs.left_padded_mask(B, N, 7 + layer)).pin_memory()
    for n in ("out", "dq", "dk", "dv"):
        t[n] = torch.empty(B, H, N, D).pin_memory()
    Ls.append(t)
p = lambda x: ctypes.c_void_p(x.data_ptr())  # noqa: E731


def step():
    caches = []
    for t in Ls:
        c = ctypes.c_void_p()
        _lib.check(lib.cotten_fwd_host_cached(ctypes.byref(desc), p(t["q"]), p(t["k"]), p(t["v"]),
                                              p(t["valid"]), 1.0, p(t["out"]), None, ctypes.byref(c)))
        caches.append(c)
    for t, c in zip(reversed(Ls), reversed(caches)):
        _lib.check(lib.cotten_bwd_host_cached(c, p(t["d_out"]), p(t["dq"]), p(t["dk"]), p(t["dv"]),
                                              None, None))
        _lib.check(lib.cotten_host_cache_free(c))


def in_new_thread(f):
    th = threading.Thread(target=lambda: (torch.cuda.set_device(0), f()))
    th.start()
    th.join()


for _ in range(5):
    step()
for mode in ("persistent", "new thread per step", "persistent"):
    win = []
    for w in range(7):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(20):
            (step() if mode == "persistent" else in_new_thread(step))
        win.append(round(20 * B / (time.perf_counter() - t0)))
    print("%-20s %s" % (mode, win))
