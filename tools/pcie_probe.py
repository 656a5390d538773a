"""PCIe probe: pinned H2D / D2H of one T-vector (99.2 M doubles), alone and
concurrently on two streams, whole and in chunks."""
import time

import torch

n = 99228483
h = torch.empty(n, dtype=torch.float64, pin_memory=True).normal_()
o = torch.empty(n, dtype=torch.float64, pin_memory=True)
d = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.randn(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


def h2d(chunks=1):
    c = n // chunks + 1
    with torch.cuda.stream(s1):
        for i in range(0, n, c):
            d[i:i + c].copy_(h[i:i + c], non_blocking=True)


def d2h(chunks=1):
    c = n // chunks + 1
    with torch.cuda.stream(s2):
        for i in range(0, n, c):
            o[i:i + c].copy_(d2[i:i + c], non_blocking=True)


gb = n * 8 / 1e9
for ch in (1, 8, 32):
    a = t(lambda: h2d(ch))
    b = t(lambda: d2h(ch))
    c = t(lambda: (h2d(ch), d2h(ch)))
    print(f"chunks={ch:3d}: H2D {a:6.2f} ms ({gb / a * 1e3:5.1f} GB/s)  D2H {b:6.2f} ms ({gb / b * 1e3:5.1f} GB/s)  "
          f"both {c:6.2f} ms")
