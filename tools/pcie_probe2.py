"""PCIe probe 2: concurrent H2D + D2H of a 3-component T-vector (99.2 M
doubles) in k slabs, as 3 k plain copies (one per component range) vs k
strided 2D copies (cudaMemcpy2DAsync: the three component ranges of a slab
in one call)."""
import ctypes
import os
import time

import torch

import nvidia.cuda_runtime as _rt

rt = ctypes.CDLL(os.path.join(_rt.__path__[0], "lib", "libcudart.so.12"))
rt.cudaMemcpy2DAsync.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_size_t,
                                 ctypes.c_size_t, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]
nn = 33076161
n = 3 * nn
h = torch.empty(n, dtype=torch.float64, pin_memory=True).normal_()
o = torch.empty(n, dtype=torch.float64, pin_memory=True)
d = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.randn(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
H, O, D, D2 = h.view(3, nn), o.view(3, nn), d.view(3, nn), d2.view(3, nn)


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


def plain(k, do_h2d=True, do_d2h=True):
    c = nn // k + 1
    for i in range(0, nn, c):
        j = min(nn, i + c)
        if do_h2d:
            with torch.cuda.stream(s1):
                for cc in range(3):
                    D[cc, i:j].copy_(H[cc, i:j], non_blocking=True)
        if do_d2h:
            with torch.cuda.stream(s2):
                for cc in range(3):
                    O[cc, i:j].copy_(D2[cc, i:j], non_blocking=True)


def twod(k, do_h2d=True, do_d2h=True):
    c = nn // k + 1
    for i in range(0, nn, c):
        j = min(nn, i + c)
        if do_h2d:
            assert rt.cudaMemcpy2DAsync(d.data_ptr() + 8 * i, nn * 8, h.data_ptr() + 8 * i, nn * 8, (j - i) * 8, 3, 1,
                                        s1.cuda_stream) == 0
        if do_d2h:
            assert rt.cudaMemcpy2DAsync(o.data_ptr() + 8 * i, nn * 8, d2.data_ptr() + 8 * i, nn * 8, (j - i) * 8, 3, 2,
                                        s2.cuda_stream) == 0


gb = n * 8 / 1e9
for k in (1, 4, 16, 32):
    for name, fn in (("plain", plain), ("2d", twod)):
        a = t(lambda: fn(k, True, False))
        b = t(lambda: fn(k, False, True))
        c = t(lambda: fn(k))
        print(f"{name:5s} slabs={k:3d}: H2D {a:6.2f} ms ({gb / a * 1e3:5.1f} GB/s)  D2H {b:6.2f} ms  both {c:6.2f} ms",
              flush=True)
ok = torch.equal(d.cpu(), h) and torch.equal(o, d2.cpu())
print("exact", ok)
