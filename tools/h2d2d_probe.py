"""Probe: PCIe H2D bandwidth of column-slab (2-D) copies vs one contiguous copy.

Decides whether the host entry point can stream X by column blocks (Gram tiles
(i, c) start once column block c has landed) without losing PCIe bandwidth.
"""
import time

import torch
from cuda.bindings import runtime as rt

n, k = 1_000_000, 500
h = torch.empty((n, k), dtype=torch.float64).pin_memory()
h.normal_()
d = torch.empty((n, k), dtype=torch.float64, device="cuda")
s = torch.cuda.current_stream().cuda_stream
H2D = rt.cudaMemcpyKind.cudaMemcpyHostToDevice


def timed(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best


def contiguous():
    d.copy_(h, non_blocking=True)


def slabs(cols):
    def run():
        for c0 in range(0, k, cols):
            w = min(cols, k - c0)
            err, = rt.cudaMemcpy2DAsync(d.data_ptr() + c0 * 8, k * 8, h.data_ptr() + c0 * 8, k * 8, w * 8, n, H2D, s)
            assert err == rt.cudaError_t.cudaSuccess, err
    return run


gb = n * k * 8 / 1e9
t = timed(contiguous)
print(f"contiguous {gb:.2f} GB: {t*1e3:.1f} ms = {gb/t:.1f} GB/s")
for cols in (32, 64, 128, 256):
    t = timed(slabs(cols))
    print(f"2D slabs of {cols} cols ({cols*8} B rows): {t*1e3:.1f} ms = {gb/t:.1f} GB/s")
