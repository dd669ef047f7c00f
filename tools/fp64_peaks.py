"""Measure cuBLAS fp64 / tf32 GEMM throughput on this B200 (roofline denominators).

Prints one JSON line. Used to set the FP64 peak the Gram kernel is judged
against (MEASURED_PEAKS.json carries no fp64/tf32 figure).
"""
import json
import time

import torch


def gemm_rate(dtype, n, seconds, tf32=False):
    torch.backends.cuda.matmul.allow_tf32 = tf32
    a = torch.randn(n, n, device="cuda", dtype=dtype)
    b = torch.randn(n, n, device="cuda", dtype=dtype)
    c = torch.empty(n, n, device="cuda", dtype=dtype)
    for _ in range(3):
        torch.matmul(a, b, out=c)
    torch.cuda.synchronize()
    best = float("inf")
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    for _ in range(5):
        e0.record(); torch.matmul(a, b, out=c); e1.record(); e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    burst = 2.0 * n ** 3 / best / 1e9
    t_end = time.time() + seconds
    reps = 0
    e0.record()
    while time.time() < t_end:
        torch.matmul(a, b, out=c)
        reps += 1
        if reps % 4 == 0:
            torch.cuda.synchronize()
    e1.record(); e1.synchronize()
    sustained = 2.0 * n ** 3 * reps / e0.elapsed_time(e1) / 1e9
    return burst, sustained


def int8_rate(n, seconds):
    """cuBLASLt int8 x int8 -> int32 (torch._int_mm): the int8 tensor peak the kind::i8 Gram is judged against."""
    a = torch.randint(-64, 65, (n, n), device="cuda", dtype=torch.int8)
    b = torch.randint(-64, 65, (n, n), device="cuda", dtype=torch.int8).t().contiguous().t()
    for _ in range(3):
        c = torch._int_mm(a, b)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    best = float("inf")
    for _ in range(5):
        e0.record(); c = torch._int_mm(a, b); e1.record(); e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    burst = 2.0 * n ** 3 / best / 1e9
    t_end = time.time() + seconds
    reps = 0
    e0.record()
    while time.time() < t_end:
        c = torch._int_mm(a, b)
        reps += 1
        if reps % 4 == 0:
            torch.cuda.synchronize()
    e1.record(); e1.synchronize()
    return burst, 2.0 * n ** 3 * reps / e0.elapsed_time(e1) / 1e9


if __name__ == "__main__":
    import sys
    if len(sys.argv) > 1 and sys.argv[1] == "int8":
        i8 = int8_rate(8192, 4.0)
        print(json.dumps({"int8_tops_burst": round(i8[0], 1), "int8_tops_sustained": round(i8[1], 1),
                          "gpu": torch.cuda.get_device_name(0),
                          "how": "torch._int_mm (cuBLASLt int8 -> int32) 8192^3, best of 5 / back to back 4 s"}))
        sys.exit(0)
    f64 = gemm_rate(torch.float64, 8192, 4.0)
    tf32 = gemm_rate(torch.float32, 8192, 4.0, tf32=True)
    f32 = gemm_rate(torch.float32, 8192, 2.0, tf32=False)
    print(json.dumps({
        "fp64_dgemm_tflops_burst": round(f64[0], 2), "fp64_dgemm_tflops_sustained": round(f64[1], 2),
        "tf32_tflops_burst": round(tf32[0], 1), "tf32_tflops_sustained": round(tf32[1], 1),
        "fp32_sgemm_tflops_burst": round(f32[0], 1), "fp32_sgemm_tflops_sustained": round(f32[1], 1),
        "gpu": torch.cuda.get_device_name(0),
        "how": "torch.matmul 8192^3, best of 5 (burst) and back-to-back loop (sustained), CUDA events",
    }))
