"""Dev probe: achievable int8 x int8 -> int32 GEMM rate on this B200 (cuBLASLt
via torch._int_mm), and fp64 DGEMM beside it, to size the sliced-Gram path."""
import sys

import torch


def bench(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


for m, n, k in [(8192, 8192, 16384), (8192, 8192, 65536), (16384, 16384, 32768), (4096, 32768, 32768)]:
    a = torch.randint(-127, 128, (m, k), dtype=torch.int8, device="cuda")
    b = torch.randint(-127, 128, (n, k), dtype=torch.int8, device="cuda").t()
    ms = bench(lambda: torch._int_mm(a, b))
    print(f"int8 TN m={m} n={n} k={k}: {ms:.3f} ms  {2 * m * n * k / ms / 1e9:.1f} TOPS", flush=True)
    del a, b
a = torch.randn(8192, 16384, dtype=torch.float64, device="cuda")
b = torch.randn(16384, 8192, dtype=torch.float64, device="cuda")
ms = bench(lambda: a @ b)
print(f"fp64 8192x8192x16384: {ms:.3f} ms {2 * 8192 * 8192 * 16384 / ms / 1e9:.1f} TFLOPS")
sys.exit(0)
