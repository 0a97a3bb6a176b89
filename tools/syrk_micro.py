"""Dev tool: the tcgen05 SYRK kernel alone vs cuBLASLt (torch._int_mm) on the
same int8 planes: n x n lower triangle over K rows (one modulus), rates in
TOPS counted on the work each does (SYRK: lower-triangle tiles; GEMM: all).
usage: python tools/syrk_micro.py [n] [K] [reps]"""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1907_05884_b200._lib import Err, check, lib

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
K = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
x = torch.randint(-127, 128, (n, K), dtype=torch.int8, device="cuda")  # plane: column a = row a here
c = torch.empty(n * n, dtype=torch.int8, device="cuda")
s = torch.cuda.current_stream().cuda_stream
t = n // 256
tiles = t * (t + 1) // 2


def syrk():
    err = Err()
    check(lib().fstk_gpu_debug_syrk(x.data_ptr(), 1, K, n, c.data_ptr(), 0, s, C.byref(err)), err)


def gemm():
    return torch._int_mm(x, x.t())


for name, f, ops in (("syrk", syrk, 2.0 * tiles * 256 * 256 * K), ("int_mm", gemm, 2.0 * n * n * K)):
    f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"{name:7s} n={n} K={K}: {ms:.3f} ms  {ops / ms / 1e9:.0f} TOPS (work-normalised)")
