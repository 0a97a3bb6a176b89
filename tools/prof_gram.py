"""Dev tool: the sliced Gram alone at C2 size (S = 262144 rows, R = 32768).
usage: python tools/prof_gram.py [slices] [rows] [n]   (profiled region = 2nd call)"""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1907_05884_b200._lib import Err, check, lib

ns = int(sys.argv[1]) if len(sys.argv) > 1 else 7
rows = int(sys.argv[2]) if len(sys.argv) > 2 else 262144
n = int(sys.argv[3]) if len(sys.argv) > 3 else 32768
a = torch.randn(n, rows, dtype=torch.float64, device="cuda")  # column-major rows x n
g = torch.zeros(n * n, dtype=torch.float64, device="cuda")
stream = torch.cuda.current_stream().cuda_stream


def run():
    err = Err()
    check(lib().fstk_gpu_gram_device(a.data_ptr(), rows, rows, n, g.data_ptr(), ns, 0, stream,
                                     C.byref(err)), err)


run()
torch.cuda.synchronize()
torch.cuda.profiler.start()
t0 = time.perf_counter()
run()
torch.cuda.synchronize()
dt = time.perf_counter() - t0
torch.cuda.profiler.stop()
flops = rows * n * (n + 1)
print(f"ns={ns} rows={rows} n={n}: {dt:.3f} s  fp64-equivalent {flops / dt / 1e12:.1f} TFLOP/s")
