"""Dev tool: the CRT Gram at C2 size with both int8 GEMM engines (tcgen05
SYRK vs cuBLASLt), checked bit-identical.
usage: python tools/syrk_time.py [slices] [rows] [n] [reps]"""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1907_05884_b200 as F
from paper_1907_05884_b200._lib import Err, check, lib

ns = int(sys.argv[1]) if len(sys.argv) > 1 else 4
rows = int(sys.argv[2]) if len(sys.argv) > 2 else 262144
n = int(sys.argv[3]) if len(sys.argv) > 3 else 32768
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
a = torch.randn(n, rows, dtype=torch.float64, device="cuda")  # column-major rows x n
stream = torch.cuda.current_stream().cuda_stream
flops = rows * n * (n + 1)
out = {}
for eng in ("tcgen05", "cublaslt", "tcgen05"):
    F.gram_engine(eng)
    g = torch.zeros(n * n, dtype=torch.float64, device="cuda")
    ts = []
    for _ in range(reps):
        err = Err()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        check(lib().fstk_gpu_gram_device(a.data_ptr(), rows, rows, n, g.data_ptr(), ns, 0, stream,
                                         C.byref(err)), err)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    out[eng] = g
    print(f"{eng:9s} ns={ns} rows={rows} n={n}: " + " ".join(f"{t:.3f}" for t in ts)
          + f" s  (fp64-equivalent {flops / min(ts) / 1e12:.0f} TFLOP/s)", flush=True)
print("bit-identical:", bool(torch.equal(out["tcgen05"], out["cublaslt"])))
