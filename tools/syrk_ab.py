"""Dev tool: A/B of the CRT Gram engines at C2 size, interleaved repetitions
in one process (medians of wall time per engine), bit-identity checked.
usage: python tools/syrk_ab.py [slices] [rows] [n] [reps]"""
import ctypes as C
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1907_05884_b200 as F
from paper_1907_05884_b200._lib import Err, check, lib

ns = int(sys.argv[1]) if len(sys.argv) > 1 else 4
rows = int(sys.argv[2]) if len(sys.argv) > 2 else 262144
n = int(sys.argv[3]) if len(sys.argv) > 3 else 32768
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 4
a = torch.randn(n, rows, dtype=torch.float64, device="cuda")
stream = torch.cuda.current_stream().cuda_stream
gs = {e: torch.zeros(n * n, dtype=torch.float64, device="cuda") for e in ("tcgen05", "cublaslt")}
ts = {e: [] for e in gs}


from torch.profiler import ProfilerActivity, profile

ks = {e: [] for e in gs}


def run(e):
    F.gram_engine(e)
    err = Err()
    time.sleep(float(os.environ.get("AB_COOL", "3")))  # same thermal state for every sample
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        t0 = time.perf_counter()
        check(lib().fstk_gpu_gram_device(a.data_ptr(), rows, rows, n, gs[e].data_ptr(), ns, 0, stream,
                                         C.byref(err)), err)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    kern = sum(ev.device_time_total for ev in prof.events() if ev.device_type.name == "CUDA") / 1e6
    ks[e].append(kern)
    return dt


for e in gs:
    run(e)
for _ in range(reps):
    for e in gs:
        ts[e].append(run(e))
for e in gs:
    print(f"{e:9s}: wall median {statistics.median(ts[e]):.3f} s ({' '.join(f'{t:.3f}' for t in ts[e])}); "
          f"kernels median {statistics.median(ks[e]):.3f} s ({' '.join(f'{t:.3f}' for t in ks[e])})")
print("bit-identical:", bool(torch.equal(gs["tcgen05"], gs["cublaslt"])))
