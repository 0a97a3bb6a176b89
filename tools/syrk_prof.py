"""Dev tool: per-kernel device time of one CRT Gram (C2 size by default) in a
normal (non-ncu) run via torch.profiler/CUPTI, next to its wall time.
usage: python tools/syrk_prof.py [slices] [rows] [n] [engine]"""
import collections
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
eng = sys.argv[4] if len(sys.argv) > 4 else "tcgen05"
F.gram_engine(eng)
a = torch.randn(n, rows, dtype=torch.float64, device="cuda")
g = torch.zeros(n * n, dtype=torch.float64, device="cuda")
stream = torch.cuda.current_stream().cuda_stream


def run():
    err = Err()
    check(lib().fstk_gpu_gram_device(a.data_ptr(), rows, rows, n, g.data_ptr(), ns, 0, stream,
                                     C.byref(err)), err)


run()
torch.cuda.synchronize()
t0 = time.perf_counter()
run()
torch.cuda.synchronize()
wall = time.perf_counter() - t0
from torch.profiler import ProfilerActivity, profile

with profile(activities=[ProfilerActivity.CUDA]) as prof:
    run()
    torch.cuda.synchronize()
agg = collections.defaultdict(lambda: [0, 0.0])
first, last = None, None
for e in prof.events():
    if e.device_type.name != "CUDA":
        continue
    agg[e.name[:70]][0] += 1
    agg[e.name[:70]][1] += e.device_time_total / 1e3 if hasattr(e, "device_time_total") else e.cuda_time_total / 1e3
tot = sum(v[1] for v in agg.values())
print(f"{eng} ns={ns} rows={rows} n={n}: wall {wall:.3f} s, kernel sum {tot / 1e3:.3f} s")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:8]:
    print(f"  {v[1]:9.2f} ms {v[0]:5d}  {k}")
