"""Dev tool: blocked int8 Cholesky vs cuSOLVER dpotrf at R = 32768 (times, backward error).
usage: python tools/chol_time.py [reps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1907_05884_b200 as F

n = 32768
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 4
g = torch.randn(n, n, dtype=torch.float64, device="cuda")
g = g @ g.t() / n + torch.eye(n, dtype=torch.float64, device="cuda")
gn = float(torch.linalg.norm(g))
for slices in (5, 0):
    for r in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        l, info = F.cholesky(g, slices=slices)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        msg = f"slices={slices} run {r}: {dt:.3f} s (incl. transposes of the 8.6 GB matrix) info {info}"
        if r == reps - 1:
            msg += f" backward {float(torch.linalg.norm(l @ l.t() - g)) / gn:.2e}"
        print(msg, flush=True)
        del l
