"""Dev tool: reconstruct --grid time (fstk_gpu_reconstruct_grid: mode tables
on the grid lines + DMMA mode products + read-back) at 256^3, ranks 32^3.
usage: python tools/grid_time.py [n]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_1907_05884_b200 import synth

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
m = synth.random_model((32, 32, 32), (48, 48, 48), 24, seed=0)
m.reconstruct_grid((n, n, n))
ts = []
for _ in range(5):
    t0 = time.perf_counter()
    g = m.reconstruct_grid((n, n, n))
    ts.append(time.perf_counter() - t0)
print(f"reconstruct_grid {n}^3 at ranks 32^3: best {min(ts) * 1e3:.1f} ms, median "
      f"{np.median(ts) * 1e3:.1f} ms ({g.nbytes / 1e6:.0f} MB read back)")
