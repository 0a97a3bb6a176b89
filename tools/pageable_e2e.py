"""Dev tool: host-buffer evaluate_batch at C2 with pageable numpy arrays vs the
pinned path the bench's e2e uses."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from bench import workload

model, pts, vals, c = workload("C2", 0, 0)
n = pts.shape[0]
model.evaluate_batch(pts[:100000])
for _ in range(2):
    t0 = time.perf_counter()
    out = model.evaluate_batch(pts)
    dt = time.perf_counter() - t0
    print(f"pageable: {n / dt:.3e} pts/s ({dt * 1e3:.1f} ms)", flush=True)
pin = torch.empty((3, n), dtype=torch.float64).pin_memory()
pin.numpy()[:] = pts.T
po = torch.empty(n, dtype=torch.float64).pin_memory()
for _ in range(2):
    t0 = time.perf_counter()
    model.evaluate_batch_into(pin.numpy().T, po.numpy())
    dt = time.perf_counter() - t0
    print(f"pinned:   {n / dt:.3e} pts/s ({dt * 1e3:.1f} ms)", flush=True)
