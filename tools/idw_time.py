"""Dev tool: GPU IDW interpolation (fstk_idw.cu) time at C1 (200k points ->
64^3) and C2 (16.8M jittered mesh points -> 256^3), with the oracle's CPU
time on all host cores beside it (C2's CPU leg on a 64^3 sub-grid, scaled).
usage: python tools/idw_time.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1907_05884_b200 as F
from oracle import oracle as O

O.set_max_threads(os.cpu_count())
for name, q, n in (("C1", 200_000, 64), ("C2", 1 << 24, 256)):
    rng = np.random.default_rng(0)
    if name == "C2":
        m = 256
        i = np.arange(q)
        base = np.stack([i % m, (i // m) % m, i // (m * m)], axis=1)
        pts = (base + 0.5 + rng.uniform(-0.4, 0.4, (q, 3))) / m
    else:
        pts = rng.random((q, 3))
    x, y, z = pts.T
    vals = np.tanh((z - 0.5 - 0.05 * np.sin(2 * np.pi * x) * np.sin(2 * np.pi * y)) / 0.02)
    pc = F.PointCloud.from_data(pts, vals)
    grid = F.StructuredGrid.unit([n, n, n])
    F.interpolate_to_grid(pc, grid)
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        g, rep = F.interpolate_to_grid(pc, grid)
        ts.append(time.perf_counter() - t0)
    nc = min(n, 64)
    t0 = time.perf_counter()
    go, _ = O.interpolate_to_grid(pts, vals, (nc, nc, nc) if name == "C2" else (n, n, n))
    tc = (time.perf_counter() - t0) * (n ** 3 / nc ** 3 if name == "C2" else 1.0)
    if name == "C1":
        print("  max |gpu - oracle| =", float(np.abs(g - go).max()))
    print(f"{name}: {q} points -> {n}^3 nodes: GPU (host arrays in/out) {min(ts):.3f} s "
          f"({n ** 3 / min(ts):.3g} nodes/s); oracle on {os.cpu_count()} cores {tc:.2f} s"
          f"{' (64^3 sub-grid scaled)' if name == 'C2' else ''}; report {rep}", flush=True)
