"""Dev tool (profiling target): one C2-size IDW interpolation (16.8M points ->
256^3) and one 256^3 grid reconstruction, for ncu captures."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_1907_05884_b200 as F
from paper_1907_05884_b200 import synth

q, m = 1 << 24, 256
rng = np.random.default_rng(0)
i = np.arange(q)
base = np.stack([i % m, (i // m) % m, i // (m * m)], axis=1)
pts = (base + 0.5 + rng.uniform(-0.4, 0.4, (q, 3))) / m
vals = np.tanh((pts[:, 2] - 0.5) / 0.02)
pc = F.PointCloud.from_data(pts, vals)
g, rep = F.interpolate_to_grid(pc, F.StructuredGrid.unit([m, m, m]))
model = synth.random_model((32, 32, 32), (48, 48, 48), 24, seed=0)
r = model.reconstruct_grid((m, m, m))
print("ok", g.shape, rep, r.shape)
