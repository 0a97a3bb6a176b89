"""Profiling driver (dev tool): refit at q_pad = 2^20 with a small core so the
transform passes are representative.  usage: python tools/prof_refit.py [transform] [r]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_1907_05884_b200 as F
from paper_1907_05884_b200 import _lib, synth

t = sys.argv[1] if len(sys.argv) > 1 else "dct"
r = int(sys.argv[2]) if len(sys.argv) > 2 else 8
m = synth.random_model((r, r, r), (20, 20, 20), 8, seed=1)
pts = synth.uniform_points(1_200_000, 3, seed=2)
vals = np.sin(pts[:, 0]) + pts[:, 1] * pts[:, 2]
F.reestimate_core(m, pts[:50000], vals[:50000], seed=1, transform=t)
_lib.profile_read()
_lib.profile_enable(True)
t0 = time.perf_counter()
new, info = F.reestimate_core(m, pts, vals, seed=1, transform=t, sample_rows=8 * r ** 3)
dt = time.perf_counter() - t0
_lib.profile_enable(False)
prof = _lib.profile_read()
cols = r ** 3 + 1
ms, n = prof["transform"]
print(f"{t} r={r}: total {dt:.3f}s transform {ms:.1f} ms over {n} launches = {ms / cols * 1e3:.1f} us/column",
      info["timings"])
