"""Dev check: sliced int8 Gram vs native fp64 Gram on one refit.
usage: python tools/gram_check.py [r] [n_points] [transform] [slices...]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_1907_05884_b200 as F
from paper_1907_05884_b200 import synth

r = int(sys.argv[1]) if len(sys.argv) > 1 else 16
npts = int(sys.argv[2]) if len(sys.argv) > 2 else 1_200_000
tr = sys.argv[3] if len(sys.argv) > 3 else "dct"
slices = [int(a) for a in sys.argv[4:]] or [0, 7, 6, 5]
m = synth.random_model((r, r, r), (24, 24, 24), 12, seed=1)
pts = synth.uniform_points(npts, 3, seed=2)
vals = synth.flame_field(pts, seed=3)
F.gram_slices(0)
F.reestimate_core(m, pts[:50000], vals[:50000], seed=1, transform=tr)
ref = None
for ns in slices:
    F.gram_slices(ns)
    t0 = time.perf_counter()
    new, info = F.reestimate_core(m, pts, vals, seed=1, transform=tr, sample_rows=8 * r ** 3)
    dt = time.perf_counter() - t0
    core = np.asarray(new.core).ravel()
    if ref is None:
        ref = core
    rel = np.linalg.norm(core - ref) / np.linalg.norm(ref)
    tm = info["timings"]
    print(f"r={r} ns={ns}: total {dt:.3f}s gram {tm['gram_s']:.3f}s solve {tm['solve_s']:.3f}s "
          f"sketch {tm['sketch_s']:.3f}s used={info['gram_slices']} steps={info['refine_steps']} "
          f"rankdef={info['rank_deficient']} rel_vs_native={rel:.3e} res={info['residual_after']:.6e}",
          flush=True)
