"""Dev tool: the C4 refit at full shape on one GPU (4D, ranks (16,16,16,8) so
R = 32,768, M = 16R = 524,288 sketch rows: A is 137 GB), on a planted model:
values = the model with a known core, so the refit must return that core.
usage: python tools/c4_refit.py [n_points] [transform] [layout shards]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_1907_05884_b200 as F
from paper_1907_05884_b200 import synth

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 22
tr = sys.argv[2] if len(sys.argv) > 2 else "dct"
c = synth.CONFIGS["C4"]
m = synth.random_model(c["ranks"], c["degrees"], c["nnz"], seed=0)
pts = synth.uniform_points(n, 4, seed=1)
vals = m.evaluate_batch(pts)  # noise-free: the planted core is the LS solution
R = int(np.prod(m.ranks))
S = c["m_factor"] * R
shuffled = np.random.default_rng(2).permutation(m.core.reshape(-1, order="F"))
start = m.with_core(shuffled.reshape(m.ranks, order="F"))  # refit from a wrong core
t0 = time.perf_counter()
new, info = F.reestimate_core(start, pts, vals, seed=3, sample_rows=S, transform=tr)
dt = time.perf_counter() - t0
want = m.core.reshape(-1, order="F")
got = new.core.reshape(-1, order="F")
rel = np.linalg.norm(got - want) / np.linalg.norm(want)
print(f"C4 refit {tr}: R={R} S={S} q={n}: {dt:.2f} s, core rel err {rel:.3e}, "
      f"residual_after {info['residual_after']:.3e}, gram level {info['gram_slices']}, "
      f"steps {info['refine_steps']}, timings {info['timings']}", flush=True)
