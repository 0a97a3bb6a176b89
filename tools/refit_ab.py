"""Dev tool: C2 refits alternating the Gram engines (tcgen05 SYRK vs
cuBLASLt), per-stage device timings of each.
usage: python tools/refit_ab.py [reps] [config]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1907_05884_b200 as F
from bench import workload

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cfg = sys.argv[2] if len(sys.argv) > 2 else "C2"
model, pts, vals, c = workload(cfg, 0, 0)
R = int(np.prod(model.ranks))
F.reestimate_core(model, pts, vals, seed=0, sample_rows=c["m_factor"] * R)  # warm-up
for i in range(reps):
    for eng in ("tcgen05", "cublaslt"):
        F.gram_engine(eng)
        time.sleep(2)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        new, info = F.reestimate_core(model, pts, vals, seed=0, sample_rows=c["m_factor"] * R)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        tm = info.get("timings", {})
        print(f"{eng:9s} {dt:.3f} s  " + " ".join(f"{k}={v:.3f}" for k, v in tm.items() if isinstance(v, float))
              + f"  steps={info.get('refine_steps')} res={info.get('residual_after'):.12g}", flush=True)
