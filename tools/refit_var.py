"""Dev tool: per-stage times of repeated C2 refits (run-to-run variance).
usage: python tools/refit_var.py [runs]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1907_05884_b200 as F
from bench import workload
from paper_1907_05884_b200.dist import refine_distributed

from paper_1907_05884_b200 import _lib

if "FSTK_DEVICE_CACHE" not in os.environ:
    _lib.set_device_cache(2)  # as bench.py: blocks stay cached between the sessions
model, pts, vals, c = workload("C2", 0, 0)
R = int(np.prod(model.ranks))
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s = F.RefitSession(model, pts, vals, seed=0, sample_rows=c["m_factor"] * R)
    t1 = time.perf_counter()
    g = torch.empty(R * R, dtype=torch.float64, device="cuda")
    rhs = torch.empty(R, dtype=torch.float64, device="cuda")
    s.normal_equations(g, rhs)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    x = refine_distributed(s, g, rhs)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    s.finish(x)
    t4 = time.perf_counter()
    tm = s.info_dict()["timings"]
    print(f"run {i}: total {t4 - t0:.3f}  begin {t1 - t0:.3f}  gram {t2 - t1:.3f}  refine {t3 - t2:.3f}  "
          f"finish {t4 - t3:.3f} | dev prepare {tm['prepare_s']:.3f} sketch {tm['sketch_s']:.3f} "
          f"gram {tm['gram_s']:.3f} solve {tm['solve_s']:.3f} steps {s.info_dict()['refine_steps']}",
          flush=True)
    s.close()
    del g
