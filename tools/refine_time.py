"""Dev tool: wall time of every stage call of the C2 refit's solve
(factor / correction / apply / certify) as dist.refine_distributed issues them
on one GPU, to locate the host time between the device-timed stages.
usage: python tools/refine_time.py [reps] [transform]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1907_05884_b200 as F
from bench import workload
from paper_1907_05884_b200 import _lib

model, pts, vals, c = workload("C2", 0, 0)
R = int(np.prod(model.ranks))
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    s = F.RefitSession(model, pts, vals, seed=0, sample_rows=c["m_factor"] * R,
                       transform=sys.argv[2] if len(sys.argv) > 2 else "dct")
    g = _lib.device_tensor(R * R, "cuda")
    rhs = torch.empty(R, dtype=torch.float64, device="cuda")
    s.normal_equations(g, rhs)
    torch.cuda.synchronize()
    x = torch.empty_like(rhs)
    sv = torch.empty_like(rhs)
    marks = []

    def t(name, f):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = f()
        torch.cuda.synchronize()
        marks.append((name, time.perf_counter() - t0))
        return r

    t0 = time.perf_counter()
    t("factor", lambda: s.factor(g, rhs, x))
    steps = []
    for it in range(8):
        t(f"correction{it}", lambda: s.correction(x, sv))
        step = t(f"apply{it}", lambda: s.apply(sv, x))
        steps.append(step)
        if step <= 1e-11 or (it >= 1 and step > 0.5 * steps[-2]):
            break
    print("   steps ||dx||/||x||: " + " ".join(f"{v:.2e}" for v in steps), flush=True)
    t("certify", lambda: s.certify(g))
    tot = time.perf_counter() - t0
    print(f"rep {rep}: total {tot:.3f} s; " + ", ".join(f"{n} {v * 1e3:.1f} ms" for n, v in marks), flush=True)
    s.close()
    del g
