"""Profiling driver (dev tool): C2-shaped evaluation on device-resident points.
usage: python tools/prof_eval.py [n_log2] [reps] [config]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1907_05884_b200 import synth

n = 1 << int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 21
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = sys.argv[3] if len(sys.argv) > 3 else "C2"
c = synth.CONFIGS[cfg]
m = synth.random_model(c["ranks"], c["degrees"], c["nnz"], seed=1)
pts = torch.rand(c["d"], n, dtype=torch.float64, device="cuda")
out = torch.empty(n, dtype=torch.float64, device="cuda")
for _ in range(reps):
    m.evaluate_device(pts, out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    m.evaluate_device(pts, out)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
print(f"{cfg} n={n}: {ms:.3f} ms/step, {n / ms * 1e3:.3e} pts/s")
