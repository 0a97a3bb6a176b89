"""Dev diagnostic: sliced vs native Gram on one refit system.
usage: python tools/gram_diag.py [config] [slices] [max_points]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1907_05884_b200 as F
from paper_1907_05884_b200 import synth

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
ns = int(sys.argv[2]) if len(sys.argv) > 2 else 7
from bench import workload

model, pts, vals, c = workload(cfg, 0, 0)
R = int(np.prod(model.ranks))
S = c["m_factor"] * R
dev = torch.device("cuda", 0)
sess = F.RefitSession(model, pts, vals, seed=0, sample_rows=S, transform="dct")
G = {}
for name, slices in (("native", 0), ("sliced", ns)):
    F.gram_slices(slices)
    g = torch.empty(R * R, dtype=torch.float64, device=dev)
    r = torch.empty(R, dtype=torch.float64, device=dev)
    sess.normal_equations(g, r)
    torch.cuda.synchronize()
    print(name, "gram_s", sess.info.t_gram, "slices", sess.info.gram_slices, flush=True)
    G[name] = (g, r)
gn = G["native"][0].view(R, R).t()  # row-major view: gn[a, b] = G[a + b R] -> column b, row a
gs = G["sliced"][0].view(R, R).t()
low = torch.tril(torch.ones(R, R, dtype=torch.bool, device=dev))
dn = torch.sqrt(torch.diagonal(gn).clamp_min(1e-300))
scale = dn[:, None] * dn[None, :]
diff = ((gs - gn).abs() / scale)[low]
print("diag min/max", float(torch.diagonal(gn).min()), float(torch.diagonal(gn).max()))
print("max scaled |Gs-Gn|", float(diff.max()), "mean", float(diff.mean()))
print("rel fro", float(torch.linalg.norm((gs - gn)[low]) / torch.linalg.norm(gn[low])))
print("rhs rel", float(torch.linalg.norm(G["sliced"][1] - G["native"][1]) / torch.linalg.norm(G["native"][1])))
for name in ("native", "sliced"):
    g, r = G[name]
    x = torch.empty_like(r)
    ok = sess.factor(g, r, x)
    print(name, "factor ok", ok, flush=True)
    if not ok:
        continue
    s = torch.empty_like(r)
    steps = []
    for it in range(10):
        sess.correction(x, s)
        steps.append(sess.apply(s, x))
    print(name, "steps", ["%.2e" % v for v in steps], flush=True)
sess.close()
