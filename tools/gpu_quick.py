"""Quick GPU bring-up check (dev tool): product vs oracle on small cases + timing."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1907_05884_b200 as F
from paper_1907_05884_b200 import synth
from oracle import oracle as O

def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)

for ranks, deg, nnz in [((3, 2, 4), (5, 5, 5), 3), ((16, 16, 16), (20, 20, 20), 12), ((32, 32, 32), (48, 48, 48), 24),
                         ((48, 48, 32), (64, 64, 64), 24), ((16, 16, 16, 8), (32, 32, 32, 16), 12), ((5,), (7,), 4), ((7, 9), (6, 6), 5)]:
    m = synth.random_model(ranks, deg, nnz, seed=1)
    pts = synth.uniform_points(5000, len(ranks), seed=2)
    g = m.evaluate_batch(pts)
    o = O.evaluate_batch(m, pts)
    mv_g = m.mode_values(0, pts[:, 0])
    mv_o = np.stack([O.mode_values(m, 0, x) for x in pts[:200, 0]])
    print(ranks, "eval rel", rel(g, o), "mode bitexact", np.array_equal(mv_g[:200], mv_o), flush=True)

# sketch bit-exactness
rng = np.random.default_rng(0)
for t in ("dct", "wht", "fft"):
    for q in (24, 100, 3000, 70000):
        w = rng.random((q, 6)); u = rng.random(q)
        s = min(40, q)
        a1, b1, p1 = F.sketch(w, u, seed=5, sample_rows=s, transform=t)
        a2, b2, p2 = O.sketch(w, u, seed=5, sample_rows=s, transform=t)
        print("sketch", t, q, "bitexact A", np.array_equal(a1, a2), "b", np.array_equal(b1, b2), "maxdiff", np.abs(a1-a2).max(), flush=True)

# refit parity small
m = synth.random_model((4, 3, 2), (5, 5, 5), 3, seed=3)
pts = synth.uniform_points(20000, 3, seed=4)
vals = O.evaluate_batch(m, pts) + 0.01 * rng.normal(size=20000)
for t in ("dct", "wht", "fft"):
    m2, info = F.reestimate_core(m, pts, vals, seed=17, transform=t)
    c_o, info_o = O.reestimate_core(m, pts, vals, seed=17, transform=t)
    print("refit", t, "core rel", rel(m2.core.reshape(-1, order="F"), c_o), info["residual_after"], info_o["residual_after"], flush=True)
    sess = F.RefitSession(m, pts, vals, seed=17, transform=t)
    a, b = sess.sketched()
    ao, bo, rows_o, vi, _ = O.refit_system(m, pts, vals, seed=17, transform=t)
    print("   rows bitexact", np.array_equal(sess.rows(), rows_o), "A bitexact", np.array_equal(a, ao), "b", np.array_equal(b, bo), flush=True)
    sess.close()

# timing C2-shaped eval
import torch
m = synth.random_model((32, 32, 32), (48, 48, 48), 24, seed=1)
n = 1 << 24
pts = torch.rand(3, n, dtype=torch.float64, device="cuda")
out = torch.empty(n, dtype=torch.float64, device="cuda")
for _ in range(3): m.evaluate_device(pts, out)
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5): m.evaluate_device(pts, out)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print(f"C2 eval: {ms:.2f} ms per 16M pts -> {n/ms*1e3:.3e} pts/s, {n*73120/ms/1e9:.2f} TFLOP/s", flush=True)
print("launches", F.launch_count())
