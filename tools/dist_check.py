"""Multi-rank refit/eval check on ONE GPU (dev tool): run with
  torchrun --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 tools/dist_check.py
Ranks share the device and talk through gloo (host-mediated), so no kernel
waits on another rank's kernel.  Compares the row-sharded refit (one
all-reduce of A^T A, sharded refinement) with the single-GPU refit."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist

import paper_1907_05884_b200 as F
from paper_1907_05884_b200 import dist as D
from paper_1907_05884_b200 import synth

dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(0)
m = synth.random_model((8, 6, 5), (10, 9, 8), 5, seed=3)
pts = synth.uniform_points(60_000, 3, seed=4)
vals = np.sin(3 * pts[:, 0]) + pts[:, 1] * pts[:, 2] + 0.01 * np.random.default_rng(5).normal(size=60_000)
new, info = D.refit_distributed(m, pts, vals, rank, world, device=0, seed=11)
lo, hi, part = D.evaluate_sharded(m, pts, rank, world)
full = m.evaluate_batch(pts)
assert np.array_equal(part, full[lo:hi]), "sharded evaluation differs"
if rank == 0:
    ref, info1 = F.reestimate_core(m, pts, vals, seed=11)
    a, b = new.core.reshape(-1, order="F"), ref.core.reshape(-1, order="F")
    rel = np.linalg.norm(a - b) / np.linalg.norm(b)
    print(f"world={world}: sharded refit vs single-GPU core rel {rel:.2e}; residual_after "
          f"{info['residual_after']:.6e} vs {info1['residual_after']:.6e}", flush=True)
    assert rel <= 1e-10, rel
dist.barrier()
dist.destroy_process_group()
