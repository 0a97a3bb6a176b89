"""Multi-rank paths on ONE GPU: two ranks share the device and talk through
gloo (host-mediated; no kernel waits on another rank's kernel).  The
row-sharded refit (one all-reduce of A^T A, sharded refinement with an
R-vector all-reduce per step) must equal the single-GPU refit, and sharded
evaluation must equal the full evaluation bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist

    from paper_1907_05884_b200 import dist as D
    from paper_1907_05884_b200 import synth

    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    m = synth.random_model((8, 6, 5), (10, 9, 8), 5, seed=3)
    pts = synth.uniform_points(60_000, 3, seed=4)
    vals = np.sin(3 * pts[:, 0]) + pts[:, 1] * pts[:, 2]
    new, info = D.refit_distributed(m, pts, vals, rank, world, device=0, seed=11, transform="wht")
    lo, hi, part = D.evaluate_sharded(m, pts, rank, world)
    out[rank] = (lo, hi, part, None if new is None else new.core, info["residual_after"])
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_one_gpu_refit_and_eval():
    import paper_1907_05884_b200 as F
    from paper_1907_05884_b200 import synth

    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _port(), out), nprocs=2, join=True)
    m = synth.random_model((8, 6, 5), (10, 9, 8), 5, seed=3)
    pts = synth.uniform_points(60_000, 3, seed=4)
    vals = np.sin(3 * pts[:, 0]) + pts[:, 1] * pts[:, 2]
    ref, info = F.reestimate_core(m, pts, vals, seed=11, transform="wht")
    core = out[0][3]
    rel = np.linalg.norm(core - ref.core) / np.linalg.norm(ref.core)
    assert rel <= 1e-10
    full = m.evaluate_batch(pts)
    for r in range(2):
        lo, hi, part, _, _ = out[r]
        assert np.array_equal(part, full[lo:hi])
    assert out[0][4] == pytest.approx(info["residual_after"], rel=1e-9)
