"""Multi-process host logic on CPU (gloo, world_size 2): the point/row
sharding rule and the single all-reduce of partial normal equations
reproduce the single-rank result.  The sketched system comes from the oracle
(the checker) so no GPU is needed."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1907_05884_b200.dist import reduce_normal_equations, shard_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, a, b, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard_range(a.shape[0], rank, world)
    g = torch.from_numpy(a[lo:hi].T @ a[lo:hi]).contiguous()
    r = torch.from_numpy(a[lo:hi].T @ b[lo:hi]).contiguous()
    reduce_normal_equations(g, r)
    out[rank] = (g.numpy().copy(), r.numpy().copy())
    dist.barrier()
    dist.destroy_process_group()


def test_shard_range_partitions():
    for n in (0, 1, 7, 262144, 1 << 20):
        for w in (1, 2, 3, 8):
            spans = [shard_range(n, r, w) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(w - 1))
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def test_gloo_world2_normal_equations_allreduce(O):
    from _models import legendre_model, random_points

    m = legendre_model((3, 2, 2), 5)
    pts = random_points(3000, 3, 7)
    vals = O.evaluate_batch(m, pts) + 0.01 * np.random.default_rng(1).normal(size=3000)
    a, b, rows, _, _ = O.refit_system(m, pts, vals, seed=3)
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), a, b, out), nprocs=world, join=True)
    full_g, full_r = a.T @ a, a.T @ b
    for r in range(world):
        g, rr = out[r]
        assert np.abs(g - full_g).max() <= 1e-12 * np.abs(full_g).max()
        assert np.abs(rr - full_r).max() <= 1e-12 * np.abs(full_r).max()
    # solving the reduced system reproduces the oracle's QR solution
    alpha = np.linalg.solve(out[0][0], out[0][1])
    want, _ = O.solve_system(a, b)
    assert np.linalg.norm(alpha - want) <= 1e-9 * np.linalg.norm(want)
