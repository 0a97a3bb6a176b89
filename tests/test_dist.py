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


# ---- refine_distributed control flow (sliced-Gram fallback), CPU-only -------
class _ScriptedSession:
    """Stands in for RefitSession: factor() outcomes and refinement step sizes
    follow a script, and every call is logged, so the escalation logic of
    dist.refine_distributed can be checked without a GPU."""

    def __init__(self, factor_ok, steps, slices=5, certified=True, deficient=False):
        import types

        self.factor_ok = list(factor_ok)
        self.steps = list(steps)
        self.calls = []
        self.certified = certified
        self.deficient = deficient
        self.R = 1
        self.info = types.SimpleNamespace(refine_steps=0, gram_slices=slices, rank_deficient=0,
                                          qr_path=0)

    def certify(self, gram):
        self.calls.append("certify")
        return self.certified

    def local_qr(self, raug):
        self.calls.append("local_qr")
        raug.fill_(float(len(self.calls)))

    def qr_solve(self, raug, x):
        self.calls.append("qr_solve")
        x.fill_(7.0)
        return self.deficient

    def factor(self, gram, rhs, x):
        self.calls.append("factor")
        return self.factor_ok.pop(0)

    def normal_equations_level(self, slices, gram, rhs):
        self.calls.append(f"upgrade{slices}" if slices else "native")

    def correction(self, x, s):
        self.calls.append("correction")

    def apply(self, s, x):
        self.calls.append("apply")
        return self.steps.pop(0)


def _refine(sess, used=None):
    import torch

    from paper_1907_05884_b200 import dist

    g, r = torch.zeros(4, dtype=torch.float64), torch.zeros(2, dtype=torch.float64)
    return dist.refine_distributed(sess, g, r, used=used)


def test_refine_converges_at_rounding_floor_without_escalation():
    # Contracting 125x in the second step, the extrapolated remainder (6e-14)
    # stays above the done floor; the third step is flat below the stall
    # floor: converged at the rounding floor.
    s = _ScriptedSession([True], [1e-9, 8e-12, 6e-12])
    _refine(s)
    assert "native" not in s.calls and "upgrade7" not in s.calls and s.info.refine_steps == 3


def test_refine_stops_by_extrapolation():
    # rho = 2e-4: the error left after the second step (~4e-17) is below the
    # done floor, so no third pass over A is made.
    s = _ScriptedSession([True], [1e-9, 2e-13, 1.5e-13])
    _refine(s)
    assert "native" not in s.calls and "upgrade7" not in s.calls and s.info.refine_steps == 2
    assert s.calls[-1] == "certify"


def test_refine_not_pd_escalates_upgrade_then_native():
    s = _ScriptedSession([False, False, True], [1e-9, 1e-16])
    _refine(s)
    assert s.calls[:5] == ["factor", "upgrade7", "factor", "native", "factor"]


def test_refine_slow_contraction_upgrades_once():
    s = _ScriptedSession([True, True], [1e-3, 5e-4, 1e-9, 1e-16])
    _refine(s)
    assert s.calls.count("upgrade7") == 1 and "native" not in s.calls
    assert s.calls.count("apply") == 4


def test_refine_seven_planes_go_straight_to_native():
    s = _ScriptedSession([True, True], [1e-3, 9e-4, 1e-9, 1e-16], slices=7)
    _refine(s)
    assert "upgrade7" not in s.calls and s.calls.count("native") == 1


def test_refine_native_stall_does_not_loop():
    # No contraction on the native Gram: only the pivoted QR can decide.
    s = _ScriptedSession([True], [1e-3, 9e-4], deficient=True)
    x = _refine(s, used=0)
    assert "native" not in s.calls and s.calls.count("apply") == 2
    assert s.calls[-2:] == ["local_qr", "qr_solve"] and "certify" not in s.calls
    assert s.info.rank_deficient == 1 and float(x[0]) == 7.0


def test_refine_converged_certified_skips_qr():
    s = _ScriptedSession([True], [1e-9, 1e-16])
    _refine(s)
    assert s.calls[-1] == "certify" and "local_qr" not in s.calls
    assert s.info.rank_deficient == 0


def test_refine_converged_uncertified_goes_to_qr():
    s = _ScriptedSession([True], [1e-9, 1e-16], certified=False)
    _refine(s)
    assert s.calls[-3:] == ["certify", "local_qr", "qr_solve"] and s.info.qr_path == 1


def test_refine_native_not_pd_goes_to_qr():
    s = _ScriptedSession([False], [], slices=0)
    _refine(s, used=0)
    assert s.calls == ["factor", "local_qr", "qr_solve"]


def test_refine_fast_contraction_keeps_five_planes():
    # 2e5x per step: the second step's extrapolated remainder ends it.
    s = _ScriptedSession([True], [1e-6, 1e-11 * 0.5, 1e-16])
    _refine(s)
    assert s.calls.count("apply") == 2 and "upgrade7" not in s.calls


def _gloo_refine_worker(rank, world, port, q):
    import os

    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # Rank 1 holds no sampled rows (gram_slices 0); the max over ranks
        # still selects the sliced ladder on both ranks.
        s = _ScriptedSession([False, True], [1e-9, 1e-16], slices=5 if rank == 0 else 0)
        _refine(s)
        q.put((rank, s.calls))
    finally:
        dist.destroy_process_group()


def _gloo_qr_worker(rank, world, port, q):
    import os

    import torch.distributed as dist

    from paper_1907_05884_b200 import dist as D

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    stacked = []
    D.refit_qr_stack = lambda top, other: stacked.append(float(other[0]))
    try:
        # Only rank 1 fails the certificate: every rank still takes the QR
        # path, rank 0 stacks rank 1's factor, and x / the flag come from rank 0.
        s = _ScriptedSession([True], [1e-9, 1e-16], certified=(rank == 0), deficient=True)
        x = _refine(s)
        q.put((rank, s.calls, stacked, float(x[0]), s.info.rank_deficient))
    finally:
        dist.destroy_process_group()


def test_refine_qr_decision_agrees_across_gloo_ranks():
    import multiprocessing as mp
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_gloo_qr_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = {r: rest for r, *rest in (q.get(timeout=120) for _ in ps)}
    for p in ps:
        p.join(timeout=60)
    calls0, st0, x0, d0 = out[0]
    calls1, st1, x1, d1 = out[1]
    assert calls0[-3:] == ["certify", "local_qr", "qr_solve"]
    assert calls1[-2:] == ["certify", "local_qr"]  # rank 1 only contributes its factor
    assert len(st0) == 1 and st1 == []
    assert x0 == x1 == 7.0 and d0 == d1 == 1


def test_refine_escalation_agrees_across_gloo_ranks():
    import multiprocessing as mp
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_gloo_refine_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert out[0] == out[1] and out[0][:3] == ["factor", "upgrade7", "factor"]
