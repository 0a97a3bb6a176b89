"""Multi-GPU plumbing: one process per GPU, torch.distributed (NCCL on GPUs,
gloo in the CPU tests).  SURVEY §8e:

* evaluation shards points into contiguous slabs, no collective on the data
  path (the caller owns each slab's output);
* the refit is one problem: every rank runs the (cheap, bit-identical) host
  plan and the sketch, keeps its contiguous block of sampled rows, forms its
  partial A^T A / A^T b, and ONE all-reduce sums them; rank 0 solves.
"""
from __future__ import annotations

import numpy as np

from . import _lib


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block [lo, hi) of n items owned by `rank` (same rule the
    library uses for sampled rows: floor(n*r/w))."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    return n * rank // world, n * (rank + 1) // world


def reduce_normal_equations(gram, rhs, group=None):
    """Sum per-rank partial normal equations in place with ONE all-reduce of
    the packed lower triangle plus the right-hand side (R(R+1)/2 + R values,
    SURVEY 8e: 4.3 GB at R = 32,768 instead of the 8.6 GB square Gram; the
    solver reads only the lower triangle).  Packing and unpacking run on the
    device (fstk_gpu_pack_normal_equations)."""
    import ctypes as C

    import torch
    import torch.distributed as dist

    if not (dist.is_initialized() and dist.get_world_size(group) > 1):
        return gram, rhs
    n = rhs.numel()
    if gram.device.type != "cuda":  # CPU tensors (tests): the plain collectives
        dist.all_reduce(gram, group=group)
        dist.all_reduce(rhs, group=group)
        return gram, rhs
    packed = _lib.device_tensor(n * (n + 1) // 2 + n, gram.device)
    stream = torch.cuda.current_stream(gram.device).cuda_stream
    err = _lib.Err()
    _lib.check(_lib.lib().fstk_gpu_pack_normal_equations(gram.data_ptr(), rhs.data_ptr(), n,
                                                         packed.data_ptr(), 0, stream,
                                                         C.byref(err)), err)
    buf = _to_backend(packed, group)
    dist.all_reduce(buf, group=group)
    if buf is not packed:
        packed.copy_(buf)
    _lib.check(_lib.lib().fstk_gpu_pack_normal_equations(gram.data_ptr(), rhs.data_ptr(), n,
                                                         packed.data_ptr(), 1, stream,
                                                         C.byref(err)), err)
    del packed
    return gram, rhs


def evaluate_sharded(model, points, rank: int, world: int):
    """Evaluates this rank's slab of `points` (Q x d); returns (lo, hi, values)."""
    lo, hi = shard_range(points.shape[0], rank, world)
    return lo, hi, model.evaluate_batch(np.asfortranarray(points[lo:hi]))


STALL_FLOOR = 1e-11  # ||dx||/||x|| below which a flat refinement has converged
DONE_FLOOR = 1e-14   # extrapolated remaining ||dx||/||x|| that ends the refinement (kDoneFloor)
UPGRADE_SLICES = 7   # escalation target of a sliced Gram before the native one


def _max_over_ranks(v: int, group=None) -> int:
    import torch
    import torch.distributed as dist

    if not (dist.is_initialized() and dist.get_world_size(group) > 1):
        return int(v)
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor([int(v)], dtype=torch.int64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return int(t.item())


def _max_over_ranks_f(v: float, group=None) -> float:
    import torch
    import torch.distributed as dist

    if not (dist.is_initialized() and dist.get_world_size(group) > 1):
        return float(v)
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor([float(v)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def _to_backend(t, group=None):
    """Tensor as the backend moves it (NCCL: the CUDA tensor; gloo: a host copy)."""
    import torch.distributed as dist

    return t if dist.get_backend(group) == "nccl" else t.cpu()


def qr_decide_distributed(sess, x, group=None):
    """The reference's rank decision (randls.cpp:112-123) for a row-sharded
    sketch: every rank folds its rows into R of [A b] (streaming TSQR), rank 0
    stacks the factors in rank order (fstk_gpu_qr_stack), runs the pivoted QR
    with Eigen's threshold and solves (QR or COD), and broadcasts x and the
    flag.  Returns rank_deficient (same on every rank)."""
    import torch
    import torch.distributed as dist

    n1 = sess.R + 1
    raug = _lib.device_tensor(n1 * n1, x.device)
    sess.local_qr(raug)
    multi = dist.is_initialized() and dist.get_world_size(group) > 1
    rank = dist.get_rank(group) if multi else 0
    if multi:
        world = dist.get_world_size(group)
        if rank == 0:
            other = _lib.device_tensor(n1 * n1, x.device)
            for src in range(1, world):
                buf = _to_backend(other, group)
                dist.recv(buf, src=src, group=group)
                if buf is not other:
                    other.copy_(buf)
                refit_qr_stack(raug, other)
        else:
            dist.send(_to_backend(raug, group), dst=0, group=group)
    flag = torch.zeros(1, dtype=torch.float64, device=x.device)
    if rank == 0:
        flag[0] = 1.0 if sess.qr_solve(raug, x) else 0.0
    if multi:
        for t in (x, flag):
            buf = _to_backend(t, group)
            dist.broadcast(buf, src=0, group=group)
            if buf is not t:
                t.copy_(buf)
    deficient = bool(flag.item() != 0.0)
    sess.info.rank_deficient = int(deficient)
    sess.info.qr_path = 1
    return deficient


def refit_qr_stack(top, other):
    from .refit import qr_stack

    qr_stack(top, other)


def refine_distributed(sess, gram, rhs, max_iter: int = 8, group=None, used=None):
    """Cholesky of the summed Gram on every rank, then iterative refinement
    against the row-sharded sketch: each step needs one all-reduce of an
    R-vector.  Returns the solution tensor x (identical on all ranks).

    `used` = digit planes of the summed Gram (None: the max over ranks of
    sess.info.gram_slices).  A sliced Gram that is not positive definite, or
    whose refinement contracts slower than 10x per step or stalls, escalates
    like fstk_gpu_refit_solve: the Gram is recomputed (and all-reduced) at
    UPGRADE_SLICES' accuracy, then natively in fp64.  Every decision depends only
    on all-reduced data, so all ranks take the same branch."""
    import torch
    import torch.distributed as dist

    x = torch.empty_like(rhs)
    if used is None:
        used = _max_over_ranks(sess.info.gram_slices, group)

    def escalate():
        nonlocal used
        if used == 0:
            return False
        used = UPGRADE_SLICES if used < UPGRADE_SLICES else 0
        sess.normal_equations_level(used, gram, rhs)
        reduce_normal_equations(gram, rhs, group=group)
        return True

    def factor():
        # A rank whose int8 Cholesky fell back to dpotrf (or failed) must not
        # branch alone: the factored flag is the minimum over ranks.
        ok_local = sess.factor(gram, rhs, x)
        return not bool(_max_over_ranks(int(not ok_local), group))

    def escalate_until_factored():
        while True:
            if not escalate():
                return False
            if factor():
                return True

    sess.info.refine_steps = 0
    ok = factor()
    if not ok:
        ok = escalate_until_factored()
    need_qr = not ok
    s = torch.empty_like(rhs)
    prev = float("inf")
    it = 0
    while ok and it < max_iter:
        sess.correction(x, s)
        if dist.is_initialized() and dist.get_world_size(group) > 1:
            dist.all_reduce(s, group=group)
        # Steps are computed from all-reduced data, but each rank's factor
        # can round differently: branch on the largest.
        step = _max_over_ranks_f(sess.apply(s, x), group)
        sess.info.refine_steps += 1
        if step <= 1e-15:
            break
        # Converged by extrapolation: contracting by rho = step / prev < 0.1, the
        # error left is ~ rho * step (see fstk_gpu_refit_solve).
        if it >= 1 and step < 0.1 * prev and step * (step / prev) <= DONE_FLOOR:
            break
        # Flat at the rounding floor is convergence (see fstk_gpu_refit_solve).
        flat = it >= 1 and step > 0.5 * prev
        if flat and step <= STALL_FLOOR:
            break
        slow = used > 0 and it >= 1 and step > STALL_FLOOR and step > 0.1 * prev
        last = it == max_iter - 1 and step > STALL_FLOOR
        if flat or slow or last:
            if used == 0 or not escalate_until_factored():
                need_qr = True  # no contraction on the native Gram
                break
            prev, it = float("inf"), 0
            continue
        prev = step
        it += 1
    if not need_qr:
        need_qr = not sess.certify(gram)
    if _max_over_ranks(int(need_qr), group):
        qr_decide_distributed(sess, x, group)
    else:
        sess.info.rank_deficient = 0
    return x


def exchange_columns(sess, group=None):
    """Column-to-row all-to-all of a layout='columns' RefitSession (SURVEY
    8e): every rank sent its transformed columns for every row slab; after
    this each rank holds its row slab and the refit continues row-sharded.
    NCCL moves device tensors directly; other backends stage through host
    memory."""
    import torch
    import torch.distributed as dist

    bufs = sess.exchange_buffers()
    if bufs is None:  # transform="none": rows are generated locally
        return
    send, sc, recv, rc = bufs
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        if dist.get_backend(group) == "nccl":
            dist.all_to_all_single(recv, send, output_split_sizes=rc, input_split_sizes=sc,
                                   group=group)
        else:
            hr = torch.empty(recv.numel(), dtype=recv.dtype)
            dist.all_to_all_single(hr, send.cpu(), output_split_sizes=rc, input_split_sizes=sc,
                                   group=group)
            recv.copy_(hr)
    else:
        recv.copy_(send)  # one shard: the packed and row layouts coincide
    torch.cuda.synchronize(recv.device)
    sess.adopt_rows()


def _check_same_dataset(points, values, device=None, group=None):
    """The sharded refit is ONE least-squares problem: every rank must pass
    the same cloud (the host plan indexes it identically on all ranks).  A
    fingerprint of the size and a strided sample is compared across ranks."""
    import torch
    import torch.distributed as dist

    if not (dist.is_initialized() and dist.get_world_size(group) > 1):
        return
    p = np.asarray(points, dtype=np.float64)
    v = np.asarray(values, dtype=np.float64)
    step = max(1, p.shape[0] // 4096)
    fp = np.array([p.shape[0], p.shape[1], float(np.sum(p[::step])), float(np.sum(v[::step]))])
    dev = torch.device("cuda", device if device is not None else torch.cuda.current_device()) \
        if dist.get_backend(group) == "nccl" else torch.device("cpu")
    t = torch.tensor(fp, dtype=torch.float64, device=dev)
    lo, hi = t.clone(), t.clone()
    dist.all_reduce(lo, op=dist.ReduceOp.MIN, group=group)
    dist.all_reduce(hi, op=dist.ReduceOp.MAX, group=group)
    if not torch.equal(lo, hi):
        raise ValueError("refit_distributed: ranks hold different point clouds; the sharded "
                         "refit needs the same dataset on every rank")


def refit_distributed(model, points, values, rank: int, world: int, device=None,
                      layout: str = "columns", **kw):
    """Sharded refit of ONE dataset (identical `points`/`values` on every rank):
    returns (new_model, info) on rank 0, (None, info) elsewhere.
    layout="columns" (default) shards the sketch transform by columns and
    exchanges once (exchange_columns); layout="rows" replicates the transform
    and keeps each rank's rows."""
    import torch
    import torch.distributed as dist

    from .refit import RefitSession

    R = int(np.prod(model.ranks))
    _check_same_dataset(points, values, device)
    sess = RefitSession(model, points, values, shard=rank, shards=world, device=device,
                        layout=layout, **kw)
    if layout == "columns":
        exchange_columns(sess)
    dev = torch.device("cuda", device if device is not None else torch.cuda.current_device())
    gram = _lib.device_tensor(R * R, dev)
    rhs = torch.empty(R, dtype=torch.float64, device=dev)
    sess.normal_equations(gram, rhs)
    reduce_normal_equations(gram, rhs)
    x = refine_distributed(sess, gram, rhs)
    new = None
    if rank == 0:
        core = sess.finish(x)
        new = model.with_core(core)
    info = sess.info_dict()
    sess.close()
    if dist.is_initialized():
        dist.barrier()
    return new, info
