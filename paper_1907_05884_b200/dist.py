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


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block [lo, hi) of n items owned by `rank` (same rule the
    library uses for sampled rows: floor(n*r/w))."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    return n * rank // world, n * (rank + 1) // world


def reduce_normal_equations(gram, rhs, group=None):
    """Sum per-rank partial normal equations in place (one collective each)."""
    import torch.distributed as dist

    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(gram, group=group)
        dist.all_reduce(rhs, group=group)
    return gram, rhs


def evaluate_sharded(model, points, rank: int, world: int):
    """Evaluates this rank's slab of `points` (Q x d); returns (lo, hi, values)."""
    lo, hi = shard_range(points.shape[0], rank, world)
    return lo, hi, model.evaluate_batch(np.asfortranarray(points[lo:hi]))


STALL_FLOOR = 1e-11  # ||dx||/||x|| below which a flat refinement has converged


def refine_distributed(sess, gram, rhs, max_iter: int = 8, group=None, sliced=None):
    """Cholesky of the summed Gram on every rank, then iterative refinement
    against the row-sharded sketch: each step needs one all-reduce of an
    R-vector.  Returns the solution tensor x (identical on all ranks).

    With the sliced int8 Gram (fstk_gpu_gram_slices > 0) a Gram that is not
    positive definite, or refinement that stops contracting, is redone once
    with the native fp64 Gram (fstk_refit.cu: fstk_gpu_refit_solve does the
    same on one GPU).  Both decisions depend only on all-reduced data, so
    every rank takes the same branch."""
    import torch
    import torch.distributed as dist

    x = torch.empty_like(rhs)
    if sliced is None:
        from .refit import gram_slices

        sliced = gram_slices() > 0

    def native():
        sess.normal_equations_native(gram, rhs)
        reduce_normal_equations(gram, rhs, group=group)
        return sess.factor(gram, rhs, x)

    sess.info.refine_steps = 0
    ok = sess.factor(gram, rhs, x)
    if not ok and sliced:
        ok, sliced = native(), False
    if not ok:
        return x
    s = torch.empty_like(rhs)
    prev = float("inf")
    it = 0
    while it < max_iter:
        sess.correction(x, s)
        if dist.is_initialized() and dist.get_world_size(group) > 1:
            dist.all_reduce(s, group=group)
        step = sess.apply(s, x)
        sess.info.refine_steps += 1
        if step <= 1e-15:
            break
        # Flat at the rounding floor is convergence (see fstk_gpu_refit_solve).
        flat = it >= 1 and step > 0.5 * prev
        if flat and step <= STALL_FLOOR:
            break
        if flat or (sliced and it == max_iter - 1 and step > STALL_FLOOR):
            if not sliced:
                break
            ok, sliced = native(), False
            if not ok:
                break
            prev, it = float("inf"), 0
            continue
        prev = step
        it += 1
    return x


def refit_distributed(model, points, values, rank: int, world: int, device=None, **kw):
    """Row-sharded refit: returns (new_model, info) on rank 0, (None, info) elsewhere."""
    import torch
    import torch.distributed as dist

    from .refit import RefitSession

    R = int(np.prod(model.ranks))
    sess = RefitSession(model, points, values, shard=rank, shards=world, device=device, **kw)
    dev = torch.device("cuda", device if device is not None else torch.cuda.current_device())
    gram = torch.empty(R * R, dtype=torch.float64, device=dev)
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
