"""Randomized least-squares core refit through the B200 C-ABI.

Python surface mirrors proj/python/module.cpp:271-294 (`reestimate_core`
returning (model, info)) and the diagnostics of proj/include/fstk/randls.hpp
(build_design_rows, sketch, mixed_matrix).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import (TRANSFORMS, Err, ReestimateInfo, SketchCfg, check, dptr, lib, make_error,
                   require_gpu)
from .model import Model


def sketch_config(seed=0, sample_rows=0, working_subset=1 << 20, transform="dct",
                  validation_fraction=0.05) -> SketchCfg:
    """module.cpp:83-102 (sketch_from_kwargs)."""
    if transform not in TRANSFORMS:
        raise make_error(1, "transform must be dct, wht, fft or none")
    return SketchCfg(int(seed), int(working_subset), int(sample_rows), TRANSFORMS[transform],
                     float(validation_fraction))


def _cloud(model: Model, points, values):
    p = np.asarray(points, dtype=np.float64)
    v = np.asarray(values, dtype=np.float64)
    if p.ndim != 2:
        raise make_error(1, "points must be a 2-D array")
    if v.ndim != 1:
        raise make_error(1, "values must be a 1-D array")
    if p.shape[0] != v.shape[0]:
        raise make_error(2, "point/value count mismatch")
    return np.asfortranarray(p), np.ascontiguousarray(v)


def _info_dict(info: ReestimateInfo) -> dict:
    return {"residual_before": info.residual_before, "residual_after": info.residual_after,
            "sample_rows": int(info.sample_rows), "working_rows": int(info.working_rows),
            "rank_deficient": bool(info.rank_deficient), "held_out": bool(info.held_out),
            "padded_rows": int(info.padded_rows), "gram_slices": int(info.gram_slices),
            "refine_steps": int(info.refine_steps), "gram_int8_ops": float(info.gram_int8_ops),
            "qr_path": bool(info.qr_path), "sigma_ratio": float(info.sigma_ratio),
            "devices": max(1, int(info.devices)),
            "transport": {0: None, 1: "nccl", 2: "p2p"}.get(int(info.multi_transport)),
            "timings": {"prepare_s": info.t_prepare, "sketch_s": info.t_sketch,
                        "gram_s": info.t_gram, "solve_s": info.t_solve,
                        "residual_s": info.t_residual, "alloc_s": info.t_alloc,
                        "exchange_s": info.t_exchange, "reduce_s": info.t_reduce}}


def gram_slices(slices: int | None = None) -> int:
    """Gram arithmetic of this process: returns the current precision level
    (the accuracy of that many 7-bit planes, 4..7; 3 and 2 = 23- and 19-bit
    entries on 8 and 7 CRT moduli, 2 being the default; 0 = native fp64 Gram); with
    `slices` given, sets it first and returns the previous value.  See
    fstk_gram.cu."""
    return int(lib().fstk_gpu_gram_slices(-1 if slices is None else int(slices)))


def gram_engine(engine: str | None = None) -> str:
    """Int8 GEMM engine of the CRT Gram: "tcgen05" (the hand-written sm_100a
    SYRK in fstk_syrk.cu, default) or "cublaslt" (library IMMA GEMMs, kept for
    comparison).  Returns the current engine; with `engine` given, sets it
    first and returns the previous one.  Both give the identical Gram."""
    names = {1: "tcgen05", 2: "cublaslt"}
    code = {"tcgen05": 1, "cublaslt": 2}
    if engine is not None and engine not in code:
        raise ValueError(f"gram engine must be one of {sorted(code)}")
    return names[int(lib().fstk_gpu_gram_engine(0 if engine is None else code[engine]))]


def gram(a, slices: int | None = None):
    """Lower triangle of A^T A for a CUDA float64 tensor A (rows x n) through
    fstk_gpu_gram_device; `slices` digit planes (default: the process
    setting, 0 = native fp64).  Returns an n x n CUDA tensor (upper triangle
    of the column-major result left zero)."""
    import torch

    if not (isinstance(a, torch.Tensor) and a.is_cuda and a.dtype == torch.float64 and a.dim() == 2):
        raise TypeError("gram: expected a 2-D CUDA float64 tensor")
    rows, n = a.shape
    at = a.t().contiguous()  # column-major A: column j at j * rows
    g = _lib.device_tensor(n * n, a.device, zero=True)
    ns = gram_slices() if slices is None else int(slices)
    err = Err()
    stream = torch.cuda.current_stream(a.device).cuda_stream
    check(lib().fstk_gpu_gram_device(at.data_ptr(), rows, rows, n, g.data_ptr(), ns,
                                     a.device.index, stream, C.byref(err)), err)
    return g.view(n, n).t()  # [row, col]


def cholesky(g, slices: int = 5, nb: int = 2048):
    """Lower Cholesky factor of a symmetric positive definite CUDA float64
    tensor (n x n; its lower triangle is read) through fstk_gpu_cholesky_device:
    panels of `nb` with the trailing updates on the int8 tensor cores at
    `slices` plane-accuracy, or cuSOLVER dpotrf (slices=0).  Returns
    (L, info): info = 0 on success, nonzero when a block is not positive
    definite."""
    import torch

    if not (isinstance(g, torch.Tensor) and g.is_cuda and g.dtype == torch.float64 and g.dim() == 2
            and g.shape[0] == g.shape[1]):
        raise TypeError("cholesky: expected a square 2-D CUDA float64 tensor")
    n = g.shape[0]
    w = g.t().contiguous()  # column-major
    info = C.c_int32(0)
    err = Err()
    stream = torch.cuda.current_stream(g.device).cuda_stream
    check(lib().fstk_gpu_cholesky_device(w.data_ptr(), n, int(nb), int(slices), g.device.index,
                                         stream, C.byref(info), C.byref(err)), err)
    return torch.tril(w.t()), int(info.value)


def reestimate_core(model: Model, points, values, seed=0, sample_rows=0,
                    working_subset=1 << 20, transform="dct", validation_fraction=0.05,
                    device=None):
    """randls.cpp:360-383.  Returns (new_model, info).  One GPU, or -- for a
    model created after set_devices([...]) with several devices -- sharded
    over all of them inside the library (fstk_multi.cu)."""
    require_gpu()
    p, v = _cloud(model, points, values)
    cfg = sketch_config(seed, sample_rows, working_subset, transform, validation_fraction)
    core = np.zeros(int(np.prod(model.ranks)))
    info = ReestimateInfo()
    err = Err()
    check(lib().fstk_gpu_reestimate_core(model.handle(device), dptr(p), dptr(v), p.shape[0],
                                         p.shape[1], C.byref(cfg), dptr(core), C.byref(info),
                                         C.byref(err)), err)
    return model.with_core(core.reshape(model.ranks, order="F")), _info_dict(info)


class _DeviceArray:
    """Zero-copy view of library-owned device memory for torch.as_tensor."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": "<f8",
                                         "data": (int(ptr), False), "version": 3,
                                         "strides": None}


class RefitSession:
    """Staged refit (fstk_gpu_refit_*): used for sharded multi-GPU runs and
    for parity tests that inspect the sampled rows / sketched system.

    layout="rows" (fstk_gpu_refit_begin): every shard transforms all columns
    and keeps its rows.  layout="columns" (fstk_gpu_refit_begin_columns): each
    shard transforms its columns; exchange_buffers() + one all-to-all +
    adopt_rows() then leave the same row slabs."""

    def __init__(self, model: Model, points, values, seed=0, sample_rows=0,
                 working_subset=1 << 20, transform="dct", validation_fraction=0.05,
                 shard=0, shards=1, device=None, layout="rows"):
        require_gpu()
        if layout not in ("rows", "columns"):
            raise ValueError("layout must be 'rows' or 'columns'")
        self.model = model
        self.device = device
        self.shards = shards
        self.layout = layout
        p, v = _cloud(model, points, values)
        self.cfg = sketch_config(seed, sample_rows, working_subset, transform,
                                 validation_fraction)
        self.info = ReestimateInfo()
        out = C.c_void_p()
        err = Err()
        begin = lib().fstk_gpu_refit_begin_columns if layout == "columns" else \
            lib().fstk_gpu_refit_begin
        check(begin(model.handle(device), dptr(p), dptr(v), p.shape[0], p.shape[1],
                    C.byref(self.cfg), shard, shards, C.byref(out), C.byref(self.info),
                    C.byref(err)), err)
        self._h = out.value
        self.R = int(np.prod(model.ranks))

    def exchange_buffers(self):
        """(send, send_counts, recv, recv_counts) of the column-to-row
        all-to-all: CUDA float64 views of the library's buffers and the
        per-peer element counts (rank order).  transform="none" has nothing to
        exchange and returns None."""
        import torch

        if self.layout != "columns" or self.cfg.transform == TRANSFORMS["none"]:
            return None
        sp, rp = C.c_void_p(), C.c_void_p()
        sc = (C.c_int64 * self.shards)()
        rc = (C.c_int64 * self.shards)()
        err = Err()
        check(lib().fstk_gpu_refit_exchange_layout(self._h, C.byref(sp), sc, C.byref(rp), rc,
                                                   C.byref(err)), err)
        dev = torch.device("cuda", self.device if self.device is not None
                           else torch.cuda.current_device())
        send = torch.as_tensor(_DeviceArray(sp.value, sum(sc)), device=dev)
        recv = torch.as_tensor(_DeviceArray(rp.value, sum(rc)), device=dev)
        return send, list(sc), recv, list(rc)

    def adopt_rows(self):
        err = Err()
        check(lib().fstk_gpu_refit_adopt_rows(self._h, C.byref(err)), err)

    def rows(self) -> np.ndarray:
        out = np.zeros(int(self.info.sample_rows), dtype=np.uint64)
        err = Err()
        check(lib().fstk_gpu_refit_rows(self._h, out.ctypes.data_as(C.POINTER(C.c_uint64)),
                                        C.byref(err)), err)
        return out

    def sketched(self):
        n = C.c_int64()
        err = Err()
        check(lib().fstk_gpu_refit_sketched(self._h, None, None, C.byref(n), C.byref(err)), err)
        a = np.zeros((n.value, self.R), order="F")
        b = np.zeros(n.value)
        check(lib().fstk_gpu_refit_sketched(self._h, dptr(a), dptr(b), C.byref(n), C.byref(err)),
              err)
        return a, b

    def sketched_columns(self, cols) -> np.ndarray:
        """Columns `cols` of the sketched A (index R = b) in reference row order."""
        c = np.ascontiguousarray(cols, dtype=np.int64)
        n = C.c_int64()
        err = Err()
        check(lib().fstk_gpu_refit_sketched(self._h, None, None, C.byref(n), C.byref(err)), err)
        out = np.zeros((n.value, c.size), order="F")
        check(lib().fstk_gpu_refit_sketched_columns(self._h, c.ctypes.data_as(C.POINTER(C.c_int64)),
                                                    c.size, dptr(out), C.byref(err)), err)
        return out

    def normal_equations(self, gram_t, rhs_t):
        """Writes this shard's partial A^T A (lower triangle, column-major) and
        A^T b into CUDA float64 tensors of R*R and R elements."""
        err = Err()
        check(lib().fstk_gpu_refit_normal_equations(self._h, gram_t.data_ptr(), rhs_t.data_ptr(),
                                                    C.byref(self.info), C.byref(err)), err)

    def normal_equations_native(self, gram_t, rhs_t):
        """normal_equations() with the native fp64 DSYRK/DGEMM Gram."""
        err = Err()
        check(lib().fstk_gpu_refit_normal_equations_native(
            self._h, gram_t.data_ptr(), rhs_t.data_ptr(), C.byref(self.info), C.byref(err)), err)

    def normal_equations_level(self, slices, gram_t, rhs_t):
        """normal_equations() at an explicit Gram precision: 2..7 (sliced,
        int8 tensor cores) or 0 (native fp64)."""
        err = Err()
        check(lib().fstk_gpu_refit_normal_equations_level(
            self._h, int(slices), gram_t.data_ptr(), rhs_t.data_ptr(), C.byref(self.info),
            C.byref(err)), err)

    def solve(self, gram_t, rhs_t) -> np.ndarray:
        core = np.zeros(self.R)
        err = Err()
        check(lib().fstk_gpu_refit_solve(self._h, gram_t.data_ptr(), rhs_t.data_ptr(), dptr(core),
                                         C.byref(self.info), C.byref(err)), err)
        return core

    # -- sharded solve stages (see include/fstk_gpu.h) --------------------------
    def factor(self, gram_t, rhs_t, x_t):
        err = Err()
        check(lib().fstk_gpu_refit_factor(self._h, gram_t.data_ptr(), rhs_t.data_ptr(),
                                          x_t.data_ptr(), C.byref(self.info), C.byref(err)), err)
        return not bool(self.info.rank_deficient)

    def correction(self, x_t, s_t):
        err = Err()
        check(lib().fstk_gpu_refit_correction(self._h, x_t.data_ptr(), s_t.data_ptr(),
                                              C.byref(err)), err)

    def apply(self, s_t, x_t) -> float:
        step = C.c_double()
        err = Err()
        check(lib().fstk_gpu_refit_apply(self._h, s_t.data_ptr(), x_t.data_ptr(), C.byref(step),
                                         C.byref(err)), err)
        return step.value

    def certify(self, gram_t) -> bool:
        """After the refinement converged: True when the Cholesky route
        certifies full rank in the reference's sense (fstk_gpu_refit_certify)."""
        ratio = C.c_double()
        ok = C.c_int32()
        err = Err()
        check(lib().fstk_gpu_refit_certify(self._h, gram_t.data_ptr(), C.byref(ratio),
                                           C.byref(ok), C.byref(err)), err)
        self.info.sigma_ratio = ratio.value
        if ok.value:
            self.info.rank_deficient = 0
        return bool(ok.value)

    def local_qr(self, raug_t):
        """(R+1)^2 CUDA float64 tensor <- upper R of this shard's [A b]
        (column-major; fstk_gpu_refit_local_qr)."""
        err = Err()
        check(lib().fstk_gpu_refit_local_qr(self._h, raug_t.data_ptr(), C.byref(err)), err)

    def qr_solve(self, raug_t, x_t) -> bool:
        """Pivoted QR of the stacked factor, Eigen's rank rule, QR or COD
        solution into x_t.  Returns rank_deficient."""
        err = Err()
        check(lib().fstk_gpu_refit_qr_solve(self._h, raug_t.data_ptr(), x_t.data_ptr(),
                                            C.byref(self.info), C.byref(err)), err)
        return bool(self.info.rank_deficient)

    def finish(self, x_t) -> np.ndarray:
        core = np.zeros(self.R)
        err = Err()
        check(lib().fstk_gpu_refit_finish(self._h, x_t.data_ptr(), dptr(core), C.byref(self.info),
                                          C.byref(err)), err)
        return core

    def info_dict(self) -> dict:
        return _info_dict(self.info)

    def close(self):
        if self._h:
            lib().fstk_gpu_refit_end(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def qr_stack(top_t, other_t):
    """top := R of [top; other] for two (n1 x n1) column-major upper factors
    (CUDA float64 tensors of n1*n1 elements)."""
    import torch

    n1 = int(round(top_t.numel() ** 0.5))
    err = Err()
    stream = torch.cuda.current_stream(top_t.device).cuda_stream
    check(lib().fstk_gpu_qr_stack(top_t.data_ptr(), other_t.data_ptr(), n1, top_t.device.index,
                                  stream, C.byref(err)), err)


def solve_system(a, b):
    """randls.cpp:112-123 on the GPU: (alpha, rank_deficient, rank) of the
    least-squares system a x = b (ColPivHouseholderQR rank with Eigen's
    threshold; COD minimum-norm solution when deficient)."""
    require_gpu()
    a = np.asfortranarray(np.asarray(a, dtype=np.float64))
    b = np.ascontiguousarray(np.asarray(b, dtype=np.float64))
    if a.ndim != 2 or b.shape != (a.shape[0],):
        raise make_error(2, "solve_system: a must be m x n and b of length m")
    m, n = a.shape
    x = np.zeros(n)
    rank, deficient = C.c_int32(), C.c_int32()
    err = Err()
    check(lib().fstk_gpu_solve_system(dptr(a), m, n, dptr(b), dptr(x), C.byref(rank),
                                      C.byref(deficient), C.byref(err)), err)
    return x, bool(deficient.value), int(rank.value)


def build_design_rows(model: Model, points) -> np.ndarray:
    """randls.cpp:134-145: Q x R, mode-0 index fastest."""
    p = np.asfortranarray(np.asarray(points, dtype=np.float64))
    if p.ndim != 2 or p.shape[1] != model.order:
        raise make_error(1, "points must have one column per mode")
    r = int(np.prod(model.ranks))
    w = np.zeros((p.shape[0], r), order="F")
    err = Err()
    check(lib().fstk_gpu_build_design_rows(model.handle(), dptr(p), p.shape[0], p.shape[1],
                                           dptr(w), C.byref(err)), err)
    return w


def sketch(w, u, seed=0, sample_rows=0, transform="dct"):
    """randls.cpp:147-184: returns (a, b, padded_rows)."""
    require_gpu()
    w = np.asfortranarray(np.asarray(w, dtype=np.float64))
    u = np.ascontiguousarray(np.asarray(u, dtype=np.float64))
    if w.ndim != 2:
        raise make_error(1, "w must be 2-D")
    q, r = w.shape
    if u.shape[0] != q:
        raise make_error(2, "rhs length mismatch")
    cfg = sketch_config(seed, sample_rows, 0, transform, 0.0)
    s = sample_rows if sample_rows > 0 else int(np.ceil(2.5 * r))
    rows = 2 * s if transform == "fft" else s
    a = np.zeros((rows, r), order="F")
    b = np.zeros(rows)
    padded = C.c_uint64()
    err = Err()
    check(lib().fstk_gpu_sketch(dptr(w), dptr(u), q, r, C.byref(cfg), dptr(a), dptr(b),
                                C.byref(padded), C.byref(err)), err)
    return a, b, int(padded.value)


def mixed_matrix(w, seed=0, transform="dct") -> np.ndarray:
    """randls.cpp:186-225."""
    require_gpu()
    w = np.asfortranarray(np.asarray(w, dtype=np.float64))
    q, r = w.shape
    q_pad = 1
    while q_pad < q:
        q_pad <<= 1
    cfg = sketch_config(seed, 0, 0, transform, 0.0)
    out = np.zeros((2 * q_pad if transform == "fft" else q_pad, r), order="F")
    err = Err()
    check(lib().fstk_gpu_mixed_matrix(dptr(w), q, r, C.byref(cfg), dptr(out), C.byref(err)), err)
    return out


def self_convergence(model: Model, points, values, s_values, seed=0, working_subset=1 << 20,
                     transform="dct", validation_fraction=0.05):
    """randls.cpp:385-413: [(S_i, ||a_{i+1}-a_i|| / ||a_{i+1}||), ...]."""
    require_gpu()
    p, v = _cloud(model, points, values)
    sv = np.ascontiguousarray(np.asarray(s_values, dtype=np.uint64))
    cfg = sketch_config(seed, 0, working_subset, transform, validation_fraction)
    deltas = np.zeros(max(sv.size - 1, 1))
    err = Err()
    check(lib().fstk_gpu_self_convergence(model.handle(), dptr(p), dptr(v), p.shape[0], p.shape[1],
                                          C.byref(cfg), sv.ctypes.data_as(C.POINTER(C.c_uint64)),
                                          int(sv.size), dptr(deltas), C.byref(err)), err)
    return [(int(sv[i]), float(deltas[i])) for i in range(sv.size - 1)]


def leverage_scores(w) -> np.ndarray:
    """randls.cpp:227-233."""
    require_gpu()
    w = np.asfortranarray(np.asarray(w, dtype=np.float64))
    q, r = w.shape
    out = np.zeros(q)
    rank = C.c_int32()
    err = Err()
    check(lib().fstk_gpu_leverage_scores(dptr(w), q, r, dptr(out), C.byref(rank), C.byref(err)),
          err)
    return out
