"""ctypes binding of libfstk_gpu.so (the C-ABI declared in include/fstk_gpu.h).

There is no CPU fallback: if the CUDA library is missing, or no GPU is
visible when a compute entry point is called, this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FSTK_GPU_LIB") or os.path.join(HERE, "libfstk_gpu.so")

KINDS = ["Parameter", "Shape", "Domain", "Data", "Io", "Decode", "Compute"]
TRANSFORMS = {"dct": 0, "wht": 1, "fft": 2, "none": 3}


class FstkError(Exception):
    """Base class; `kind` is the fstk::ErrorKind name (error.hpp:11-19)."""

    def __init__(self, kind: str, message: str, mode: int = -1, index: int = -1,
                 value: float = 0.0):
        super().__init__(message)
        self.kind = kind
        self.mode = mode
        self.index = index
        self.value = value


class FstkValueError(FstkError, ValueError):
    """Parameter/Shape/Domain/Data/Compute errors -> ValueError (module.cpp:112-125)."""


class FstkIOError(FstkError, OSError):
    """Io/Decode errors -> IOError (module.cpp:117-119)."""


def make_error(code: int, message: str, mode=-1, index=-1, value=0.0) -> FstkError:
    kind = KINDS[code - 1] if 1 <= code <= len(KINDS) else "Compute"
    cls = FstkIOError if kind in ("Io", "Decode") else FstkValueError
    return cls(kind, message, mode, index, value)


class Err(C.Structure):
    _fields_ = [("kind", C.c_int32), ("mode", C.c_int32), ("index", C.c_int64),
                ("value", C.c_double), ("message", C.c_char * 256)]


class InterpReport(C.Structure):
    _fields_ = [("box_covered", C.c_int32), ("max_nearest_distance", C.c_double),
                ("extrapolated_fraction", C.c_double)]


class ModelDesc(C.Structure):
    _fields_ = [("d", C.c_int32), ("ranks", C.POINTER(C.c_int64)),
                ("core", C.POINTER(C.c_double)), ("family", C.POINTER(C.c_int32)),
                ("degree", C.POINTER(C.c_int32)), ("resolution", C.POINTER(C.c_int32)),
                ("lo", C.POINTER(C.c_double)), ("hi", C.POINTER(C.c_double)),
                ("nnz", C.POINTER(C.c_uint32)), ("indices", C.POINTER(C.c_uint32)),
                ("coeffs", C.POINTER(C.c_double))]


class SketchCfg(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("working_subset", C.c_uint64),
                ("sample_rows", C.c_uint64), ("transform", C.c_int32),
                ("validation_fraction", C.c_double)]


class ReestimateInfo(C.Structure):
    _fields_ = [("residual_before", C.c_double), ("residual_after", C.c_double),
                ("sample_rows", C.c_uint64), ("working_rows", C.c_uint64),
                ("padded_rows", C.c_uint64), ("rank_deficient", C.c_int32),
                ("held_out", C.c_int32), ("t_prepare", C.c_double), ("t_sketch", C.c_double),
                ("t_gram", C.c_double), ("t_solve", C.c_double), ("t_residual", C.c_double),
                ("t_alloc", C.c_double), ("gram_slices", C.c_int32),
                ("refine_steps", C.c_int32), ("gram_int8_ops", C.c_double),
                ("qr_path", C.c_int32), ("sigma_ratio", C.c_double),
                ("t_exchange", C.c_double), ("t_reduce", C.c_double), ("devices", C.c_int32),
                ("multi_transport", C.c_int32)]


# Every symbol include/fstk_gpu.h declares (checked by tests/test_abi.py).
EXPORTS = [
    "fstk_gpu_abi_version", "fstk_gpu_device_count", "fstk_gpu_launch_count",
    "fstk_gpu_trim_device_cache",
    "fstk_gpu_set_device_cache",
    "fstk_gpu_model_create", "fstk_gpu_model_destroy", "fstk_gpu_model_set_core",
    "fstk_gpu_model_get_core", "fstk_gpu_evaluate_batch", "fstk_gpu_evaluate",
    "fstk_gpu_evaluate_batch_device", "fstk_gpu_mode_values", "fstk_gpu_build_design_rows",
    "fstk_gpu_sketch", "fstk_gpu_mixed_matrix", "fstk_gpu_reestimate_core",
    "fstk_gpu_refit_begin", "fstk_gpu_refit_normal_equations", "fstk_gpu_refit_solve",
    "fstk_gpu_refit_end", "fstk_gpu_refit_rows", "fstk_gpu_refit_sketched",
    "fstk_gpu_profile_enable", "fstk_gpu_profile_read", "fstk_gpu_fp64_peak",
    "fstk_gpu_refit_factor", "fstk_gpu_refit_correction", "fstk_gpu_refit_apply",
    "fstk_gpu_refit_finish", "fstk_gpu_evaluate_grid", "fstk_gpu_reconstruct_grid",
    "fstk_gpu_self_convergence", "fstk_gpu_leverage_scores", "fstk_gpu_point_major_to_soa",
    "fstk_gpu_refit_normal_equations_native", "fstk_gpu_gram_slices", "fstk_gpu_gram_engine", "fstk_gpu_gram_device",
    "fstk_gpu_refit_normal_equations_level", "fstk_gpu_refit_begin_columns",
    "fstk_gpu_refit_exchange_layout", "fstk_gpu_refit_adopt_rows",
    "fstk_gpu_sample_without_replacement", "fstk_gpu_make_plan", "fstk_gpu_set_devices",
    "fstk_gpu_cholesky_device", "fstk_gpu_refit_certify", "fstk_gpu_refit_local_qr",
    "fstk_gpu_refit_qr_solve", "fstk_gpu_qr_stack", "fstk_gpu_solve_system",
    "fstk_gpu_refit_sketched_columns", "fstk_gpu_eval_serialize",
    "fstk_gpu_interpolate_to_grid", "fstk_gpu_interpolate_to_grid_device", "fstk_gpu_debug_syrk",
    "fstk_gpu_pack_normal_equations",
]
PROF_KINDS = ["mode_tables", "contract", "transform", "gram", "solve"]

_LIB = None
DP = C.POINTER(C.c_double)
VP = C.c_void_p


def lib():
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            " (there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    L.fstk_gpu_abi_version.restype = C.c_int32
    L.fstk_gpu_device_count.restype = C.c_int32
    L.fstk_gpu_launch_count.restype = C.c_uint64
    L.fstk_gpu_eval_serialize.argtypes = [C.c_int32]
    L.fstk_gpu_eval_serialize.restype = C.c_int32
    L.fstk_gpu_set_device_cache.argtypes = [C.c_int32]
    L.fstk_gpu_set_device_cache.restype = C.c_int32
    L.fstk_gpu_trim_device_cache.argtypes = [C.c_int32]
    L.fstk_gpu_trim_device_cache.restype = C.c_uint64
    L.fstk_gpu_model_create.argtypes = [C.POINTER(ModelDesc), C.c_int32, C.POINTER(VP),
                                        C.POINTER(Err)]
    L.fstk_gpu_model_destroy.argtypes = [VP]
    L.fstk_gpu_model_destroy.restype = None
    L.fstk_gpu_model_set_core.argtypes = [VP, DP, C.POINTER(Err)]
    L.fstk_gpu_model_get_core.argtypes = [VP, DP, C.POINTER(Err)]
    L.fstk_gpu_evaluate_batch.argtypes = [VP, DP, C.c_int64, C.c_int32, DP, C.POINTER(Err)]
    L.fstk_gpu_evaluate.argtypes = [VP, DP, C.c_int32, DP, C.POINTER(Err)]
    L.fstk_gpu_evaluate_batch_device.argtypes = [VP, VP, C.c_int64, C.c_int64, C.c_int32, VP,
                                                 VP, C.POINTER(Err)]
    L.fstk_gpu_mode_values.argtypes = [VP, C.c_int32, DP, C.c_int64, DP, C.POINTER(Err)]
    L.fstk_gpu_build_design_rows.argtypes = [VP, DP, C.c_int64, C.c_int32, DP, C.POINTER(Err)]
    L.fstk_gpu_sketch.argtypes = [DP, DP, C.c_int64, C.c_int64, C.POINTER(SketchCfg), DP, DP,
                                  C.POINTER(C.c_uint64), C.POINTER(Err)]
    L.fstk_gpu_mixed_matrix.argtypes = [DP, C.c_int64, C.c_int64, C.POINTER(SketchCfg), DP,
                                        C.POINTER(Err)]
    L.fstk_gpu_reestimate_core.argtypes = [VP, DP, DP, C.c_int64, C.c_int32,
                                           C.POINTER(SketchCfg), DP, C.POINTER(ReestimateInfo),
                                           C.POINTER(Err)]
    L.fstk_gpu_refit_begin.argtypes = [VP, DP, DP, C.c_int64, C.c_int32, C.POINTER(SketchCfg),
                                       C.c_int32, C.c_int32, C.POINTER(VP),
                                       C.POINTER(ReestimateInfo), C.POINTER(Err)]
    L.fstk_gpu_refit_normal_equations.argtypes = [VP, VP, VP, C.POINTER(ReestimateInfo),
                                                  C.POINTER(Err)]
    L.fstk_gpu_refit_normal_equations_native.argtypes = [VP, VP, VP, C.POINTER(ReestimateInfo),
                                                         C.POINTER(Err)]
    L.fstk_gpu_gram_slices.argtypes = [C.c_int32]
    L.fstk_gpu_gram_slices.restype = C.c_int32
    L.fstk_gpu_gram_engine.argtypes = [C.c_int32]
    L.fstk_gpu_gram_engine.restype = C.c_int32
    L.fstk_gpu_pack_normal_equations.argtypes = [VP, VP, C.c_int64, VP, C.c_int32, VP, C.POINTER(Err)]
    L.fstk_gpu_debug_syrk.argtypes = [VP, C.c_int32, C.c_int64, C.c_int64, VP, C.c_int32, VP, C.POINTER(Err)]
    L.fstk_gpu_refit_begin_columns.argtypes = [VP, DP, DP, C.c_int64, C.c_int32,
                                               C.POINTER(SketchCfg), C.c_int32, C.c_int32,
                                               C.POINTER(VP), C.POINTER(ReestimateInfo),
                                               C.POINTER(Err)]
    L.fstk_gpu_refit_exchange_layout.argtypes = [VP, C.POINTER(VP), C.POINTER(C.c_int64),
                                                 C.POINTER(VP), C.POINTER(C.c_int64),
                                                 C.POINTER(Err)]
    L.fstk_gpu_refit_adopt_rows.argtypes = [VP, C.POINTER(Err)]
    L.fstk_gpu_set_devices.argtypes = [C.c_int32, C.POINTER(C.c_int32), C.POINTER(Err)]
    L.fstk_gpu_sample_without_replacement.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64,
                                                      C.POINTER(C.c_uint64), C.POINTER(Err)]
    L.fstk_gpu_make_plan.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, DP,
                                     C.POINTER(C.c_uint64), DP, C.POINTER(C.c_uint64),
                                     C.POINTER(Err)]
    L.fstk_gpu_refit_normal_equations_level.argtypes = [VP, C.c_int32, VP, VP,
                                                        C.POINTER(ReestimateInfo), C.POINTER(Err)]
    L.fstk_gpu_gram_device.argtypes = [VP, C.c_int64, C.c_int64, C.c_int32, VP, C.c_int32,
                                       C.c_int32, VP, C.POINTER(Err)]
    L.fstk_gpu_cholesky_device.argtypes = [VP, C.c_int32, C.c_int32, C.c_int32, C.c_int32, VP,
                                           C.POINTER(C.c_int32), C.POINTER(Err)]
    L.fstk_gpu_refit_solve.argtypes = [VP, VP, VP, DP, C.POINTER(ReestimateInfo),
                                       C.POINTER(Err)]
    L.fstk_gpu_refit_factor.argtypes = [VP, VP, VP, VP, C.POINTER(ReestimateInfo),
                                        C.POINTER(Err)]
    L.fstk_gpu_refit_correction.argtypes = [VP, VP, VP, C.POINTER(Err)]
    L.fstk_gpu_refit_apply.argtypes = [VP, VP, VP, DP, C.POINTER(Err)]
    L.fstk_gpu_refit_finish.argtypes = [VP, VP, DP, C.POINTER(ReestimateInfo), C.POINTER(Err)]
    L.fstk_gpu_refit_certify.argtypes = [VP, VP, DP, C.POINTER(C.c_int32), C.POINTER(Err)]
    L.fstk_gpu_refit_local_qr.argtypes = [VP, VP, C.POINTER(Err)]
    L.fstk_gpu_refit_sketched_columns.argtypes = [VP, C.POINTER(C.c_int64), C.c_int64, DP,
                                                  C.POINTER(Err)]
    L.fstk_gpu_refit_qr_solve.argtypes = [VP, VP, VP, C.POINTER(ReestimateInfo), C.POINTER(Err)]
    L.fstk_gpu_qr_stack.argtypes = [VP, VP, C.c_int64, C.c_int32, VP, C.POINTER(Err)]
    L.fstk_gpu_solve_system.argtypes = [DP, C.c_int64, C.c_int64, DP, DP, C.POINTER(C.c_int32),
                                        C.POINTER(C.c_int32), C.POINTER(Err)]
    L.fstk_gpu_refit_end.argtypes = [VP]
    L.fstk_gpu_refit_end.restype = None
    L.fstk_gpu_refit_rows.argtypes = [VP, C.POINTER(C.c_uint64), C.POINTER(Err)]
    L.fstk_gpu_refit_sketched.argtypes = [VP, DP, DP, C.POINTER(C.c_int64), C.POINTER(Err)]
    L.fstk_gpu_evaluate_grid.argtypes = [VP, DP, C.POINTER(C.c_int64), C.c_int32, DP,
                                         C.POINTER(Err)]
    L.fstk_gpu_reconstruct_grid.argtypes = [VP, C.POINTER(C.c_int64), C.c_int32, DP,
                                            C.POINTER(Err)]
    L.fstk_gpu_self_convergence.argtypes = [VP, DP, DP, C.c_int64, C.c_int32,
                                            C.POINTER(SketchCfg), C.POINTER(C.c_uint64), C.c_int32,
                                            DP, C.POINTER(Err)]
    L.fstk_gpu_leverage_scores.argtypes = [DP, C.c_int64, C.c_int64, DP, C.POINTER(C.c_int32),
                                           C.POINTER(Err)]
    L.fstk_gpu_point_major_to_soa.argtypes = [VP, C.c_int64, C.c_int32, VP, VP, C.POINTER(Err)]
    L.fstk_gpu_interpolate_to_grid.argtypes = [VP, VP, C.c_int64, C.c_int32, VP, VP, VP, VP, VP,
                                               C.c_int32, C.c_double, VP, C.POINTER(InterpReport),
                                               VP, C.c_int32, C.POINTER(Err)]
    L.fstk_gpu_interpolate_to_grid_device.argtypes = [VP, VP, C.c_int64, C.c_int32, VP, VP, VP, VP,
                                                      VP, C.c_int32, C.c_double, VP,
                                                      C.POINTER(InterpReport), VP, VP, C.POINTER(Err)]
    L.fstk_gpu_profile_enable.argtypes = [C.c_int32]
    L.fstk_gpu_profile_enable.restype = None
    L.fstk_gpu_profile_read.argtypes = [DP, C.POINTER(C.c_uint64), C.POINTER(Err)]
    L.fstk_gpu_fp64_peak.argtypes = [C.c_int32, DP, DP, C.POINTER(Err)]
    _LIB = L
    return L


def check(rc: int, err: Err):
    if rc != 0:
        raise make_error(rc, err.message.decode(errors="replace"), err.mode, err.index, err.value)


def dptr(a):
    return a.ctypes.data_as(DP)


def launch_count() -> int:
    return int(lib().fstk_gpu_launch_count())


def eval_serialize(on: bool) -> bool:
    """Measurement mode: chunks of a device evaluation on one stream (no
    mode/contraction overlap).  Returns the previous setting."""
    return bool(lib().fstk_gpu_eval_serialize(1 if on else 0))


def set_device_cache(policy: int) -> int:
    """Device-cache policy (0 off, 1 per refit session [default], 2
    persistent); returns the previous one.  See fstk_gpu_set_device_cache."""
    return int(lib().fstk_gpu_set_device_cache(int(policy)))


def trim_device_cache(device: int = -1) -> int:
    """Hand the library's cached large device blocks back to the driver
    (bytes released).  Refit sessions reuse them otherwise."""
    return int(lib().fstk_gpu_trim_device_cache(device))


def device_tensor(n: int, device, zero: bool = False):
    """A float64 CUDA tensor of n elements for Gram-sized buffers.  On a torch
    out-of-memory error the library's cached device blocks are handed back and
    the allocation is retried once (torch's allocator does not know about them)."""
    import torch

    make = torch.zeros if zero else torch.empty
    try:
        return make(n, dtype=torch.float64, device=device)
    except torch.OutOfMemoryError:
        d = torch.device(device)
        trim_device_cache(d.index if d.index is not None else torch.cuda.current_device())
        return make(n, dtype=torch.float64, device=device)


def device_count() -> int:
    return int(lib().fstk_gpu_device_count())


def require_gpu():
    if device_count() < 1:
        raise RuntimeError("fstk_gpu: no CUDA device visible (the B200 path has no CPU fallback)")


def profile_enable(on: bool = True):
    lib().fstk_gpu_profile_enable(1 if on else 0)


def profile_read() -> dict:
    """Per kernel class: (summed device ms, launches) since the last read."""
    import numpy as np

    ms = np.zeros(len(PROF_KINDS))
    n = np.zeros(len(PROF_KINDS), dtype=np.uint64)
    err = Err()
    check(lib().fstk_gpu_profile_read(dptr(ms), n.ctypes.data_as(C.POINTER(C.c_uint64)),
                                      C.byref(err)), err)
    return {k: (float(ms[i]), int(n[i])) for i, k in enumerate(PROF_KINDS)}


def fp64_peak(device: int = 0):
    """(DMMA TFLOP/s, DFMA TFLOP/s) measured on `device`."""
    a, b = C.c_double(), C.c_double()
    err = Err()
    check(lib().fstk_gpu_fp64_peak(device, C.byref(a), C.byref(b), C.byref(err)), err)
    return a.value, b.value


DEVICE_LIST: list = []  # fstk_gpu_set_devices (empty: one device per model handle)


def set_devices(ids) -> None:
    """fstk_gpu_set_devices: models created afterwards through Model.handle()
    replicate on these devices and a host evaluate_batch splits across them."""
    ids = [int(i) for i in ids]
    arr = (C.c_int32 * max(len(ids), 1))(*ids)
    err = Err()
    check(lib().fstk_gpu_set_devices(len(ids), arr, C.byref(err)), err)
    DEVICE_LIST[:] = ids
