"""B200-native hot path of the functional sparse Tucker compressor
(arXiv 1907.05884 reference `fstk`): point evaluation and randomized-LS core
refit, behind the C-ABI in include/fstk_gpu.h.

The Python surface mirrors the reference module (proj/python/fstk/__init__.py,
proj/python/module.cpp): `Model.evaluate_batch`, `load_model`,
`reestimate_core`, `BasisSpec`, plus the refit diagnostics.  All compute runs
in libfstk_gpu.so on the GPU; there is no CPU fallback.
"""
from ._lib import FstkError, FstkIOError, FstkValueError, launch_count, set_devices
from .cloud import (InterpolationOptions, InterpolationReport, PointCloud, StructuredGrid,
                    interpolate_to_grid, read_cloud, read_cloud_binary, read_cloud_csv,
                    read_cloud_device, read_points_csv, write_cloud_binary, write_cloud_csv)
from .model import (BasisSpec, Model, ModelMetadata, ModeFunction, eval_basis, evaluate_fields,
                    load_model, save_model)
from .refit import (RefitSession, build_design_rows, cholesky, gram, gram_engine, gram_slices, leverage_scores, mixed_matrix,
                    reestimate_core, self_convergence, sketch, sketch_config)


def set_max_threads(n: int) -> None:
    """Reference knob (parallel.cpp:21); results never depend on it, and the GPU
    path has no host worker pool, so it is accepted and ignored."""
    return None


__all__ = [
    "BasisSpec", "Model", "ModelMetadata", "ModeFunction", "load_model", "save_model",
    "evaluate_fields", "eval_basis",
    "reestimate_core", "RefitSession", "build_design_rows", "sketch", "mixed_matrix",
    "sketch_config", "self_convergence", "leverage_scores", "gram_slices", "gram_engine", "gram", "cholesky",
    "set_max_threads", "FstkError", "FstkValueError", "FstkIOError",
    "launch_count", "set_devices", "PointCloud", "read_cloud", "read_cloud_binary", "read_cloud_csv",
    "read_cloud_device", "read_points_csv", "write_cloud_binary", "write_cloud_csv",
    "StructuredGrid", "InterpolationOptions", "InterpolationReport", "interpolate_to_grid",
]
