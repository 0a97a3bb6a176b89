"""fstk CPU ORACLE (Python side) — TEST INFRASTRUCTURE ONLY.

ctypes front-end over oracle/liboracle.so (the C++ restatement of the
reference hot path, oracle/fstk_oracle.cpp) plus the one piece of the
reference that is Eigen-only and therefore restated here with LAPACK: the
column-pivoted Householder QR solve with its minimum-norm fallback
(proj/src/randls.cpp:112-123, Eigen ColPivHouseholderQR /
CompleteOrthogonalDecomposition) → scipy.linalg.qr(pivoting=True) (LAPACK
dgeqp3) + Eigen's default rank threshold.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this module, and only as the checker or the
CPU baseline.  The product package never imports it.

``ref`` exposes oracle/_ref/libfstk_ref.so — the reference's own rng.cpp,
transforms.cpp and parallel.cpp compiled as-is — used to pin the restatement.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None
_REF = None

TRANSFORMS = {"dct": 0, "wht": 1, "fft": 2, "none": 3}
KINDS = ["Parameter", "Shape", "Domain", "Data", "Io", "Decode", "Compute"]


class OracleError(Exception):
    def __init__(self, code, msg):
        super().__init__(f"{KINDS[code - 1] if 0 < code <= len(KINDS) else code}: {msg}")
        self.kind = KINDS[code - 1] if 0 < code <= len(KINDS) else str(code)
        self.msg = msg


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _u64p(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint64))


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            raise RuntimeError("oracle/liboracle.so missing: run `make -C oracle`")
        L = C.CDLL(path)
        L.oracle_last_error.restype = C.c_char_p
        L.oracle_mix_seed.restype = C.c_uint64
        L.oracle_mix_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.oracle_next_pow2.restype = C.c_uint64
        L.oracle_next_pow2.argtypes = [C.c_uint64]
        _LIB = L
    return _LIB


def ref():
    """The reference's own Eigen-free sources compiled as-is (or None)."""
    global _REF
    if _REF is None:
        path = os.path.join(HERE, "_ref", "libfstk_ref.so")
        if not os.path.exists(path):
            return None
        R = C.CDLL(path)
        R.ref_last_error.restype = C.c_char_p
        R.ref_mix_seed.restype = C.c_uint64
        R.ref_mix_seed.argtypes = [C.c_uint64, C.c_uint64]
        R.ref_next_pow2.restype = C.c_uint64
        R.ref_next_pow2.argtypes = [C.c_uint64]
        for n in ("ref_u64_stream", "ref_sign_stream", "ref_sample_without_replacement"):
            getattr(R, n).restype = None
        R.ref_plan_stream.restype = None
        R.ref_parallel_chunks.restype = None
        _REF = R
    return _REF


def _check(rc):
    if rc != 0:
        raise OracleError(rc, lib().oracle_last_error().decode())


def set_max_threads(n: int):
    lib().oracle_set_max_threads(C.c_int(int(n)))


def max_threads() -> int:
    return int(lib().oracle_max_threads())


# ----------------------------------------------------------------- model ---
@dataclass
class Flat:
    """Flat model arrays (functions listed mode-major)."""

    d: int
    ranks: np.ndarray
    core: np.ndarray
    family: np.ndarray
    degree: np.ndarray
    resolution: np.ndarray
    lo: np.ndarray
    hi: np.ndarray
    nnz: np.ndarray
    idx: np.ndarray
    coeffs: np.ndarray


def flat_of(model) -> Flat:
    """Accepts any object exposing the flat attributes (or a .flat() method)."""
    f = model.flat() if hasattr(model, "flat") else model
    return Flat(
        int(f.d),
        np.ascontiguousarray(f.ranks, dtype=np.int64),
        np.ascontiguousarray(f.core, dtype=np.float64).reshape(-1, order="F"),
        np.ascontiguousarray(f.family, dtype=np.int32),
        np.ascontiguousarray(f.degree, dtype=np.int32),
        np.ascontiguousarray(f.resolution, dtype=np.int32),
        np.ascontiguousarray(f.lo, dtype=np.float64),
        np.ascontiguousarray(f.hi, dtype=np.float64),
        np.ascontiguousarray(f.nnz, dtype=np.uint32),
        np.ascontiguousarray(f.idx, dtype=np.uint32),
        np.ascontiguousarray(f.coeffs, dtype=np.float64),
    )


def _margs(f: Flat):
    i32 = lambda a: a.ctypes.data_as(C.POINTER(C.c_int))
    u32 = lambda a: a.ctypes.data_as(C.POINTER(C.c_uint32))
    # keep refs alive via the Flat object
    idx = f.idx if f.idx.size else np.zeros(1, np.uint32)
    co = f.coeffs if f.coeffs.size else np.zeros(1, np.float64)
    f._keep = (idx, co)
    return [C.c_int(f.d), f.ranks.ctypes.data_as(C.POINTER(C.c_int64)), _dp(f.core),
            i32(f.family), i32(f.degree), i32(f.resolution), _dp(f.lo), _dp(f.hi),
            u32(f.nnz), u32(idx), _dp(co)]


def _fpoints(points, d=None):
    p = np.asarray(points, dtype=np.float64)
    if p.ndim == 1:
        p = p.reshape(1, -1) if d is None or p.size == d else p.reshape(-1, 1)
    return np.asfortranarray(p)


def validate_model(model):
    f = flat_of(model)
    _check(lib().oracle_validate_model(*_margs(f)))


def legendre_values(p: int, t: float) -> np.ndarray:
    out = np.zeros(p + 1)
    _check(lib().oracle_legendre_values(C.c_int(p), C.c_double(t), _dp(out)))
    return out


def eval_basis(degree, lo, hi, x, family=0, resolution=0):
    out = np.zeros((degree + 1) << (resolution if family == 1 else 0))
    _check(lib().oracle_eval_basis(C.c_int(family), C.c_int(degree), C.c_int(resolution),
                                   C.c_double(lo), C.c_double(hi), C.c_double(x), _dp(out)))
    return out


def gauss_legendre(n):
    a, b = np.zeros(n), np.zeros(n)
    _check(lib().oracle_gauss_legendre(C.c_int(n), _dp(a), _dp(b)))
    return a, b


def mother_coords(p):
    out = np.zeros((2 * (p + 1), p + 1), order="F")
    _check(lib().oracle_mother_coords(C.c_int(p), _dp(out)))
    return out


def mode_values(model, mode: int, x: float) -> np.ndarray:
    f = flat_of(model)
    r = int(f.ranks[mode]) if 0 <= mode < f.d else 1
    out = np.zeros(max(r, 1))
    _check(lib().oracle_mode_values(*_margs(f), C.c_int(mode), C.c_double(x), _dp(out)))
    return out


def evaluate(model, y) -> float:
    f = flat_of(model)
    y = np.ascontiguousarray(y, dtype=np.float64)
    out = np.zeros(1)
    _check(lib().oracle_evaluate(*_margs(f), _dp(y), C.c_int(y.size), _dp(out)))
    return float(out[0])


def evaluate_batch(model, points) -> np.ndarray:
    """proj/src/model.cpp:208-227 — points Q x d (any order; copied to F-order)."""
    f = flat_of(model)
    p = _fpoints(points)
    out = np.zeros(p.shape[0])
    _check(lib().oracle_evaluate_batch(*_margs(f), _dp(p), C.c_int64(p.shape[0]),
                                       C.c_int(p.shape[1]), _dp(out)))
    return out


def build_design_rows(model, points) -> np.ndarray:
    f = flat_of(model)
    p = _fpoints(points)
    r = int(np.prod(f.ranks))
    w = np.zeros((p.shape[0], r), order="F")
    _check(lib().oracle_build_design_rows(*_margs(f), _dp(p), C.c_int64(p.shape[0]),
                                          C.c_int(p.shape[1]), _dp(w)))
    return w


# ------------------------------------------------------------ transforms ---
def mix_seed(seed, tag):
    return int(lib().oracle_mix_seed(seed, tag))


def next_pow2(n):
    return int(lib().oracle_next_pow2(n))


def sample_without_replacement(seed, n, k):
    out = np.zeros(min(k, n), dtype=np.uint64)
    _check(lib().oracle_sample_without_replacement(C.c_uint64(seed), C.c_uint64(n),
                                                   C.c_uint64(k), _u64p(out)))
    return out


def make_plan(q_w, s, seed):
    q_pad = next_pow2(q_w)
    signs = np.zeros(q_pad)
    rows = np.zeros(s, dtype=np.uint64)
    scale = np.zeros(1)
    _check(lib().oracle_make_plan(C.c_uint64(q_w), C.c_uint64(s), C.c_uint64(seed),
                                  _dp(signs), _u64p(rows), _dp(scale)))
    return signs, rows, float(scale[0])


def dct2(x):
    y = np.array(x, dtype=np.float64, copy=True)
    _check(lib().oracle_dct2(_dp(y), C.c_uint64(y.size)))
    return y


def wht(x):
    y = np.array(x, dtype=np.float64, copy=True)
    _check(lib().oracle_wht(_dp(y), C.c_uint64(y.size)))
    return y


def fft_pow2(x, inverse=False):
    y = np.array(x, dtype=np.complex128, copy=True)
    _check(lib().oracle_fft_pow2(y.ctypes.data_as(C.POINTER(C.c_double)),
                                 C.c_uint64(y.size), C.c_int(int(inverse))))
    return y


def unitary_fft(x, inverse=False):
    y = np.array(x, dtype=np.complex128, copy=True)
    _check(lib().oracle_unitary_fft(y.ctypes.data_as(C.POINTER(C.c_double)),
                                    C.c_uint64(y.size), C.c_int(int(inverse))))
    return y


# ---------------------------------------------------------------- sketch ---
def sketch(w, u, seed=0, sample_rows=0, transform="dct"):
    """proj/src/randls.cpp:147-184 (public sketch(): plan seeded with cfg.seed)."""
    w = np.asfortranarray(w, dtype=np.float64)
    u = np.ascontiguousarray(u, dtype=np.float64)
    q, r = w.shape
    s = sample_rows if sample_rows > 0 else int(np.ceil(2.5 * r))
    t = TRANSFORMS[transform]
    rows = 2 * s if t == 2 else s
    a = np.zeros((rows, r), order="F")
    b = np.zeros(rows)
    padded = np.zeros(1, dtype=np.uint64)
    _check(lib().oracle_sketch(_dp(w), _dp(u), C.c_int64(q), C.c_int64(r), C.c_uint64(seed),
                               C.c_uint64(sample_rows), C.c_int(t), _dp(a), _dp(b), _u64p(padded)))
    return a, b, int(padded[0])


def mixed_matrix(w, seed=0, transform="dct"):
    w = np.asfortranarray(w, dtype=np.float64)
    q, r = w.shape
    q_pad = next_pow2(q)
    t = TRANSFORMS[transform]
    out = np.zeros((2 * q_pad if t == 2 else q_pad, r), order="F")
    _check(lib().oracle_mixed_matrix(_dp(w), C.c_int64(q), C.c_int64(r), C.c_uint64(seed),
                                     C.c_int(t), _dp(out)))
    return out


# ------------------------------------------------------- QR solve (Eigen) ---
def solve_system_rank(a, b):
    """Restates randls.cpp:112-123 with LAPACK: ColPivHouseholderQR (dgeqp3);
    rank = #{|R_ii| > min(m,n) eps max|R_ii|} (Eigen's default threshold,
    ColPivHouseholderQR::rank()); full rank -> the QR solution; otherwise the
    CompleteOrthogonalDecomposition minimum-norm solution, i.e. the min-norm
    solution of the rank-k system [R11 R12] P^T x = (Q^T b)_k, computed from
    the QR of [R11 R12]^T.  Returns (alpha, rank_deficient, rank)."""
    import scipy.linalg as sla

    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    m, n = a.shape
    q, r, piv = sla.qr(a, mode="economic", pivoting=True, check_finite=False)
    diag = np.abs(np.diag(r))
    thresh = min(m, n) * np.finfo(np.float64).eps
    maxp = float(diag.max()) if diag.size else 0.0
    rank = int(np.sum(diag > thresh * maxp)) if maxp > 0 else 0
    c = q.T @ b
    alpha = np.zeros(n)
    if rank == n:
        alpha[piv] = sla.solve_triangular(r, c, check_finite=False)
        return alpha, False, rank
    if rank > 0:
        q3, u = np.linalg.qr(r[:rank, :].T)  # [R11 R12]^T = Q3 U
        z = sla.solve_triangular(u, c[:rank], trans="T", check_finite=False)
        alpha[piv] = q3 @ z
    return alpha, True, rank


def solve_system(a, b):
    """(alpha, rank_deficient) of solve_system_rank."""
    alpha, deficient, _ = solve_system_rank(a, b)
    return alpha, deficient


# ------------------------------------------------------- reestimate_core ---
class _Sizes(C.Structure):
    _fields_ = [("sample_rows", C.c_uint64), ("working_rows", C.c_uint64),
                ("padded_rows", C.c_uint64), ("n_val", C.c_uint64),
                ("system_rows", C.c_int64), ("held_out", C.c_int)]


def refit_system(model, points, values, seed=0, sample_rows=0, working_subset=1 << 20,
                 transform="dct", validation_fraction=0.05):
    """prepare + solve_sketched up to the sketched system (randls.cpp:246-348)."""
    f = flat_of(model)
    p = _fpoints(points)
    v = np.ascontiguousarray(values, dtype=np.float64)
    t = TRANSFORMS[transform]
    sz = _Sizes()
    args = _margs(f)
    _check(lib().oracle_refit_sizes(*args, C.c_int64(p.shape[0]), C.c_uint64(seed),
                                    C.c_uint64(working_subset), C.c_uint64(sample_rows),
                                    C.c_int(t), C.c_double(validation_fraction), C.byref(sz)))
    r = int(np.prod(f.ranks))
    a = np.zeros((sz.system_rows, r), order="F")
    b = np.zeros(sz.system_rows)
    rows = np.zeros(sz.sample_rows, dtype=np.uint64)
    val_index = np.zeros(sz.n_val, dtype=np.uint64)
    _check(lib().oracle_refit_system(*args, _dp(p), _dp(v), C.c_int64(p.shape[0]),
                                     C.c_int(p.shape[1]), C.c_uint64(seed),
                                     C.c_uint64(working_subset), C.c_uint64(sample_rows),
                                     C.c_int(t), C.c_double(validation_fraction), _dp(a), _dp(b),
                                     _u64p(rows), _u64p(val_index)))
    info = dict(sample_rows=int(sz.sample_rows), working_rows=int(sz.working_rows),
                padded_rows=int(sz.padded_rows), held_out=bool(sz.held_out))
    return a, b, rows, val_index, info


def refit_columns(model, points, values, col_begin, col_end, seed=0, sample_rows=0,
                  working_subset=1 << 20, transform="dct", validation_fraction=0.05):
    """Sketched columns [col_begin, col_end) only (CPU-baseline sampling)."""
    f = flat_of(model)
    p = _fpoints(points)
    v = np.ascontiguousarray(values, dtype=np.float64)
    t = TRANSFORMS[transform]
    sz = _Sizes()
    args = _margs(f)
    _check(lib().oracle_refit_sizes(*args, C.c_int64(p.shape[0]), C.c_uint64(seed),
                                    C.c_uint64(working_subset), C.c_uint64(sample_rows),
                                    C.c_int(t), C.c_double(validation_fraction), C.byref(sz)))
    a = np.zeros((sz.system_rows, col_end - col_begin), order="F")
    _check(lib().oracle_refit_columns(*args, _dp(p), _dp(v), C.c_int64(p.shape[0]),
                                      C.c_int(p.shape[1]), C.c_uint64(seed),
                                      C.c_uint64(working_subset), C.c_uint64(sample_rows),
                                      C.c_int(t), C.c_double(validation_fraction),
                                      C.c_int64(col_begin), C.c_int64(col_end), _dp(a)))
    return a


def refit_column_set(model, points, values, cols, seed=0, sample_rows=0,
                     working_subset=1 << 20, transform="dct", validation_fraction=0.05):
    """Sketched columns at the given indices (index R = the right-hand side b)
    and the plan's sampled rows: (a (system_rows x len(cols)), rows)."""
    f = flat_of(model)
    p = _fpoints(points)
    v = np.ascontiguousarray(values, dtype=np.float64)
    t = TRANSFORMS[transform]
    sz = _Sizes()
    args = _margs(f)
    _check(lib().oracle_refit_sizes(*args, C.c_int64(p.shape[0]), C.c_uint64(seed),
                                    C.c_uint64(working_subset), C.c_uint64(sample_rows),
                                    C.c_int(t), C.c_double(validation_fraction), C.byref(sz)))
    c = np.ascontiguousarray(cols, dtype=np.int64)
    a = np.zeros((sz.system_rows, c.size), order="F")
    rows = np.zeros(int(sz.sample_rows), dtype=np.uint64)
    _check(lib().oracle_refit_column_set(*args, _dp(p), _dp(v), C.c_int64(p.shape[0]),
                                         C.c_int(p.shape[1]), C.c_uint64(seed),
                                         C.c_uint64(working_subset), C.c_uint64(sample_rows),
                                         C.c_int(t), C.c_double(validation_fraction),
                                         c.ctypes.data_as(C.POINTER(C.c_int64)),
                                         C.c_int64(c.size), _dp(a), _u64p(rows)))
    return a, rows


def relative_residual(model_flat, points, values):
    """randls.cpp:350-356."""
    pred = evaluate_batch(model_flat, points)
    denom = np.linalg.norm(values)
    diff = np.linalg.norm(pred - values)
    return diff / denom if denom > 0 else diff


def reestimate_core(model, points, values, seed=0, sample_rows=0, working_subset=1 << 20,
                    transform="dct", validation_fraction=0.05):
    """randls.cpp:360-383: returns (new_core (flat, mode-0 fastest), info)."""
    f = flat_of(model)
    p = _fpoints(points)
    v = np.ascontiguousarray(values, dtype=np.float64)
    a, b, rows, val_index, info = refit_system(f, p, v, seed, sample_rows, working_subset,
                                               transform, validation_fraction)
    alpha, rank_def = solve_system(a, b)
    vi = val_index.astype(np.int64)
    vp, vv = p[vi], v[vi]
    info["residual_before"] = relative_residual(f, vp, vv)
    f2 = Flat(**{k: getattr(f, k) for k in Flat.__dataclass_fields__})
    f2.core = alpha.copy()
    info["residual_after"] = relative_residual(f2, vp, vv)
    info["rank_deficient"] = bool(rank_def)
    info["rows"] = rows
    return alpha, info


def leverage_scores(w):
    """randls.cpp:227-233 restated: thin SVD, rank by Eigen's SVDBase rule."""
    w = np.asarray(w, dtype=np.float64)
    q, r = w.shape
    if q < r:
        raise OracleError(1, "leverage scores need at least as many rows as columns")
    u, s, _ = np.linalg.svd(w, full_matrices=False)
    thr = min(q, r) * np.finfo(np.float64).eps * (s[0] if s.size else 0.0)
    rank = int(np.sum(s > thr))
    return np.sum(u[:, :rank] ** 2, axis=1)


def self_convergence(model, points, values, s_values, seed=0, working_subset=1 << 20,
                     transform="dct", validation_fraction=0.05):
    """randls.cpp:385-413 restated on top of the oracle's sketched systems."""
    s_values = [int(s) for s in s_values]
    if len(s_values) < 2:
        raise OracleError(1, "need at least two sample counts")
    alphas = []
    for s in s_values:
        a, b, _, _, _ = refit_system(model, points, values, seed, s, working_subset, transform,
                                     validation_fraction)
        alphas.append(solve_system(a, b)[0])
    out = []
    for i in range(len(s_values) - 1):
        den = np.linalg.norm(alphas[i + 1])
        dl = np.linalg.norm(alphas[i + 1] - alphas[i])
        out.append((s_values[i], dl / den if den > 0 else dl))
    return out


def interpolate_to_grid(points, values, sizes, intervals=None, neighbors=0, power=2.0, box=None,
                        return_neighbors=False):
    """ingest.cpp:265-383 restated (kNN inverse-distance weighting over a
    uniform-binning spatial index).  points: (Q, d); sizes: grid sizes;
    intervals: [(lo, hi)] per mode (default unit box); box: optional (lo, hi)
    arrays (default: the points' bounding box, PointCloud::from_data).
    Returns (grid values of shape sizes, mode-0 fastest; report dict) and,
    with return_neighbors, per node the retained ids sorted by (d2, id)."""
    p = np.asfortranarray(np.asarray(points, dtype=np.float64))
    q, d = p.shape
    v = np.ascontiguousarray(values, dtype=np.float64)
    sz = np.ascontiguousarray(sizes, dtype=np.int64)
    iv = intervals if intervals is not None else [(0.0, 1.0)] * d
    glo = np.ascontiguousarray([a for a, _ in iv], dtype=np.float64)
    ghi = np.ascontiguousarray([b for _, b in iv], dtype=np.float64)
    n = int(np.prod(sz))
    out = np.empty(n, dtype=np.float64)
    rep = np.zeros(3, dtype=np.float64)
    kn = int(neighbors) if neighbors > 0 else 2 * d + 2
    nbr = np.empty(n * kn, dtype=np.uint32) if return_neighbors else None
    blo = bhi = None
    if box is not None:
        blo = np.ascontiguousarray(box[0], dtype=np.float64)
        bhi = np.ascontiguousarray(box[1], dtype=np.float64)
    L = lib()
    _check(L.oracle_interpolate_to_grid(
        _dp(p), _dp(v), C.c_int64(q), C.c_int(d), _dp(blo) if blo is not None else None,
        _dp(bhi) if bhi is not None else None, sz.ctypes.data_as(C.POINTER(C.c_int64)), _dp(glo),
        _dp(ghi), C.c_int(int(neighbors)), C.c_double(float(power)), _dp(out), _dp(rep),
        nbr.ctypes.data_as(C.POINTER(C.c_uint32)) if nbr is not None else None))
    report = {"box_covered": bool(rep[0]), "max_nearest_distance": float(rep[1]),
              "extrapolated_fraction": float(rep[2])}
    grid = out.reshape(tuple(int(x) for x in sz), order="F")
    if return_neighbors:
        return grid, report, nbr.reshape(n, kn)
    return grid, report
