"""Host-side mirror of the reference `fstk.Model` / FSTK interface.

Mirrors proj/python/module.cpp:196-251 (class Model: order, ranks, core,
domain, evaluate, evaluate_batch, storage, compression_ratio, save) and
proj/include/fstk/model.hpp:33-59 (FunctionalSparseTuckerModel), with the
compute going through the B200 C-ABI (include/fstk_gpu.h).  The FSTK v1
container reader/writer follows proj/src/model.cpp:280-426 and
proj/docs/format.md:56-92.
"""
from __future__ import annotations

import ctypes as C
import collections
import json
import struct
import threading
from dataclasses import dataclass, field
from typing import List, Sequence, Tuple

import numpy as np

from . import _lib
from ._lib import Err, FstkIOError, FstkValueError, ModelDesc, check, dptr, lib, make_error

K_MAX_ORDER = 8  # tensor.hpp:16
FSTK_MAGIC = b"FSTK"
FSTK_VERSION = 1


@dataclass(frozen=True)
class BasisSpec:
    """proj/include/fstk/basis.hpp:22-38."""

    family: str = "legendre"  # "legendre" | "wavelet"
    degree: int = 0
    resolution: int = 0
    lo: float = -1.0
    hi: float = 1.0

    @staticmethod
    def legendre(p: int, lo: float = -1.0, hi: float = 1.0) -> "BasisSpec":
        s = BasisSpec("legendre", int(p), 0, float(lo), float(hi))
        s.validate()
        return s

    @staticmethod
    def wavelet(s: int, p: int, lo: float = -1.0, hi: float = 1.0) -> "BasisSpec":
        b = BasisSpec("wavelet", int(p), int(s), float(lo), float(hi))
        b.validate()
        return b

    def with_domain(self, lo: float, hi: float) -> "BasisSpec":
        b = BasisSpec(self.family, self.degree, self.resolution, float(lo), float(hi))
        b.validate()
        return b

    def dimension(self) -> int:
        return self.degree + 1 if self.family == "legendre" else (self.degree + 1) << self.resolution

    def validate(self):
        """basis.cpp:30-47."""
        def bad(msg):
            raise make_error(1, msg)
        if not (0 <= self.degree <= 64):
            bad("basis degree must be in [0, 64]")
        if self.family == "legendre":
            if self.resolution != 0:
                bad("Legendre basis has no resolution parameter")
        elif self.family == "wavelet":
            if not (0 <= self.resolution <= 20):
                bad("wavelet resolution must be in [0, 20]")
            if (self.degree + 1) << self.resolution > (1 << 24):
                bad("basis dimension too large")
        else:
            raise make_error(6, f"unknown basis family: {self.family}")
        if not (self.lo < self.hi):
            bad("basis domain must satisfy lo < hi")
        if not (np.isfinite(self.lo) and np.isfinite(self.hi)):
            bad("basis domain must be finite")


@dataclass
class ModeFunction:
    """SparseFit (lars.hpp:41-50) + flag (model.hpp:15-20)."""

    basis: BasisSpec
    coeffs: List[Tuple[int, float]] = field(default_factory=list)  # ascending index
    chosen_lambda: float = 0.0
    loo_error: float = 0.0
    residual_rel: float = 0.0
    flagged: bool = False


@dataclass
class ModelMetadata:
    grid_sizes: List[int] = field(default_factory=list)
    epsilon: float = 0.0
    achieved_error: float = 0.0
    flagged_fits: int = 0
    provenance: str = ""


class _Flat:
    __slots__ = ("d", "ranks", "core", "family", "degree", "resolution", "lo", "hi", "nnz",
                 "idx", "coeffs")


class Model:
    """Functional sparse Tucker model, device-resident through the C-ABI.

    Immutable like the reference (model.hpp:33-59): `with_core` returns a new
    model.  The device copy is created lazily per CUDA device.
    """

    def __init__(self, core, modes: Sequence[Sequence[ModeFunction]],
                 metadata: ModelMetadata | None = None):
        core = np.asarray(core, dtype=np.float64)
        if core.ndim == 0:
            core = core.reshape(1)
        self._core = np.asfortranarray(core)
        self._modes = [list(m) for m in modes]
        self.metadata = metadata or ModelMetadata()
        self._handles = {}
        self._lock = threading.Lock()
        self._validate_structure()

    # -- reference accessors -------------------------------------------------
    @property
    def order(self) -> int:
        return self._core.ndim

    @property
    def ranks(self) -> List[int]:
        return list(self._core.shape)

    @property
    def core(self) -> np.ndarray:
        return self._core.copy(order="F")

    @property
    def modes(self):
        return self._modes

    @property
    def flagged_fits(self) -> int:
        return self.metadata.flagged_fits

    def domain(self, mode: int) -> Tuple[float, float]:
        """model.cpp:55-60."""
        if not (0 <= mode < self.order):
            raise make_error(1, "mode out of range")
        b = self._modes[mode][0].basis
        return (b.lo, b.hi)

    def _validate_structure(self):
        """model.cpp:31-53."""
        d = self._core.ndim
        if len(self._modes) != d:
            raise make_error(2, "model: mode count does not match core order")
        if not (1 <= d <= K_MAX_ORDER):
            raise make_error(2, "model: bad order")
        for k in range(d):
            fns = self._modes[k]
            if len(fns) != self._core.shape[k]:
                raise make_error(2, "model: function count does not match rank")
            if not fns:
                raise make_error(2, "model: empty mode")
            lo, hi = fns[0].basis.lo, fns[0].basis.hi
            for fn in fns:
                fn.basis.validate()
                if fn.basis.lo != lo or fn.basis.hi != hi:
                    raise make_error(2, "model: inconsistent domains within a mode")
                n = fn.basis.dimension()
                for i, _ in fn.coeffs:
                    if not (0 <= int(i) < n):
                        raise make_error(2, "model: coefficient index outside basis dimension")

    def with_core(self, core) -> "Model":
        """model.cpp:62-69."""
        core = np.asarray(core, dtype=np.float64)
        if core.ndim == 1 and core.size == int(np.prod(self.ranks)):
            core = core.reshape(self.ranks, order="F")
        if list(core.shape) != self.ranks:
            raise make_error(2, "replacement core has wrong shape")
        return Model(core, self._modes, self.metadata)

    # -- flat descriptor (also accepted by the test oracle) -------------------
    def flat(self) -> _Flat:
        f = _Flat()
        f.d = self.order
        f.ranks = np.asarray(self.ranks, dtype=np.int64)
        f.core = np.ascontiguousarray(self._core.reshape(-1, order="F"))
        fns = [fn for m in self._modes for fn in m]
        f.family = np.asarray([0 if fn.basis.family == "legendre" else 1 for fn in fns], np.int32)
        f.degree = np.asarray([fn.basis.degree for fn in fns], np.int32)
        f.resolution = np.asarray([fn.basis.resolution for fn in fns], np.int32)
        f.lo = np.asarray([fn.basis.lo for fn in fns], np.float64)
        f.hi = np.asarray([fn.basis.hi for fn in fns], np.float64)
        f.nnz = np.asarray([len(fn.coeffs) for fn in fns], np.uint32)
        f.idx = np.asarray([int(i) for fn in fns for i, _ in fn.coeffs], np.uint32)
        f.coeffs = np.asarray([float(c) for fn in fns for _, c in fn.coeffs], np.float64)
        return f

    # -- device handle ---------------------------------------------------------
    def handle(self, device: int | None = None):
        """The fstk_gpu_model* for `device` (default: current torch/CUDA device
        0, or -- after set_devices(ids) -- a model replicated on those devices,
        whose host evaluate_batch splits the points across them)."""
        if device is None:
            device = -1 if _lib.DEVICE_LIST else _current_device()
        with self._lock:
            h = self._handles.get(device)
            if h is None:
                _lib.require_gpu()
                f = self.flat()
                keep = [np.ascontiguousarray(a) for a in
                        (f.ranks, f.core, f.family, f.degree, f.resolution, f.lo, f.hi, f.nnz,
                         f.idx if f.idx.size else np.zeros(1, np.uint32),
                         f.coeffs if f.coeffs.size else np.zeros(1, np.float64))]
                desc = ModelDesc(
                    f.d, keep[0].ctypes.data_as(C.POINTER(C.c_int64)), dptr(keep[1]),
                    keep[2].ctypes.data_as(C.POINTER(C.c_int32)),
                    keep[3].ctypes.data_as(C.POINTER(C.c_int32)),
                    keep[4].ctypes.data_as(C.POINTER(C.c_int32)), dptr(keep[5]), dptr(keep[6]),
                    keep[7].ctypes.data_as(C.POINTER(C.c_uint32)),
                    keep[8].ctypes.data_as(C.POINTER(C.c_uint32)), dptr(keep[9]))
                out = C.c_void_p()
                err = Err()
                check(lib().fstk_gpu_model_create(C.byref(desc), device, C.byref(out), C.byref(err)),
                      err)
                h = _Handle(out.value)
                self._handles[device] = h
            return h.ptr

    # -- evaluation ------------------------------------------------------------
    def evaluate(self, y) -> float:
        """model.cpp:195-206."""
        y = np.ascontiguousarray(y, dtype=np.float64).reshape(-1)
        if y.size != self.order:
            raise make_error(1, "evaluation point has wrong dimension")
        out = np.zeros(1)
        err = Err()
        check(lib().fstk_gpu_evaluate(self.handle(), dptr(y), y.size, dptr(out), C.byref(err)), err)
        return float(out[0])

    def evaluate_batch(self, points) -> np.ndarray:
        """model.cpp:208-227: points Q x d (any layout; used column-major like Eigen)."""
        p = np.asarray(points, dtype=np.float64)
        if p.ndim != 2:
            raise FstkValueError("Parameter", "points must be a 2-D array")
        if p.shape[1] != self.order:
            raise make_error(1, "points must have one column per mode")
        p = np.asfortranarray(p)
        out = np.empty(p.shape[0])
        if p.shape[0] == 0:
            return out
        err = Err()
        check(lib().fstk_gpu_evaluate_batch(self.handle(), dptr(p), p.shape[0], p.shape[1],
                                            dptr(out), C.byref(err)), err)
        return out

    def evaluate_batch_into(self, points, out) -> np.ndarray:
        """evaluate_batch writing into `out` (float64, Q); `points` must already
        be a column-major (Q, d) float64 array (e.g. a pinned buffer view), so
        no host copy is made."""
        if not (isinstance(points, np.ndarray) and points.dtype == np.float64
                and points.ndim == 2 and points.flags.f_contiguous):
            raise make_error(1, "points must be a column-major float64 (Q, d) array")
        if points.shape[1] != self.order:
            raise make_error(1, "points must have one column per mode")
        if not (out.dtype == np.float64 and out.flags.c_contiguous and out.size == points.shape[0]):
            raise make_error(1, "out must be a contiguous float64 array of Q values")
        if points.shape[0] == 0:
            return out
        err = Err()
        check(lib().fstk_gpu_evaluate_batch(self.handle(), dptr(points), points.shape[0],
                                            points.shape[1], dptr(out), C.byref(err)), err)
        return out

    def evaluate_grid(self, coords) -> np.ndarray:
        """All nodes of the tensor grid coords[0] x coords[1] x ... as an array of
        shape (len(coords[0]), ...), mode-0 fastest in memory (FTEN order)."""
        if len(coords) != self.order:
            raise make_error(1, "grid needs one size per mode")
        cs = [np.ascontiguousarray(np.atleast_1d(np.asarray(c, dtype=np.float64))) for c in coords]
        sizes = np.asarray([c.size for c in cs], dtype=np.int64)
        flat = np.ascontiguousarray(np.concatenate(cs))
        out = np.empty(int(np.prod(sizes)))
        err = Err()
        check(lib().fstk_gpu_evaluate_grid(self.handle(), dptr(flat),
                                           sizes.ctypes.data_as(C.POINTER(C.c_int64)), self.order,
                                           dptr(out), C.byref(err)), err)
        return out.reshape(tuple(int(v) for v in sizes), order="F")

    def reconstruct_grid(self, sizes) -> np.ndarray:
        """reconstruct --grid (pipeline.cpp:531-569): uniform nodes on the domain."""
        sz = np.asarray(sizes, dtype=np.int64)
        if sz.size != self.order:
            raise make_error(1, "--grid needs one size per mode")
        out = np.empty(int(np.prod(sz)))
        err = Err()
        check(lib().fstk_gpu_reconstruct_grid(self.handle(),
                                              sz.ctypes.data_as(C.POINTER(C.c_int64)), self.order,
                                              dptr(out), C.byref(err)), err)
        return out.reshape(tuple(int(v) for v in sz), order="F")

    def slice(self, mode_x: int, mode_y: int, fixed: dict, width: int = 0, height: int = 0):
        """slice (pipeline.cpp:571-640): values on a width x height grid over
        (mode_x, mode_y) with the other modes fixed; returns (h, w), row i = y_i."""
        d = self.order
        if not (0 <= mode_x < d and 0 <= mode_y < d):
            raise make_error(1, "slice modes must name existing modes")
        if mode_x == mode_y:
            raise make_error(1, "slice modes must differ")
        gsz = self.metadata.grid_sizes
        dflt = lambda k: gsz[k] if k < len(gsz) and gsz[k] >= 2 else 128
        w = width if width > 0 else dflt(mode_x)
        h = height if height > 0 else dflt(mode_y)
        if w < 2 or h < 2:
            raise make_error(1, "slice resolution must be at least 2 per axis")
        coords = []
        for k in range(d):
            lo, hi = self.domain(k)
            if k == mode_x:
                coords.append(lo + (hi - lo) * np.arange(w, dtype=np.float64) / (w - 1))
            elif k == mode_y:
                coords.append(lo + (hi - lo) * np.arange(h, dtype=np.float64) / (h - 1))
            else:
                if k not in fixed:
                    raise make_error(1, f"missing fixed value for mode {k}")
                v = float(fixed[k])
                if not (v >= lo - 1e-12 * (hi - lo) and v <= hi + 1e-12 * (hi - lo)):
                    raise make_error(3, f"fixed value for mode {k} outside the model domain")
                coords.append(np.array([v]))
        g = self.evaluate_grid(coords)
        g = g.reshape([g.shape[k] for k in range(d) if k in (mode_x, mode_y)], order="F")
        return g.T if mode_x < mode_y else g

    def evaluate_device(self, points_t, out_t=None, stream=None):
        """Device-resident evaluation: `points_t` is a CUDA torch tensor of shape
        (d, Q) (row k = coordinate k, i.e. the column-major Q x d buffer) or a
        (Q, d) column-major view.  Returns a CUDA tensor of Q values."""
        import torch

        t = points_t
        if t.dim() != 2:
            raise make_error(1, "points must be 2-D")
        if t.shape[0] == self.order and t.stride(1) == 1:
            q, ld = t.shape[1], t.stride(0)
        elif t.shape[1] == self.order and t.stride(0) == 1:
            q, ld = t.shape[0], t.stride(1)
        else:
            raise make_error(1, "points must be (d, Q) row-major or (Q, d) column-major")
        if t.dtype != torch.float64 or not t.is_cuda:
            raise make_error(1, "points must be a CUDA float64 tensor")
        if out_t is None:
            out_t = torch.empty(q, dtype=torch.float64, device=t.device)
        s = stream if stream is not None else torch.cuda.current_stream(t.device)
        err = Err()
        check(lib().fstk_gpu_evaluate_batch_device(self.handle(t.device.index), t.data_ptr(), ld,
                                                   q, self.order, out_t.data_ptr(), s.cuda_stream,
                                                   C.byref(err)), err)
        return out_t

    def mode_values(self, mode: int, x) -> np.ndarray:
        """model.cpp:71-94; scalar x -> vector r_mode, array x -> (n, r_mode)."""
        scalar = np.ndim(x) == 0
        xs = np.ascontiguousarray(np.atleast_1d(np.asarray(x, dtype=np.float64)))
        if not (0 <= mode < self.order):
            raise make_error(1, "mode out of range")
        r = self.ranks[mode]
        out = np.zeros((xs.size, r), order="F")
        err = Err()
        check(lib().fstk_gpu_mode_values(self.handle(), mode, dptr(xs), xs.size, dptr(out),
                                         C.byref(err)), err)
        return out[0] if scalar else out

    # -- accounting (model.cpp:229-250) ------------------------------------------
    def storage(self) -> dict:
        nnz = sum(len(fn.coeffs) for m in self._modes for fn in m)
        coeff = int(np.prod(self.ranks)) + nnz
        return {"coefficients": coeff, "value_bytes": 8 * coeff, "index_bytes": 4 * nnz,
                "total_bytes": 8 * coeff + 4 * nnz}

    def compression_ratio(self, original_point_count: int, include_indices: bool = True) -> float:
        if original_point_count <= 0:
            raise make_error(1, "original point count must be positive")
        s = self.storage()
        b = s["total_bytes"] if include_indices else s["value_bytes"]
        return original_point_count * 8.0 / b

    def save(self, path: str):
        save_model(self, path)


class _Handle:
    def __init__(self, ptr):
        self.ptr = ptr

    def __del__(self):
        try:
            if self.ptr and _lib._LIB is not None:
                _lib._LIB.fstk_gpu_model_destroy(self.ptr)
        except Exception:
            pass
        self.ptr = None


def _current_device() -> int:
    try:
        import torch

        if torch.cuda.is_available():
            return torch.cuda.current_device()
    except Exception:
        pass
    return 0


# ------------------------------------------------------------- FSTK I/O ---
def _header_json(model: Model) -> str:
    """JSON header (model.cpp:282-309); nlohmann::json objects are key-sorted."""
    modes = []
    for m in model.modes:
        jm = []
        for fn in m:
            b = fn.basis
            jm.append({"degree": b.degree, "family": b.family, "flagged": bool(fn.flagged),
                       "hi": b.hi, "lambda": fn.chosen_lambda, "lo": b.lo, "loo": fn.loo_error,
                       "nnz": len(fn.coeffs), "residual": fn.residual_rel,
                       "resolution": b.resolution})
        modes.append(jm)
    md = model.metadata
    meta = {"achieved_error": md.achieved_error, "d": model.order, "epsilon": md.epsilon,
            "flagged_fits": md.flagged_fits,
            "grid_sizes": list(md.grid_sizes), "modes": modes, "provenance": md.provenance,
            "ranks": model.ranks}
    return json.dumps(meta, separators=(",", ":"), sort_keys=True, ensure_ascii=False,
                      allow_nan=True)


# eval_basis models, least recently used last out.  Each is a one-mode
# model holding only its coefficient tables (the evaluation workspaces are
# allocated on a model's first evaluate call, which eval_basis never makes).
_BASIS_MODELS: "collections.OrderedDict" = collections.OrderedDict()
_BASIS_MODELS_MAX = 32


def eval_basis(spec: "BasisSpec", x):
    """fstk.eval_basis (basis.cpp:226-234, module.cpp:152-156): the
    spec.dimension() basis values at x (scalar -> vector, array -> (n, dim)).
    Runs on the GPU through the C-ABI: a cached one-mode model whose function
    j is basis element j with coefficient 1.0, read out with mode_values
    (bit-exact: 0 + 1.0 * phi_j = phi_j).  Domain errors as the reference."""
    key = (spec.family, spec.degree, spec.resolution, spec.lo, spec.hi)
    m = _BASIS_MODELS.get(key)
    if m is None:
        spec.validate()
        n = spec.dimension()
        fns = [ModeFunction(spec, [(j, 1.0)]) for j in range(n)]
        m = Model(np.ones(n), [fns], ModelMetadata(grid_sizes=[0]))
        _BASIS_MODELS[key] = m
        while len(_BASIS_MODELS) > _BASIS_MODELS_MAX:
            _BASIS_MODELS.popitem(last=False)
    else:
        _BASIS_MODELS.move_to_end(key)
    return m.mode_values(0, x)


def evaluate_fields(models, points, device=None) -> np.ndarray:
    """Several models at one shared point set (BASELINE C5's visualisation
    stream): the points travel to the GPU once and every field is evaluated
    from HBM through fstk_gpu_evaluate_batch_device.  Returns (Q, n_fields),
    column f bit-identical to models[f].evaluate_batch(points)."""
    import torch

    models = list(models)
    if not models:
        raise make_error(1, "no models")
    d = models[0].order
    if any(m.order != d for m in models):
        raise make_error(2, "models of different order")
    p = np.asarray(points, dtype=np.float64)
    if p.ndim != 2 or p.shape[1] != d:
        raise make_error(1, "points must be Q x d")
    dev = torch.device("cuda", device if device is not None else torch.cuda.current_device())
    pt = torch.from_numpy(np.ascontiguousarray(p.T)).to(dev)  # (d, Q): the Q x d col-major buffer
    nf, q = len(models), p.shape[0]
    out = torch.empty((nf, q), dtype=torch.float64, device=dev)
    # Field f's values stream back to pinned host memory on a copy stream
    # while field f+1 is evaluated; only the last field's read-back is exposed.
    host = torch.empty((nf, q), dtype=torch.float64, pin_memory=True)
    comp = torch.cuda.current_stream(dev)
    copy = torch.cuda.Stream(dev)
    for f, m in enumerate(models):
        m.evaluate_device(pt, out[f])
        ev = torch.cuda.Event()
        ev.record(comp)
        copy.wait_event(ev)
        with torch.cuda.stream(copy):
            host[f].copy_(out[f], non_blocking=True)
    copy.synchronize()
    return host.numpy().T


def save_model(model: Model, path: str):
    """model.cpp:280-333 / format.md:56-69."""
    header = _header_json(model).encode("utf-8")
    try:
        with open(path, "wb") as f:
            f.write(FSTK_MAGIC)
            f.write(struct.pack("<IQ", FSTK_VERSION, len(header)))
            f.write(header)
            f.write(np.asarray(model._core.reshape(-1, order="F"), "<f8").tobytes())
            for m in model.modes:
                for fn in m:
                    f.write(struct.pack("<I", len(fn.coeffs)))
                    f.write(np.asarray([i for i, _ in fn.coeffs], "<u4").tobytes())
                    f.write(np.asarray([c for _, c in fn.coeffs], "<f8").tobytes())
    except OSError as e:
        raise FstkIOError("Io", f"cannot open for write: {path}") from e


def load_model(path: str) -> Model:
    """model.cpp:335-426."""
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError as e:
        raise FstkIOError("Io", f"cannot open: {path}") from e

    def dec(msg):
        return FstkIOError("Decode", msg)

    if len(data) < 4 or data[:4] != FSTK_MAGIC:
        raise dec(f"not a FSTK model file: {path}")
    if len(data) < 8 or struct.unpack_from("<I", data, 4)[0] != FSTK_VERSION:
        raise dec("unsupported FSTK version")
    if len(data) < 16:
        raise dec("bad FSTK header length")
    hlen = struct.unpack_from("<Q", data, 8)[0]
    if not (0 < hlen < (1 << 30)):
        raise dec("bad FSTK header length")
    off = 16
    if off + hlen > len(data):
        raise dec("FSTK header truncated")
    try:
        meta = json.loads(data[off:off + hlen].decode("utf-8"))
    except Exception as e:
        raise dec(f"FSTK metadata is not valid JSON: {e}")
    off += hlen
    try:
        d = int(meta["d"])
        if not (1 <= d <= K_MAX_ORDER):
            raise dec("bad model order")
        ranks = [int(r) for r in meta["ranks"]]
        if len(ranks) != d:
            raise dec("rank list does not match order")
        md = ModelMetadata([int(g) for g in meta["grid_sizes"]], float(meta["epsilon"]),
                           float(meta["achieved_error"]), int(meta["flagged_fits"]),
                           str(meta["provenance"]))
        rtot = int(np.prod(ranks))
        if off + 8 * rtot > len(data):
            raise dec("FSTK core truncated")
        core = np.frombuffer(data, "<f8", rtot, off).astype(np.float64)
        off += 8 * rtot
        jmodes = meta["modes"]
        if len(jmodes) != d:
            raise dec("mode list does not match order")
        modes = []
        for k in range(d):
            jm = jmodes[k]
            if len(jm) != ranks[k]:
                raise dec("function count does not match rank")
            fns = []
            for jf in jm:
                fam = jf["family"]
                if fam not in ("legendre", "wavelet"):
                    raise dec(f"unknown basis family: {fam}")
                b = BasisSpec(fam, int(jf["degree"]), int(jf["resolution"]), float(jf["lo"]),
                              float(jf["hi"]))
                b.validate()
                nnz_meta = int(jf["nnz"])
                if off + 4 > len(data):
                    raise dec("FSTK coefficient count mismatch")
                nnz = struct.unpack_from("<I", data, off)[0]
                off += 4
                if nnz != nnz_meta:
                    raise dec("FSTK coefficient count mismatch")
                if off + 12 * nnz > len(data):
                    raise dec("FSTK coefficients truncated")
                idx = np.frombuffer(data, "<u4", nnz, off)
                off += 4 * nnz
                val = np.frombuffer(data, "<f8", nnz, off)
                off += 8 * nnz
                fns.append(ModeFunction(b, [(int(i), float(c)) for i, c in zip(idx, val)],
                                        float(jf["lambda"]), float(jf["loo"]),
                                        float(jf["residual"]), bool(jf["flagged"])))
            modes.append(fns)
        if off != len(data):
            raise dec("FSTK trailing bytes")
    except FstkIOError:
        raise
    except (KeyError, TypeError, ValueError) as e:
        if isinstance(e, FstkValueError):
            raise
        raise dec(f"FSTK metadata missing fields: {e}")
    return Model(core.reshape(ranks, order="F"), modes, md)
