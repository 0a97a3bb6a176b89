"""Point clouds: FPTC (binary) and CSV I/O, mirroring proj/src/ingest.cpp:19-49
(PointCloud::from_data / validate) and :600-754 (CSV + FPTC readers/writers,
docs/format.md:29-55), FPTC ingest straight to a device SoA buffer
(SURVEY 8f-4): the point-major payload is uploaded as-is and transposed by
fstk_gpu_point_major_to_soa on the GPU, and scattered-to-grid IDW
interpolation (interpolate_to_grid, ingest.cpp:265-383) on the GPU
(fstk_idw.cu).
"""
from __future__ import annotations

import ctypes as C
import struct
from dataclasses import dataclass

import numpy as np

from ._lib import Err, FstkIOError, InterpReport, check, lib, make_error

FPTC_MAGIC = b"FPTC"
FPTC_VERSION = 1
K_MAX_ORDER = 8


@dataclass
class PointCloud:
    points: np.ndarray   # Q x d, column-major (Eigen layout)
    values: np.ndarray   # Q
    box_lo: np.ndarray   # d
    box_hi: np.ndarray   # d

    @property
    def dim(self) -> int:
        return self.points.shape[1]

    @property
    def count(self) -> int:
        return self.points.shape[0]

    @staticmethod
    def from_data(points, values) -> "PointCloud":
        """ingest.cpp:19-31: bounding box from the data, then validate."""
        p = np.asfortranarray(np.asarray(points, dtype=np.float64))
        v = np.ascontiguousarray(np.asarray(values, dtype=np.float64))
        if p.ndim != 2 or not (1 <= p.shape[1] <= K_MAX_ORDER):
            raise make_error(2, "point cloud dimension must be in [1, 8]")
        if p.shape[0] < 1:
            raise make_error(4, "point cloud is empty")
        pc = PointCloud(p, v, p.min(axis=0), p.max(axis=0))
        pc.validate()
        return pc

    def validate(self):
        """ingest.cpp:33-49."""
        if self.points.shape[0] != self.values.shape[0]:
            raise make_error(2, "point/value count mismatch")
        if self.points.shape[0] < 1:
            raise make_error(4, "point cloud is empty")
        if not (1 <= self.dim <= K_MAX_ORDER):
            raise make_error(2, "point cloud dimension must be in [1, 8]")
        if self.box_lo.size != self.dim or self.box_hi.size != self.dim:
            raise make_error(2, "bounding box dimension mismatch")
        if not np.all(np.isfinite(self.points)):
            raise make_error(4, "point coordinates must be finite")
        if not np.all(np.isfinite(self.values)):
            raise make_error(4, "sample values must be finite")
        if np.any(self.points.min(axis=0) < self.box_lo) or np.any(
                self.points.max(axis=0) > self.box_hi):
            raise make_error(4, "bounding box does not cover the points")


# ------------------------------------------------------------------ FPTC ---
def write_cloud_binary(pc: PointCloud, path: str):
    """ingest.cpp:689-704 / format.md:29-44."""
    pc.validate()
    try:
        with open(path, "wb") as f:
            f.write(FPTC_MAGIC)
            f.write(struct.pack("<IIQ", FPTC_VERSION, pc.dim, pc.count))
            f.write(np.asarray(pc.box_lo, "<f8").tobytes())
            f.write(np.asarray(pc.box_hi, "<f8").tobytes())
            f.write(np.ascontiguousarray(pc.points, dtype="<f8").tobytes())  # point-major
            f.write(np.asarray(pc.values, "<f8").tobytes())
    except OSError as e:
        raise FstkIOError("Io", f"cannot open for write: {path}") from e


def _read_fptc_raw(path: str):
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError as e:
        raise FstkIOError("Io", f"cannot open: {path}") from e
    dec = lambda m: FstkIOError("Decode", m)
    if len(data) < 4 or data[:4] != FPTC_MAGIC:
        raise dec(f"not a FPTC file: {path}")
    if len(data) < 8 or struct.unpack_from("<I", data, 4)[0] != FPTC_VERSION:
        raise dec("unsupported FPTC version")
    if len(data) < 12:
        raise dec("bad FPTC dimension")
    d = struct.unpack_from("<I", data, 8)[0]
    if not (1 <= d <= K_MAX_ORDER):
        raise dec("bad FPTC dimension")
    if len(data) < 20:
        raise dec("bad FPTC point count")
    q = struct.unpack_from("<Q", data, 12)[0]
    if not (1 <= q < (1 << 40)):
        raise dec("bad FPTC point count")
    need = 20 + 16 * d + 8 * q * d + 8 * q
    if len(data) < need:
        raise dec("FPTC truncated")
    if len(data) > need:
        raise dec(f"FPTC trailing bytes: {path}")
    off = 20
    lo = np.frombuffer(data, "<f8", d, off).copy()
    hi = np.frombuffer(data, "<f8", d, off + 8 * d).copy()
    off += 16 * d
    pm = np.frombuffer(data, "<f8", q * d, off).reshape(q, d)  # point-major view
    vals = np.frombuffer(data, "<f8", q, off + 8 * q * d).copy()
    return pm, vals, lo, hi


def read_cloud_binary(path: str) -> PointCloud:
    """ingest.cpp:706-742 (box stored, not recomputed: bit-exact round trip)."""
    pm, vals, lo, hi = _read_fptc_raw(path)
    pc = PointCloud(np.asfortranarray(pm), vals, lo, hi)
    pc.validate()
    return pc


def read_cloud_device(path: str, device=None):
    """FPTC -> device SoA without a host transpose: returns (points_t (d, Q)
    CUDA float64, values_t (Q,), box_lo, box_hi).  points_t is exactly the
    column-major Q x d buffer the C-ABI takes (Model.evaluate_device)."""
    import torch

    pm, vals, lo, hi = _read_fptc_raw(path)
    if not (np.all(np.isfinite(vals))):
        raise make_error(4, "sample values must be finite")
    dev = torch.device("cuda", device if device is not None else torch.cuda.current_device())
    src = torch.from_numpy(np.ascontiguousarray(pm)).to(dev)
    q, d = pm.shape
    out = torch.empty((d, q), dtype=torch.float64, device=dev)
    err = Err()
    check(lib().fstk_gpu_point_major_to_soa(src.data_ptr(), q, d, out.data_ptr(),
                                            torch.cuda.current_stream(dev).cuda_stream,
                                            C.byref(err)), err)
    return out, torch.from_numpy(vals).to(dev), lo, hi


# ------------------------------------------------------------------- CSV ---
def _fmt(v: float) -> str:
    return "%.17g" % v


def write_cloud_csv(pc: PointCloud, path: str):
    """ingest.cpp:600-619: header y0,...,value; %.17g round-trips f64."""
    pc.validate()
    try:
        with open(path, "w") as f:
            f.write(",".join([f"y{k}" for k in range(pc.dim)] + ["value"]) + "\n")
            for q in range(pc.count):
                f.write(",".join([_fmt(x) for x in pc.points[q]] + [_fmt(pc.values[q])]) + "\n")
    except OSError as e:
        raise FstkIOError("Io", f"cannot open for write: {path}") from e


def _csv_lines(path: str):
    try:
        with open(path, "r") as f:
            return f.read().split("\n")
    except OSError as e:
        raise FstkIOError("Io", f"cannot open: {path}") from e


def _parse(s: str, path: str) -> float:
    try:
        return float(s.strip())
    except ValueError:
        raise FstkIOError("Decode", f"bad number in {path}")


def read_cloud_csv(path: str) -> PointCloud:
    """ingest.cpp:621-652."""
    lines = _csv_lines(path)
    if not lines or lines == [""]:
        raise FstkIOError("Decode", f"empty CSV: {path}")
    header = lines[0].split(",")
    if len(header) < 2:
        raise FstkIOError("Decode", f"bad CSV header: {path}")
    d = len(header) - 1
    if d > K_MAX_ORDER:
        raise FstkIOError("Decode", f"too many CSV columns: {path}")
    rows = []
    for ln in lines[1:]:
        if ln == "" or ln == "\r":
            continue
        fields = ln.split(",")
        if len(fields) != d + 1:
            raise FstkIOError("Decode", f"CSV row width mismatch in {path}")
        rows.append([_parse(x, path) for x in fields])
    if not rows:
        raise FstkIOError("Decode", f"CSV has no data rows: {path}")
    a = np.asarray(rows)
    return PointCloud.from_data(a[:, :d], a[:, d])


def read_points_csv(path: str, expected_dim: int) -> np.ndarray:
    """ingest.cpp:654-687: coordinates only; a trailing `value` column is ignored."""
    lines = _csv_lines(path)
    if not lines or lines == [""]:
        raise FstkIOError("Decode", f"empty CSV: {path}")
    header = lines[0].split(",")
    d = len(header)
    has_value = header[-1].rstrip("\r ") == "value"
    if has_value:
        d -= 1
    if d != expected_dim:
        raise make_error(1, f"points file has dimension {d}, expected {expected_dim}")
    rows = []
    for ln in lines[1:]:
        if ln == "" or ln == "\r":
            continue
        fields = ln.split(",")
        if len(fields) != d + (1 if has_value else 0):
            raise FstkIOError("Decode", f"CSV row width mismatch in {path}")
        rows.append([_parse(x, path) for x in fields[:d]])
    return np.asfortranarray(np.asarray(rows, dtype=np.float64).reshape(len(rows), d))


def read_cloud(path: str) -> PointCloud:
    """ingest.cpp:744-752: dispatch on the magic bytes."""
    try:
        with open(path, "rb") as f:
            magic = f.read(4)
    except OSError as e:
        raise FstkIOError("Io", f"cannot open: {path}") from e
    return read_cloud_binary(path) if magic == FPTC_MAGIC else read_cloud_csv(path)


# ------------------------------------------------- grid interpolation ---
@dataclass
class StructuredGrid:
    """ingest.hpp:28-39: sizes I_k >= 2 and intervals [lo, hi] per mode."""
    sizes: list
    intervals: list

    @property
    def dim(self) -> int:
        return len(self.sizes)

    def node(self, mode: int, i: int) -> float:
        """ingest.cpp:57-61."""
        lo, hi = self.intervals[mode]
        return lo + (hi - lo) * float(i) / float(self.sizes[mode] - 1)

    def coords(self, mode: int) -> np.ndarray:
        return np.array([self.node(mode, i) for i in range(self.sizes[mode])], dtype=np.float64)

    def validate(self):
        """ingest.cpp:70-80."""
        if not (1 <= len(self.sizes) <= K_MAX_ORDER):
            raise make_error(1, "grid dimension must be in [1, 8]")
        if len(self.sizes) != len(self.intervals):
            raise make_error(1, "grid sizes/intervals mismatch")
        for s, (lo, hi) in zip(self.sizes, self.intervals):
            if s < 2:
                raise make_error(1, "grid sizes must be >= 2")
            if not lo < hi:
                raise make_error(1, "grid intervals must be nondegenerate")

    @staticmethod
    def unit(sizes) -> "StructuredGrid":
        g = StructuredGrid(list(int(s) for s in sizes), [(0.0, 1.0)] * len(sizes))
        g.validate()
        return g


@dataclass
class InterpolationOptions:
    """ingest.hpp:44-47."""
    neighbors: int = 0    # 0 -> 2d + 2
    power: float = 2.0    # inverse-distance exponent


@dataclass
class InterpolationReport:
    """ingest.hpp:49-54."""
    box_covered: bool = True
    max_nearest_distance: float = 0.0
    extrapolated_fraction: float = 0.0


def interpolate_to_grid(pc: PointCloud, grid: StructuredGrid, options: InterpolationOptions | None = None,
                        device=None, return_neighbors: bool = False):
    """interpolate_to_grid (ingest.cpp:265-383) on the GPU (fstk_idw.cu):
    kNN inverse-distance weighting over the reference's spatial index.
    Returns (values with shape grid.sizes, mode-0 fastest like DenseTensor;
    InterpolationReport), plus the (n_nodes, k) retained sample ids in
    ascending (distance, id) order with return_neighbors."""
    opts = options or InterpolationOptions()
    pc.validate()
    grid.validate()
    if pc.dim != grid.dim:
        raise make_error(2, "cloud/grid dimension mismatch")
    d = pc.dim
    sizes = np.ascontiguousarray(grid.sizes, dtype=np.int64)
    glo = np.ascontiguousarray([a for a, _ in grid.intervals], dtype=np.float64)
    ghi = np.ascontiguousarray([b for _, b in grid.intervals], dtype=np.float64)
    n = int(np.prod(sizes))
    k = int(opts.neighbors) if opts.neighbors > 0 else 2 * d + 2
    out = np.empty(n, dtype=np.float64)
    nbr = np.empty(n * k, dtype=np.uint32) if return_neighbors else None
    pts = np.asfortranarray(pc.points, dtype=np.float64)
    vals = np.ascontiguousarray(pc.values, dtype=np.float64)
    blo = np.ascontiguousarray(pc.box_lo, dtype=np.float64)
    bhi = np.ascontiguousarray(pc.box_hi, dtype=np.float64)
    if device is None:
        import torch

        device = torch.cuda.current_device() if torch.cuda.is_available() else 0
    rep = InterpReport()
    err = Err()
    check(lib().fstk_gpu_interpolate_to_grid(
        pts.ctypes.data, vals.ctypes.data, pc.count, d, blo.ctypes.data, bhi.ctypes.data,
        sizes.ctypes.data, glo.ctypes.data, ghi.ctypes.data, int(opts.neighbors), float(opts.power),
        out.ctypes.data, C.byref(rep), nbr.ctypes.data if nbr is not None else None, int(device),
        C.byref(err)), err)
    report = InterpolationReport(bool(rep.box_covered), float(rep.max_nearest_distance),
                                 float(rep.extrapolated_fraction))
    tensor = out.reshape(tuple(int(x) for x in sizes), order="F")
    if return_neighbors:
        return tensor, report, nbr.reshape(n, k)
    return tensor, report
