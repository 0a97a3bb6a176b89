"""The C++ shim (include/fstk_gpu.hpp) driven on the GPU the way the
reference's C++ callers would use it (pipeline.cpp:473 -> reestimate_core,
randls.cpp:360-383; pipeline.cpp:519 -> evaluate_batch, model.cpp:208-227):
a C++ program builds a model of the reference's shape (the member names of
model.hpp:33-59 / lars.hpp:41-50 / basis.hpp:22-38), flattens it through the
shim, evaluates a batch, a single point, mode values, refits the core and
provokes a Domain error -- all through libfstk_gpu.so -- and the results are
checked against the CPU oracle."""
import os
import struct
import subprocess

import numpy as np
import pytest

from conftest import ROOT, rel
from paper_1907_05884_b200 import synth

pytestmark = pytest.mark.gpu

SRC = r'''
#include <cstdio>
#include <cstdint>
#include <fstream>
#include <utility>
#include <vector>
#include "fstk_gpu.hpp"
namespace ref {  // the reference's member names (model.hpp / lars.hpp / basis.hpp), not its code
enum class BasisFamily : unsigned char { Legendre = 0, Wavelet = 1 };
struct BasisSpec { BasisFamily family; int degree; int resolution; double lo, hi; };
struct SparseFit { BasisSpec basis; std::vector<std::pair<std::uint32_t, double>> coeffs; };
struct ModeFunction { SparseFit fit; bool flagged = false; };
struct DenseTensor { std::vector<double> v; const double* data() const { return v.data(); } };
struct FunctionalSparseTuckerModel {
  std::vector<std::size_t> r; DenseTensor c; std::vector<std::vector<ModeFunction>> m;
  int order() const { return (int)r.size(); }
  const std::vector<std::size_t>& ranks() const { return r; }
  const DenseTensor& core() const { return c; }
  const std::vector<std::vector<ModeFunction>>& modes() const { return m; }
};
}
template <class T> T rd(std::ifstream& f) { T x; f.read(reinterpret_cast<char*>(&x), sizeof(T)); return x; }
template <class T> void rdv(std::ifstream& f, std::vector<T>& v, size_t n) {
  v.resize(n); f.read(reinterpret_cast<char*>(v.data()), n * sizeof(T)); }
template <class T> void wrv(std::ofstream& f, const std::vector<T>& v) {
  f.write(reinterpret_cast<const char*>(v.data()), v.size() * sizeof(T)); }
int main(int argc, char** argv) {
  std::ifstream in(argv[1], std::ios::binary);
  ref::FunctionalSparseTuckerModel md;
  const int d = rd<int32_t>(in);
  size_t total = 1;
  for (int k = 0; k < d; ++k) { md.r.push_back((size_t)rd<int64_t>(in)); total *= md.r.back(); }
  rdv(in, md.c.v, total);
  md.m.resize(d);
  for (int k = 0; k < d; ++k)
    for (size_t j = 0; j < md.r[k]; ++j) {
      ref::ModeFunction fn;
      fn.fit.basis.family = (ref::BasisFamily)rd<int32_t>(in);
      fn.fit.basis.degree = rd<int32_t>(in);
      fn.fit.basis.resolution = rd<int32_t>(in);
      fn.fit.basis.lo = rd<double>(in);
      fn.fit.basis.hi = rd<double>(in);
      const uint32_t nnz = rd<uint32_t>(in);
      for (uint32_t e = 0; e < nnz; ++e) {
        const uint32_t i = rd<uint32_t>(in);
        fn.fit.coeffs.emplace_back(i, rd<double>(in));
      }
      md.m[k].push_back(fn);
    }
  const int64_t q = rd<int64_t>(in);
  std::vector<double> pts, vals;
  rdv(in, pts, (size_t)q * d);   // Eigen Q x d column-major
  rdv(in, vals, (size_t)q);
  const uint64_t seed = rd<uint64_t>(in);

  auto gm = fstk_gpu_shim::Model::from_reference(md);
  const std::vector<double> y = gm.evaluate_batch(pts.data(), q, d);
  std::vector<double> p0(d);
  for (int k = 0; k < d; ++k) p0[k] = pts[(size_t)k * q + 3];
  const double y3 = gm.evaluate(p0);
  std::vector<double> mv(md.r[0] * 5);
  std::vector<double> xs = {0.0, 0.25, 0.5, 0.75, 1.0};
  gm.mode_values(0, xs.data(), 5, mv.data());
  fstk_sketch_cfg cfg = fstk_gpu_shim::default_sketch_config();
  cfg.seed = seed;
  fstk_reestimate_info info{};
  const std::vector<double> core =
      fstk_gpu_shim::reestimate_core(gm, pts.data(), vals.data(), q, d, cfg, (int64_t)total, &info);
  // Domain error (basis.cpp:218-219): point 5 of mode 1 far outside [0, 1].
  std::vector<double> bad = pts;
  bad[(size_t)1 * q + 5] = 1.5;
  int kind = -1, mode = -1; long long index = -1; double value = 0.0;
  try {
    gm.evaluate_batch(bad.data(), q, d);
  } catch (const fstk_gpu_shim::Error& e) {
    kind = e.kind(); mode = e.mode(); index = (long long)e.index(); value = e.value();
  }
  // interpolate_to_grid through the shim: the cloud (pts, vals) onto 7 x 6 x 5.
  fstk_interp_report rep{};
  const std::vector<double> grid = fstk_gpu_shim::interpolate_to_grid(
      pts.data(), vals.data(), q, d, nullptr, nullptr, {7, 6, 5}, {0.0, 0.0, 0.0}, {1.0, 1.0, 1.0}, 0, 2.0, &rep);
  std::ofstream out(argv[2], std::ios::binary);
  wrv(out, grid);
  wrv(out, y);
  out.write(reinterpret_cast<const char*>(&y3), 8);
  wrv(out, mv);
  wrv(out, core);
  const double res[2] = {info.residual_before, info.residual_after};
  out.write(reinterpret_cast<const char*>(res), 16);
  const int32_t rk = info.rank_deficient;
  out.write(reinterpret_cast<const char*>(&rk), 4);
  out.write(reinterpret_cast<const char*>(&kind), 4);
  out.write(reinterpret_cast<const char*>(&mode), 4);
  out.write(reinterpret_cast<const char*>(&index), 8);
  out.write(reinterpret_cast<const char*>(&value), 8);
  std::printf("ok\n");
  return 0;
}
'''


def _write_inputs(path, m, pts, vals, seed):
    f = m.flat()
    with open(path, "wb") as fh:
        fh.write(struct.pack("<i", f.d))
        fh.write(np.asarray(f.ranks, np.int64).tobytes())
        fh.write(np.asarray(f.core, np.float64).tobytes())
        off = 0
        for j in range(len(f.family)):
            fh.write(struct.pack("<iiiddI", int(f.family[j]), int(f.degree[j]), int(f.resolution[j]),
                                 float(f.lo[j]), float(f.hi[j]), int(f.nnz[j])))
            for e in range(int(f.nnz[j])):
                fh.write(struct.pack("<Id", int(f.idx[off + e]), float(f.coeffs[off + e])))
            off += int(f.nnz[j])
        q = pts.shape[0]
        fh.write(struct.pack("<q", q))
        fh.write(np.asfortranarray(pts).reshape(-1, order="F").astype(np.float64).tobytes())
        fh.write(np.asarray(vals, np.float64).tobytes())
        fh.write(struct.pack("<Q", seed))


def test_cpp_shim_evaluates_and_refits_on_the_gpu(tmp_path, O):
    m = synth.random_model((6, 5, 4), (8, 8, 8), 4, seed=31)
    q = 30_000
    pts = synth.uniform_points(q, 3, seed=32)
    vals = O.evaluate_batch(m, pts) + 1e-3 * np.random.default_rng(33).normal(size=q)
    seed = 11
    src = tmp_path / "shim_gpu.cpp"
    src.write_text(SRC)
    exe = tmp_path / "shim_gpu"
    libdir = os.path.join(ROOT, "paper_1907_05884_b200")
    r = subprocess.run(["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"), str(src),
                        "-L", libdir, "-lfstk_gpu", f"-Wl,-rpath,{libdir}",
                        "-L/usr/local/cuda/lib64", "-Wl,-rpath,/usr/local/cuda/lib64",
                        "-o", str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    inp, outp = tmp_path / "in.bin", tmp_path / "out.bin"
    _write_inputs(inp, m, pts, vals, seed)
    run = subprocess.run([str(exe), str(inp), str(outp)], capture_output=True, text=True, timeout=300)
    assert run.returncode == 0, run.stderr
    raw = outp.read_bytes()
    R = int(np.prod(m.ranks))
    o = 0

    def take(n, dt=np.float64):
        nonlocal o
        a = np.frombuffer(raw, dtype=dt, count=n, offset=o)
        o += n * np.dtype(dt).itemsize
        return a

    grid = take(7 * 6 * 5)
    y = take(q)
    y3 = take(1)[0]
    mv = take(m.ranks[0] * 5)
    core = take(R)
    res = take(2)
    rk = take(1, np.int32)[0]
    kind, mode = take(2, np.int32)
    index = take(1, np.int64)[0]
    value = take(1)[0]

    want = O.evaluate_batch(m, pts)
    assert rel(y, want) <= 1e-12
    assert y3 == y[3]  # evaluate == a batch of one, bit for bit (test_model.cpp:178-199)
    mv_o = np.stack([O.mode_values(m, 0, x) for x in (0.0, 0.25, 0.5, 0.75, 1.0)], axis=1)
    assert np.array_equal(mv.reshape(m.ranks[0], 5), mv_o)  # function-major, like fstk_gpu_mode_values
    core_o, info_o = O.reestimate_core(m, pts, vals, seed=seed)
    assert rel(core, core_o) <= 1e-9
    assert abs(res[0] - info_o["residual_before"]) <= 1e-12 * max(1.0, info_o["residual_before"])
    assert abs(res[1] - info_o["residual_after"]) <= 1e-9 * max(1.0, info_o["residual_after"])
    assert bool(rk) == info_o["rank_deficient"]
    assert kind == 3 - 1  # FSTK_E_DOMAIN = ErrorKind::Domain + 1 (error.hpp:11-19)
    assert (int(mode), int(index), float(value)) == (1, 5, 1.5)
    go, _ = O.interpolate_to_grid(pts, vals, (7, 6, 5))
    assert float(np.abs(grid - go.reshape(-1, order="F")).max()) <= 1e-12
