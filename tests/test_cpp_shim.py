"""The C++ shim (include/fstk_gpu.hpp) compiles against a mock of the
reference's model type (model.hpp:33-59 / lars.hpp:41-50 / basis.hpp:22-38
member names) and flatten() yields the descriptor the C-ABI expects.  Links
libfstk_gpu.so but makes no GPU call."""
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT

SRC = r'''
#include <cstdio>
#include <utility>
#include <vector>
#include "fstk_gpu.hpp"
namespace mock {  // the reference's member names, not its code
enum class BasisFamily : unsigned char { Legendre = 0, Wavelet = 1 };
struct BasisSpec { BasisFamily family; int degree; int resolution; double lo, hi; };
struct SparseFit { BasisSpec basis; std::vector<std::pair<unsigned, double>> coeffs; };
struct ModeFunction { SparseFit fit; bool flagged = false; };
struct Tensor { std::vector<double> v; const double* data() const { return v.data(); } };
struct Model {
  std::vector<long> r; Tensor c; std::vector<std::vector<ModeFunction>> m;
  int order() const { return (int)r.size(); }
  std::vector<long> ranks() const { return r; }
  const Tensor& core() const { return c; }
  const std::vector<std::vector<ModeFunction>>& modes() const { return m; }
};
}
int main() {
  mock::Model md;
  md.r = {2, 1};
  md.c.v = {1.5, -2.0};
  mock::BasisSpec b{mock::BasisFamily::Legendre, 3, 0, 0.0, 1.0};
  md.m = {{{{b, {{0, 1.0}, {2, 0.5}}}}, {{b, {{1, -1.0}}}}}, {{{b, {{3, 2.0}}}}}};
  const auto f = fstk_gpu_shim::flatten(md);
  const fstk_model_desc d = f.desc();
  std::printf("%d %ld %ld %g %g %u %u %u %u %u %u %g %g %g %g %d %g\n", d.d, (long)d.ranks[0],
              (long)d.ranks[1], d.core[0], d.core[1], d.nnz[0], d.nnz[1], d.nnz[2], d.indices[0],
              d.indices[1], d.indices[3], d.coeffs[0], d.coeffs[1], d.coeffs[2], d.coeffs[3],
              d.degree[2], d.hi[1]);
  fstk_sketch_cfg c = fstk_gpu_shim::default_sketch_config();
  std::printf("%llu %d %g\n", (unsigned long long)c.working_subset, c.transform,
              c.validation_fraction);
  return 0;
}
'''


def test_shim_flatten(tmp_path):
    src = tmp_path / "shim.cpp"
    src.write_text(SRC)
    exe = tmp_path / "shim"
    libdir = os.path.join(ROOT, "paper_1907_05884_b200")
    r = subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"), str(src),
                        "-L", libdir, "-lfstk_gpu", f"-Wl,-rpath,{libdir}",
                        "-L/usr/local/cuda/lib64", f"-Wl,-rpath,/usr/local/cuda/lib64",
                        "-o", str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    a, b = out.stdout.strip().splitlines()
    assert a.split() == "2 2 1 1.5 -2 2 1 1 0 2 3 1 0.5 -1 2 3 1".split()
    assert b.split() == ["1048576", "0", "0.05"]
