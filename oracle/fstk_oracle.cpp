// ============================================================================
// fstk CPU ORACLE — TEST INFRASTRUCTURE ONLY.
//
// This file is a line-by-line CPU restatement of the reference hot path
// (evaluation + randomized-LS refit) of /root/reference/proj.  It exists so
// that tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg can
// CHECK the B200 product path.  Nothing in paper_1907_05884_b200/ may import,
// link or call it; the product fails loudly if its CUDA library is missing.
//
// Pinning: the Eigen-free reference files (rng.cpp, transforms.cpp,
// parallel.cpp) are compiled as-is into oracle/_ref/libfstk_ref.so by
// oracle/Makefile, and tests/test_oracle_pins.py checks the restatements below
// against them bit for bit (plus the committed golden vectors in
// tests/golden/).  The Eigen-dependent functions (Legendre recurrence,
// mode_values, contract_core GEMV chain, ColPivHouseholderQR) cannot be built
// here (Eigen 3.3 is REQUIRED by proj/CMakeLists.txt:14 and absent), so they
// are restated and pinned by the reference's own known-answer tests
// (test_basis.cpp:37-63,165-183; test_model.cpp:113-137,178-210;
// test_randls.cpp:75-206).  Eigen's GEMV summation order is not reproducible
// without Eigen: the restatement uses the column-axpy order, and parity with
// the GPU path is therefore a tolerance (1e-12 relative L2), not bit-exact.
//
// Built with g++ -O3 -ffp-contract=off, x86-64 baseline (no FMA), matching the
// reference's Release build (proj/CMakeLists.txt:8-10, no -march).
// ============================================================================
#include <algorithm>
#include <atomic>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <exception>
#include <functional>
#include <limits>
#include <map>
#include <mutex>
#include <numeric>
#include <random>
#include <string>
#include <thread>
#include <utility>
#include <vector>

namespace oracle {

// ---------------------------------------------------------------- errors ---
// ErrorKind order follows proj/include/fstk/error.hpp:11-19.
enum ErrorKind { Parameter = 0, Shape, Domain, Data, Io, Decode, Compute };

struct Error {
  int kind;
  std::string msg;
};

[[noreturn]] static void fail(int kind, const std::string& m) {
  throw Error{kind, m};
}
static void require(bool c, int kind, const char* m) {
  if (!c) fail(kind, m);
}

// --------------------------------------------------------- parallel_for ---
// proj/src/parallel.cpp:12-65.
static std::atomic<int> g_max_threads{0};

static int max_threads() {
  const int n = g_max_threads.load();
  if (n > 0) return n;
  const unsigned h = std::thread::hardware_concurrency();
  return h == 0 ? 1 : static_cast<int>(h);
}

static void parallel_for(std::size_t n,
                         const std::function<void(std::size_t, std::size_t)>& fn) {
  if (n == 0) return;
  const int threads = static_cast<int>(
      std::min<std::size_t>(static_cast<std::size_t>(max_threads()), n));
  if (threads <= 1) {
    fn(0, n);
    return;
  }
  const std::size_t chunk =
      std::max<std::size_t>(1, n / (4 * static_cast<std::size_t>(threads)));
  std::atomic<std::size_t> cursor{0};
  std::mutex err_mutex;
  std::exception_ptr first_error;
  auto worker = [&] {
    for (;;) {
      const std::size_t begin = cursor.fetch_add(chunk);
      if (begin >= n) return;
      const std::size_t end = std::min(begin + chunk, n);
      try {
        fn(begin, end);
      } catch (...) {
        std::lock_guard<std::mutex> lock(err_mutex);
        if (!first_error) first_error = std::current_exception();
        return;
      }
    }
  };
  std::vector<std::thread> pool;
  pool.reserve(static_cast<std::size_t>(threads - 1));
  for (int t = 0; t < threads - 1; ++t) pool.emplace_back(worker);
  worker();
  for (auto& th : pool) th.join();
  if (first_error) std::rethrow_exception(first_error);
}

// ------------------------------------------------------------------- RNG ---
// proj/include/fstk/rng.hpp:21-48 and proj/src/rng.cpp:11-61.
struct Rng {
  std::mt19937_64 engine;
  explicit Rng(std::uint64_t seed) : engine(seed) {}
  std::uint64_t next_u64() { return engine(); }
  std::uint64_t uniform_index(std::uint64_t n) {  // rng.cpp:11-19
    require(n > 0, Parameter, "uniform_index: n must be positive");
    const std::uint64_t limit = UINT64_MAX - UINT64_MAX % n;
    std::uint64_t x;
    do {
      x = next_u64();
    } while (x >= limit);
    return x % n;
  }
  double uniform_double() {  // rng.hpp:31-33
    return static_cast<double>(next_u64() >> 11) * 0x1.0p-53;
  }
  double sign() { return (next_u64() & 1ull) ? -1.0 : 1.0; }  // rng.hpp:34
  // rng.cpp:36-53: partial Fisher-Yates over an iota table, prefix sorted.
  std::vector<std::uint64_t> sample_without_replacement(std::uint64_t n,
                                                        std::uint64_t k) {
    if (k >= n) {
      std::vector<std::uint64_t> all(n);
      std::iota(all.begin(), all.end(), 0);
      return all;
    }
    std::vector<std::uint64_t> idx(n);
    std::iota(idx.begin(), idx.end(), 0);
    for (std::uint64_t i = 0; i < k; ++i) {
      const std::uint64_t j = i + uniform_index(n - i);
      std::swap(idx[i], idx[j]);
    }
    idx.resize(k);
    std::sort(idx.begin(), idx.end());
    return idx;
  }
};

// rng.cpp:55-61 (splitmix64 finalizer over seed ^ tag).
static std::uint64_t mix_seed(std::uint64_t seed, std::uint64_t tag) {
  std::uint64_t z = (seed ^ tag) + 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

// ------------------------------------------------------------ transforms ---
// proj/src/transforms.cpp:20-104.
static bool is_pow2(std::size_t n) { return n != 0 && (n & (n - 1)) == 0; }

static std::size_t next_pow2(std::size_t n) {  // :20-24
  std::size_t p = 1;
  while (p < n) p <<= 1;
  return p;
}

using cd = std::complex<double>;

static void fft_pow2(cd* x, std::size_t n, bool inverse) {  // :26-53
  require(is_pow2(n), Parameter, "transform length must be a power of two");
  for (std::size_t i = 1, j = 0; i < n; ++i) {  // bit reversal
    std::size_t bit = n >> 1;
    for (; j & bit; bit >>= 1) j ^= bit;
    j ^= bit;
    if (i < j) std::swap(x[i], x[j]);
  }
  for (std::size_t len = 2; len <= n; len <<= 1) {
    const double ang = (inverse ? 2.0 : -2.0) * M_PI / static_cast<double>(len);
    const cd wlen(std::cos(ang), std::sin(ang));
    for (std::size_t i = 0; i < n; i += len) {
      cd w(1.0, 0.0);  // recurrence twiddles, :40-45
      for (std::size_t k = 0; k < len / 2; ++k) {
        const cd u = x[i + k];
        const cd v = x[i + k + len / 2] * w;
        x[i + k] = u + v;
        x[i + k + len / 2] = u - v;
        w *= wlen;
      }
    }
  }
  if (inverse) {
    const double inv = 1.0 / static_cast<double>(n);
    for (std::size_t i = 0; i < n; ++i) x[i] *= inv;
  }
}

static void unitary_fft(cd* x, std::size_t n, bool inverse) {  // :55-67
  require(is_pow2(n), Parameter, "transform length must be a power of two");
  if (inverse) {
    fft_pow2(x, n, true);
    const double s = std::sqrt(static_cast<double>(n));
    for (std::size_t i = 0; i < n; ++i) x[i] *= s;
  } else {
    fft_pow2(x, n, false);
    const double s = 1.0 / std::sqrt(static_cast<double>(n));
    for (std::size_t i = 0; i < n; ++i) x[i] *= s;
  }
}

static void wht_orthonormal(double* x, std::size_t n) {  // :69-83
  require(is_pow2(n), Parameter, "transform length must be a power of two");
  for (std::size_t len = 1; len < n; len <<= 1)
    for (std::size_t i = 0; i < n; i += len << 1)
      for (std::size_t k = 0; k < len; ++k) {
        const double a = x[i + k];
        const double b = x[i + k + len];
        x[i + k] = a + b;
        x[i + k + len] = a - b;
      }
  const double s = 1.0 / std::sqrt(static_cast<double>(n));
  for (std::size_t i = 0; i < n; ++i) x[i] *= s;
}

static void dct2_orthonormal(double* x, std::size_t n) {  // :85-104
  require(is_pow2(n), Parameter, "transform length must be a power of two");
  if (n == 1) return;
  std::vector<cd> v(n);  // Makhoul reorder
  for (std::size_t m = 0; m < n / 2; ++m) {
    v[m] = x[2 * m];
    v[n - 1 - m] = x[2 * m + 1];
  }
  fft_pow2(v.data(), n, false);
  const double c0 = std::sqrt(1.0 / static_cast<double>(n));
  const double ck = std::sqrt(2.0 / static_cast<double>(n));
  for (std::size_t k = 0; k < n; ++k) {
    const double ang =
        -M_PI * static_cast<double>(k) / (2.0 * static_cast<double>(n));
    const cd rot(std::cos(ang), std::sin(ang));
    const double val = (rot * v[k]).real();
    x[k] = (k == 0 ? c0 : ck) * val;
  }
}

// ----------------------------------------------------------------- basis ---
// proj/include/fstk/basis.hpp:22-38, proj/src/basis.cpp:30-61,215-234.
struct BasisSpec {
  int family = 0;  // 0 Legendre, 1 Wavelet
  int degree = 0;
  int resolution = 0;
  double lo = -1.0, hi = 1.0;
  int dimension() const {
    return family == 0 ? degree + 1 : (degree + 1) << resolution;
  }
  bool operator==(const BasisSpec& o) const {
    return family == o.family && degree == o.degree &&
           resolution == o.resolution && lo == o.lo && hi == o.hi;
  }
};

static void validate(const BasisSpec& spec) {  // basis.cpp:30-47
  require(spec.degree >= 0 && spec.degree <= 64, Parameter,
          "basis degree must be in [0, 64]");
  if (spec.family == 0) {
    require(spec.resolution == 0, Parameter,
            "Legendre basis has no resolution parameter");
  } else {
    require(spec.resolution >= 0 && spec.resolution <= 20, Parameter,
            "wavelet resolution must be in [0, 20]");
    require(static_cast<long long>(spec.degree + 1) << spec.resolution <=
                (1 << 24),
            Parameter, "basis dimension too large");
  }
  require(spec.lo < spec.hi, Parameter, "basis domain must satisfy lo < hi");
  require(std::isfinite(spec.lo) && std::isfinite(spec.hi), Parameter,
          "basis domain must be finite");
}

static void legendre_values(int p, double t, double* out) {  // :49-61
  double pm1 = 1.0, pm0 = t;
  out[0] = 1.0;
  if (p >= 1) out[1] = std::sqrt(3.0) * t;
  for (int n = 1; n < p; ++n) {
    const double pn1 = ((2 * n + 1) * t * pm0 - n * pm1) / (n + 1);
    pm1 = pm0;
    pm0 = pn1;
    out[n + 1] = std::sqrt(2.0 * (n + 1) + 1.0) * pn1;
  }
}

static double to_reference(const BasisSpec& spec, double x) {  // :215-222
  const double span = spec.hi - spec.lo;
  const double slack = 1e-12 * span;
  require(x >= spec.lo - slack && x <= spec.hi + slack, Domain,
          "point outside basis domain");
  const double clamped = std::min(spec.hi, std::max(spec.lo, x));
  return -1.0 + 2.0 * (clamped - spec.lo) / span;
}

// basis.cpp:63-102 (Tricomi initial guess + Newton on P_n).
static void gauss_legendre(int n, std::vector<double>& nodes, std::vector<double>& weights) {
  require(n >= 1, Parameter, "quadrature order must be positive");
  nodes.assign(n, 0.0);
  weights.assign(n, 0.0);
  const int m = (n + 1) / 2;
  for (int j = 0; j < m; ++j) {
    double x = std::cos(M_PI * (j + 0.75) / (n + 0.5));
    double dp = 0.0;
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = x;
      for (int k = 1; k < n; ++k) {
        const double p2 = ((2 * k + 1) * x * p1 - k * p0) / (k + 1);
        p0 = p1;
        p1 = p2;
      }
      dp = n * (x * p1 - p0) / (x * x - 1.0);
      const double dx = p1 / dp;
      x -= dx;
      if (std::abs(dx) < 1e-15) break;
    }
    {
      double p0 = 1.0, p1 = x;
      for (int k = 1; k < n; ++k) {
        const double p2 = ((2 * k + 1) * x * p1 - k * p0) / (k + 1);
        p0 = p1;
        p1 = p2;
      }
      dp = n * (x * p1 - p0) / (x * x - 1.0);
    }
    nodes[j] = -x;
    nodes[n - 1 - j] = x;
    const double w = 2.0 / ((1.0 - x * x) * dp * dp);
    weights[j] = w;
    weights[n - 1 - j] = w;
  }
  if (n % 2 == 1) nodes[n / 2] = 0.0;
}

// Dense column-major helper and a Householder QR returning the full m x m Q
// (stands in for Eigen::HouseholderQR::householderQ(), basis.cpp:147-148,173-174).
struct Mat {
  int r = 0, c = 0;
  std::vector<double> a;
  Mat(int rr, int cc) : r(rr), c(cc), a(static_cast<size_t>(rr) * cc, 0.0) {}
  double& operator()(int i, int j) { return a[static_cast<size_t>(j) * r + i]; }
  double operator()(int i, int j) const { return a[static_cast<size_t>(j) * r + i]; }
};

static Mat householder_q(Mat A) {
  const int m = A.r, n = A.c;
  std::vector<std::vector<double>> vs;
  std::vector<double> taus;
  for (int k = 0; k < std::min(m - 1, n); ++k) {
    double norm = 0.0;
    for (int i = k; i < m; ++i) norm += A(i, k) * A(i, k);
    norm = std::sqrt(norm);
    std::vector<double> v(m, 0.0);
    double tau = 0.0;
    if (norm > 0.0) {
      const double alpha = A(k, k) >= 0 ? -norm : norm;
      for (int i = k; i < m; ++i) v[i] = A(i, k);
      v[k] -= alpha;
      double vn = 0.0;
      for (int i = k; i < m; ++i) vn += v[i] * v[i];
      if (vn > 0.0) {
        tau = 2.0 / vn;
        for (int j = k; j < n; ++j) {
          double d = 0.0;
          for (int i = k; i < m; ++i) d += v[i] * A(i, j);
          d *= tau;
          for (int i = k; i < m; ++i) A(i, j) -= d * v[i];
        }
      }
    }
    vs.push_back(v);
    taus.push_back(tau);
  }
  Mat Q(m, m);
  for (int i = 0; i < m; ++i) Q(i, i) = 1.0;
  for (int k = static_cast<int>(vs.size()) - 1; k >= 0; --k) {
    const auto& v = vs[k];
    if (taus[k] == 0.0) continue;
    for (int j = 0; j < m; ++j) {
      double d = 0.0;
      for (int i = k; i < m; ++i) d += v[i] * Q(i, j);
      d *= taus[k];
      for (int i = k; i < m; ++i) Q(i, j) -= d * v[i];
    }
  }
  return Q;
}

// basis.cpp:116-189: mother multiwavelets of degree p in the split basis.
static Mat build_mother(int p) {
  const int n = p + 1;
  std::vector<double> qx, qw;
  gauss_legendre(2 * p + 4, qx, qw);
  const int nq = static_cast<int>(qx.size());
  Mat q(2 * n, n);
  std::vector<double> lg(n), lh(n);
  for (int side = 0; side < 2; ++side)
    for (int a = 0; a < nq; ++a) {
      const double t = qx[a];
      const double x = side == 0 ? 0.5 * (t - 1.0) : 0.5 * (t + 1.0);
      legendre_values(p, x, lg.data());
      legendre_values(p, t, lh.data());
      const double w = qw[a] * std::sqrt(2.0) / 4.0;
      for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) q(side * n + i, j) += w * lh[i] * lg[j];
    }
  const Mat full = householder_q(q);
  Mat comp(2 * n, n);
  for (int i = 0; i < 2 * n; ++i)
    for (int j = 0; j < n; ++j) comp(i, j) = full(i, n + j);
  Mat moments(n, n);
  for (int side = 0; side < 2; ++side)
    for (int a = 0; a < nq; ++a) {
      const double t = qx[a];
      const double x = side == 0 ? 0.5 * (t - 1.0) : 0.5 * (t + 1.0);
      legendre_values(p, t, lh.data());
      const double w = qw[a] * std::sqrt(2.0) / 4.0;
      double xpow = std::pow(x, p + 1);
      for (int trow = 0; trow < n; ++trow) {
        for (int i = 0; i < n; ++i) {
          const double chi_val = w * lh[i];
          for (int c = 0; c < n; ++c) moments(trow, c) += xpow * chi_val * comp(side * n + i, c);
        }
        xpow *= x;
      }
    }
  Mat mt(n, n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) mt(i, j) = moments(j, i);
  const Mat rot = householder_q(mt);
  Mat coords(2 * n, n);
  for (int i = 0; i < 2 * n; ++i)
    for (int j = 0; j < n; ++j) {
      double v = 0.0;
      for (int k = 0; k < n; ++k) v += comp(i, k) * rot(k, j);
      coords(i, j) = v;
    }
  for (int m = 0; m < n; ++m)
    for (int i = 2 * n - 1; i >= 0; --i)
      if (std::abs(coords(i, m)) > 1e-10) {
        if (coords(i, m) < 0.0)
          for (int r = 0; r < 2 * n; ++r) coords(r, m) = -coords(r, m);
        break;
      }
  return coords;
}

static const Mat& mother_wavelet(int p) {  // basis.cpp:191-198
  static std::mutex mu;
  static std::map<int, Mat> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(p);
  if (it == cache.end()) it = cache.emplace(p, build_mother(p)).first;
  return it->second;
}

static void mother_values(const Mat& mw, int p, double t, double* out) {  // :201-213
  const int n = p + 1;
  std::vector<double> leg(n);
  const int side = t < 0.0 ? 0 : 1;
  const double local = side == 0 ? 2.0 * t + 1.0 : 2.0 * t - 1.0;
  legendre_values(p, local, leg.data());
  const double s2 = std::sqrt(2.0);
  for (int m = 0; m < n; ++m) {
    double v = 0.0;
    for (int i = 0; i < n; ++i) v += mw(side * n + i, m) * s2 * leg[i];
    out[m] = v;
  }
}

static void eval_basis(const BasisSpec& spec, double x, double* out) {  // :226-254
  validate(spec);
  const double t = to_reference(spec, x);
  const int p = spec.degree;
  const int n1 = p + 1;
  if (spec.family == 0) {
    legendre_values(p, t, out);
    return;
  }
  const int dim = spec.dimension();
  std::fill(out, out + dim, 0.0);
  legendre_values(p, t, out);
  if (spec.resolution == 0) return;
  const Mat& mw = mother_wavelet(p);
  std::vector<double> psi(n1);
  for (int level = 1; level <= spec.resolution; ++level) {
    const std::int64_t n_int = std::int64_t(1) << (level - 1);
    const double h = 2.0 / static_cast<double>(n_int);
    std::int64_t i = static_cast<std::int64_t>(std::floor((t + 1.0) / h));
    i = std::min<std::int64_t>(n_int - 1, std::max<std::int64_t>(0, i));
    const double a = -1.0 + h * static_cast<double>(i);
    const double local = 2.0 * (t - a) / h - 1.0;
    mother_values(mw, p, local, psi.data());
    const double scale = std::pow(2.0, 0.5 * (level - 1));
    double* block = out + n1 * (std::int64_t(1) << (level - 1)) + i * n1;
    for (int m = 0; m < n1; ++m) block[m] = scale * psi[m];
  }
}

// ----------------------------------------------------------------- model ---
// proj/include/fstk/model.hpp:15-59, proj/src/model.cpp:15-94,176-227.
struct Fn {
  BasisSpec basis;
  std::vector<std::pair<std::uint32_t, double>> coeffs;  // sorted by index
};

struct Model {
  int d = 0;
  std::vector<std::int64_t> ranks;
  std::vector<double> core;  // mode-0 fastest (tensor.hpp:18-22)
  std::vector<std::vector<Fn>> modes;
  std::int64_t size() const {
    std::int64_t r = 1;
    for (auto x : ranks) r *= x;
    return r;
  }
};

static void validate_structure(const Model& m) {  // model.cpp:31-53
  require(m.d >= 1 && m.d <= 8, Shape, "model: bad order");
  for (int k = 0; k < m.d; ++k) {
    const auto& fns = m.modes[static_cast<std::size_t>(k)];
    require(static_cast<std::int64_t>(fns.size()) == m.ranks[k], Shape,
            "model: function count does not match rank");
    require(!fns.empty(), Shape, "model: empty mode");
    const double lo = fns.front().basis.lo, hi = fns.front().basis.hi;
    for (const auto& fn : fns) {
      validate(fn.basis);
      require(fn.basis.lo == lo && fn.basis.hi == hi, Shape,
              "model: inconsistent domains within a mode");
      const int n = fn.basis.dimension();
      for (const auto& ic : fn.coeffs)
        require(static_cast<int>(ic.first) < n, Shape,
                "model: coefficient index outside basis dimension");
    }
  }
}

static std::vector<double> mode_values(const Model& m, int mode, double x) {
  // model.cpp:71-94
  require(mode >= 0 && mode < m.d, Parameter, "mode out of range");
  const auto& fns = m.modes[static_cast<std::size_t>(mode)];
  std::vector<double> out(fns.size());
  std::vector<int> done(fns.size(), 0);
  std::vector<double> phi;
  for (std::size_t j = 0; j < fns.size(); ++j) {
    if (done[j]) continue;
    phi.resize(static_cast<std::size_t>(fns[j].basis.dimension()));
    eval_basis(fns[j].basis, x, phi.data());
    for (std::size_t l = j; l < fns.size(); ++l) {
      if (done[l] || !(fns[l].basis == fns[j].basis)) continue;
      double v = 0.0;
      for (const auto& ic : fns[l].coeffs) v += ic.second * phi[ic.first];
      out[l] = v;
      done[l] = 1;
    }
  }
  return out;
}

// model.cpp:176-191. Eigen's col-major GEMV is restated as column axpys.
static double contract_core(const Model& m,
                            const std::vector<std::vector<double>>& v,
                            std::vector<double>& a, std::vector<double>& b) {
  const int d = m.d;
  std::int64_t rows = m.size() / m.ranks[d - 1];
  a.assign(static_cast<std::size_t>(rows), 0.0);
  {
    const double* mat = m.core.data();
    const auto& vec = v[static_cast<std::size_t>(d - 1)];
    for (std::int64_t j = 0; j < m.ranks[d - 1]; ++j) {
      const double s = vec[static_cast<std::size_t>(j)];
      const double* col = mat + rows * j;
      for (std::int64_t i = 0; i < rows; ++i) a[i] += col[i] * s;
    }
  }
  for (int k = d - 2; k >= 0; --k) {
    rows /= m.ranks[k];
    b.assign(static_cast<std::size_t>(rows), 0.0);
    const auto& vec = v[static_cast<std::size_t>(k)];
    for (std::int64_t j = 0; j < m.ranks[k]; ++j) {
      const double s = vec[static_cast<std::size_t>(j)];
      const double* col = a.data() + rows * j;
      for (std::int64_t i = 0; i < rows; ++i) b[i] += col[i] * s;
    }
    std::swap(a, b);
  }
  return a[0];
}

static double evaluate(const Model& m, const double* y, int ny) {  // :195-206
  require(ny == m.d, Parameter, "evaluation point has wrong dimension");
  std::vector<std::vector<double>> v(static_cast<std::size_t>(m.d));
  for (int k = 0; k < m.d; ++k) v[k] = mode_values(m, k, y[k]);
  std::vector<double> a, b;
  return contract_core(m, v, a, b);
}

// model.cpp:208-227. points: Q x d column-major (Eigen default).
static void evaluate_batch(const Model& m, const double* pts, std::int64_t q,
                           int d, double* out) {
  require(d == m.d, Parameter, "points must have one column per mode");
  parallel_for(static_cast<std::size_t>(q), [&](std::size_t begin,
                                                std::size_t end) {
    std::vector<std::vector<double>> v(static_cast<std::size_t>(m.d));
    std::vector<double> a, b;
    for (std::size_t i = begin; i < end; ++i) {
      for (int k = 0; k < m.d; ++k)
        v[k] = mode_values(m, k, pts[static_cast<std::int64_t>(k) * q +
                                     static_cast<std::int64_t>(i)]);
      out[i] = contract_core(m, v, a, b);
    }
  });
}

// ---------------------------------------------------------- randomized LS ---
// proj/src/randls.cpp.
static constexpr std::uint64_t kValidationTag = 0x76616c69ull;  // :16
static constexpr std::uint64_t kSubsetTag = 0x73756273ull;      // :17
static constexpr std::uint64_t kSketchTag = 0x736b6574ull;      // :18

enum Transform { Dct = 0, Wht = 1, Fft = 2, None = 3 };  // randls.hpp:13 (+ None: extension)

// :21-41. Tables are Q x r_k column-major.
static std::vector<std::vector<double>> mode_value_tables(const Model& m,
                                                          const double* pts,
                                                          std::int64_t q) {
  std::vector<std::vector<double>> t(static_cast<std::size_t>(m.d));
  for (int k = 0; k < m.d; ++k)
    t[k].assign(static_cast<std::size_t>(q * m.ranks[k]), 0.0);
  parallel_for(static_cast<std::size_t>(q), [&](std::size_t begin,
                                                std::size_t end) {
    for (std::size_t i = begin; i < end; ++i)
      for (int k = 0; k < m.d; ++k) {
        const auto v = mode_values(m, k, pts[k * q + static_cast<std::int64_t>(i)]);
        for (std::int64_t j = 0; j < m.ranks[k]; ++j)
          t[k][static_cast<std::size_t>(j * q + static_cast<std::int64_t>(i))] = v[j];
      }
  });
  return t;
}

// :44-52.
static void design_column(const Model& m,
                          const std::vector<std::vector<double>>& tables,
                          std::int64_t q, std::int64_t ell, double* out) {
  std::int64_t rem = ell;
  const double* c0 = tables[0].data() + (rem % m.ranks[0]) * q;
  for (std::int64_t i = 0; i < q; ++i) out[i] = c0[i];
  rem /= m.ranks[0];
  for (int k = 1; k < m.d; ++k) {
    const double* ck = tables[k].data() + (rem % m.ranks[k]) * q;
    for (std::int64_t i = 0; i < q; ++i) out[i] *= ck[i];
    rem /= m.ranks[k];
  }
}

struct SketchPlan {  // :54-59
  std::vector<double> signs;
  std::vector<std::uint64_t> rows;
  std::uint64_t q_pad = 0;
  double scale = 1.0;
};

static SketchPlan make_plan(std::uint64_t q_w, std::uint64_t s,
                            std::uint64_t seed) {  // :61-75
  SketchPlan plan;
  plan.q_pad = next_pow2(q_w);
  require(s >= 1, Parameter, "sample rows must be positive");
  require(s <= plan.q_pad, Parameter, "sample rows exceed the padded row count");
  Rng rng(seed);
  plan.signs.resize(plan.q_pad);
  for (auto& x : plan.signs) x = rng.sign();
  plan.rows = rng.sample_without_replacement(plan.q_pad, s);
  plan.scale = std::sqrt(static_cast<double>(plan.q_pad) / static_cast<double>(s));
  return plan;
}

// Extension (not in the reference; the north_star's literal estimator):
// transform None samples S of the Q_w working rows uniformly without
// replacement from Rng(mix_seed(seed, kSketchTag)) and scales them by
// sqrt(Q_w / S); no mixing.
static SketchPlan make_plan_none(std::uint64_t q_w, std::uint64_t s, std::uint64_t seed) {
  SketchPlan plan;
  plan.q_pad = q_w;
  require(s >= 1, Parameter, "sample rows must be positive");
  require(s <= q_w, Parameter, "sample rows exceed the working subset");
  Rng rng(seed);
  plan.rows = rng.sample_without_replacement(q_w, s);
  plan.scale = std::sqrt(static_cast<double>(q_w) / static_cast<double>(s));
  return plan;
}

template <typename Getter>
static void sketch_column(const SketchPlan& plan, int transform,
                          std::uint64_t q_w, Getter&& getter,
                          std::vector<double>& scratch, std::vector<cd>& cscratch,
                          double* out_re, double* out_im) {  // :79-105
  if (transform == None) {
    for (std::size_t s = 0; s < plan.rows.size(); ++s)
      out_re[s] = plan.scale * getter(plan.rows[s]);
    return;
  }
  const std::size_t n = plan.q_pad;
  if (transform == Fft) {
    cscratch.assign(n, {0.0, 0.0});
    for (std::uint64_t i = 0; i < q_w; ++i) cscratch[i] = plan.signs[i] * getter(i);
    unitary_fft(cscratch.data(), n, false);
    for (std::size_t s = 0; s < plan.rows.size(); ++s) {
      out_re[s] = plan.scale * cscratch[plan.rows[s]].real();
      out_im[s] = plan.scale * cscratch[plan.rows[s]].imag();
    }
    return;
  }
  scratch.assign(n, 0.0);
  for (std::uint64_t i = 0; i < q_w; ++i) scratch[i] = plan.signs[i] * getter(i);
  if (transform == Dct)
    dct2_orthonormal(scratch.data(), n);
  else
    wht_orthonormal(scratch.data(), n);
  for (std::size_t s = 0; s < plan.rows.size(); ++s)
    out_re[s] = plan.scale * scratch[plan.rows[s]];
}

static std::uint64_t resolve_sample_rows(std::uint64_t sample_rows,
                                         std::int64_t r) {  // :125-130
  return sample_rows > 0
             ? sample_rows
             : static_cast<std::uint64_t>(std::ceil(2.5 * static_cast<double>(r)));
}

struct SketchCfg {  // randls.hpp:15-24
  std::uint64_t seed;
  std::uint64_t working_subset;
  std::uint64_t sample_rows;
  int transform;
  double validation_fraction;
};

// Result of prepare() (:246-311): index bookkeeping, working subset and tables.
struct Workspace {
  std::vector<double> train_points;  // q_w x d col-major
  std::vector<double> train_values;
  std::vector<std::uint64_t> val_index;  // rows of the dataset used for residuals
  std::uint64_t q_w = 0;
  bool held_out = true;
};

static void validate_cloud(const double* pts, const double* vals, std::int64_t q,
                           int d) {
  // ingest.cpp:19-49 (PointCloud::from_data computes the bbox, validate checks
  // finiteness; the bbox then covers the points by construction).
  require(d >= 1 && d <= 8, Shape, "point cloud dimension must be in [1, 8]");
  require(q >= 1, Data, "point cloud is empty");
  for (std::int64_t i = 0; i < q * d; ++i)
    require(std::isfinite(pts[i]), Data, "point coordinates must be finite");
  for (std::int64_t i = 0; i < q; ++i)
    require(std::isfinite(vals[i]), Data, "sample values must be finite");
}

static Workspace prepare(const Model& m, const double* pts, const double* vals,
                         std::int64_t q_count, int d, const SketchCfg& cfg) {
  validate_cloud(pts, vals, q_count, d);
  require(d == m.d, Shape, "dataset/model dimension mismatch");
  const auto q = static_cast<std::uint64_t>(q_count);
  std::uint64_t n_val = 0;
  if (cfg.validation_fraction > 0.0) {
    n_val = static_cast<std::uint64_t>(
        std::llround(cfg.validation_fraction * static_cast<double>(q)));
    n_val = std::min<std::uint64_t>(std::min(n_val, q - 1), 100000);
  }
  Workspace ws;
  std::vector<char> in_val(q, 0);
  if (n_val >= 1) {
    Rng rng(mix_seed(cfg.seed, kValidationTag));
    for (const auto i : rng.sample_without_replacement(q, n_val)) in_val[i] = 1;
  } else {
    ws.held_out = false;
  }
  std::vector<std::uint64_t> train, val;
  for (std::uint64_t i = 0; i < q; ++i) (in_val[i] ? val : train).push_back(i);
  if (!ws.held_out) val = train;
  const std::uint64_t q_w =
      cfg.working_subset == 0
          ? train.size()
          : std::min<std::uint64_t>(cfg.working_subset, train.size());
  require(q_w >= 1, Parameter, "no training points left");
  std::vector<std::uint64_t> subset;
  if (q_w == train.size()) {
    subset = train;
  } else {
    Rng rng(mix_seed(cfg.seed, kSubsetTag));
    for (const auto i : rng.sample_without_replacement(train.size(), q_w))
      subset.push_back(train[i]);
  }
  ws.q_w = subset.size();
  ws.train_points.resize(subset.size() * static_cast<std::size_t>(d));
  ws.train_values.resize(subset.size());
  for (std::size_t i = 0; i < subset.size(); ++i) {
    for (int k = 0; k < d; ++k)
      ws.train_points[static_cast<std::size_t>(k) * subset.size() + i] =
          pts[static_cast<std::int64_t>(k) * q_count +
              static_cast<std::int64_t>(subset[i])];
    ws.train_values[i] = vals[subset[i]];
  }
  ws.val_index = std::move(val);
  return ws;
}

}  // namespace oracle

// =============================================================== C API ====
// Flat model descriptor: functions are listed mode-major (all of mode 0, then
// mode 1, ...); coefficient arrays are concatenated in that order.
using namespace oracle;

namespace {

thread_local std::string g_last_error;

Model build_model(int d, const std::int64_t* ranks, const double* core,
                  const int* family, const int* degree, const int* resolution,
                  const double* lo, const double* hi, const std::uint32_t* nnz,
                  const std::uint32_t* idx, const double* coeffs) {
  Model m;
  m.d = d;
  m.ranks.assign(ranks, ranks + d);
  m.core.assign(core, core + m.size());
  m.modes.resize(static_cast<std::size_t>(d));
  std::size_t f = 0, c = 0;
  for (int k = 0; k < d; ++k)
    for (std::int64_t j = 0; j < ranks[k]; ++j, ++f) {
      Fn fn;
      fn.basis.family = family[f];
      fn.basis.degree = degree[f];
      fn.basis.resolution = resolution[f];
      fn.basis.lo = lo[f];
      fn.basis.hi = hi[f];
      for (std::uint32_t s = 0; s < nnz[f]; ++s, ++c)
        fn.coeffs.emplace_back(idx[c], coeffs[c]);
      m.modes[static_cast<std::size_t>(k)].push_back(std::move(fn));
    }
  validate_structure(m);
  return m;
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const Error& e) {
    g_last_error = e.msg;
    return e.kind + 1;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return Compute + 1;
  }
}

// ------------------------------------------- IDW interpolation (§8f-4) ---
// ingest.cpp:117-383 restated: uniform-binning spatial index over the grid
// box (build_index :140-190), fixed-size max-heap of (d2, id) pairs under
// lexicographic order (NeighborHeap :194-212, std::push_heap/pop_heap as the
// reference uses them, so the weight sums run in the reference's order),
// Chebyshev rings (for_ring :217-260) with the reference's stop rule, exact
// hits, inverse-distance weights and the report (:265-383).
struct IdwIndex {
  int d;
  std::vector<std::int64_t> nbins;
  std::vector<double> lo, width;
  std::vector<std::uint32_t> offsets, items;
  double min_width = 0.0, bin_diag = 0.0;
  std::int64_t bin_of(int k, double x) const {
    const auto b = static_cast<std::int64_t>(std::floor((x - lo[k]) / width[k]));
    return std::min<std::int64_t>(nbins[k] - 1, std::max<std::int64_t>(0, b));
  }
  std::int64_t flat(const std::vector<std::int64_t>& c) const {
    std::int64_t f = 0;
    for (int k = d - 1; k >= 0; --k) f = f * nbins[k] + c[k];
    return f;
  }
};

static IdwIndex idw_build_index(const double* pts, std::int64_t q, int d, const double* box_lo,
                                const double* box_hi, const std::int64_t* sizes, const double* glo,
                                const double* ghi) {
  IdwIndex ix;
  ix.d = d;
  ix.nbins.resize(d);
  ix.lo.resize(d);
  ix.width.resize(d);
  const double per_mode = std::pow(std::max(1.0, static_cast<double>(q) / 4.0), 1.0 / d);
  std::int64_t total = 1;
  for (int k = 0; k < d; ++k) {
    const std::int64_t cells = sizes[k] - 1;
    ix.nbins[k] = std::max<std::int64_t>(
        1, std::min<std::int64_t>(cells, static_cast<std::int64_t>(std::llround(per_mode))));
    total *= ix.nbins[k];
  }
  while (total > (std::int64_t(1) << 22)) {
    total = 1;
    for (int k = 0; k < d; ++k) {
      ix.nbins[k] = std::max<std::int64_t>(1, ix.nbins[k] / 2);
      total *= ix.nbins[k];
    }
  }
  double min_w = std::numeric_limits<double>::infinity();
  double diag2 = 0.0;
  for (int k = 0; k < d; ++k) {
    ix.lo[k] = std::min(glo[k], box_lo[k]);
    const double hi = std::max(ghi[k], box_hi[k]);
    ix.width[k] = (hi - ix.lo[k]) / static_cast<double>(ix.nbins[k]);
    if (ix.width[k] <= 0.0) ix.width[k] = 1.0;
    min_w = std::min(min_w, ix.width[k]);
    diag2 += ix.width[k] * ix.width[k];
  }
  ix.min_width = min_w;
  ix.bin_diag = std::sqrt(diag2);
  std::vector<std::uint32_t> bin_id(static_cast<std::size_t>(q));
  std::vector<std::uint32_t> counts(static_cast<std::size_t>(total) + 1, 0);
  std::vector<std::int64_t> c(d);
  for (std::int64_t i = 0; i < q; ++i) {
    for (int k = 0; k < d; ++k) c[k] = ix.bin_of(k, pts[i + k * q]);
    bin_id[i] = static_cast<std::uint32_t>(ix.flat(c));
    ++counts[bin_id[i] + 1];
  }
  for (std::size_t b = 1; b < counts.size(); ++b) counts[b] += counts[b - 1];
  ix.items.resize(static_cast<std::size_t>(q));
  std::vector<std::uint32_t> cursor(counts.begin(), counts.end() - 1);
  for (std::int64_t i = 0; i < q; ++i) ix.items[cursor[bin_id[i]]++] = static_cast<std::uint32_t>(i);
  ix.offsets = std::move(counts);
  return ix;
}

struct IdwHeap {
  std::vector<std::pair<double, std::uint32_t>> heap;
  std::size_t cap;
  explicit IdwHeap(std::size_t k) : cap(k) { heap.reserve(k); }
  bool full() const { return heap.size() >= cap; }
  double worst() const { return heap.front().first; }
  void push(double d2, std::uint32_t id) {
    const std::pair<double, std::uint32_t> p{d2, id};
    if (heap.size() < cap) {
      heap.push_back(p);
      std::push_heap(heap.begin(), heap.end());
    } else if (p < heap.front()) {
      std::pop_heap(heap.begin(), heap.end());
      heap.back() = p;
      std::push_heap(heap.begin(), heap.end());
    }
  }
};

template <typename Fn>
static void idw_for_ring(const IdwIndex& ix, const std::vector<std::int64_t>& center, std::int64_t rho,
                         Fn&& fn) {
  const int d = ix.d;
  std::vector<std::int64_t> c(d);
  if (rho == 0) {
    for (int k = 0; k < d; ++k) c[k] = center[k];
    fn(c);
    return;
  }
  std::vector<std::int64_t> lo(d), hi(d);
  for (int axis = 0; axis < d; ++axis) {
    for (int side = 0; side < 2; ++side) {
      const std::int64_t fixed = center[axis] + (side == 0 ? -rho : rho);
      if (fixed < 0 || fixed >= ix.nbins[axis]) continue;
      bool empty = false;
      for (int k = 0; k < d; ++k) {
        if (k == axis) {
          lo[k] = hi[k] = fixed;
          continue;
        }
        const std::int64_t r = k < axis ? rho - 1 : rho;
        lo[k] = std::max<std::int64_t>(0, center[k] - r);
        hi[k] = std::min(ix.nbins[k] - 1, center[k] + r);
        if (lo[k] > hi[k]) empty = true;
      }
      if (empty) continue;
      for (int k = 0; k < d; ++k) c[k] = lo[k];
      for (;;) {
        fn(c);
        int k = 0;
        while (k < d && (k == axis || ++c[k] > hi[k])) {
          if (k != axis) c[k] = lo[k];
          ++k;
        }
        if (k == d) break;
      }
    }
  }
}

// out: prod(sizes) values, mode-0 fastest.  report: box_covered,
// max_nearest_distance, extrapolated_fraction.  nbr (optional): per node the
// k retained ids sorted by (d2, id), padded with UINT32_MAX.
static void interpolate_to_grid(const double* pts, const double* vals, std::int64_t q, int d,
                                const double* box_lo_in, const double* box_hi_in,
                                const std::int64_t* sizes, const double* glo, const double* ghi,
                                int neighbors, double power, double* out, double* report,
                                std::uint32_t* nbr) {
  require(d >= 1 && d <= 8, Shape, "point cloud dimension must be in [1, 8]");
  require(q >= 1, Data, "point cloud is empty");
  std::vector<double> box_lo(d), box_hi(d);
  for (int k = 0; k < d; ++k) {
    double mn = pts[k * q], mx = pts[k * q];
    for (std::int64_t i = 0; i < q; ++i) {
      require(std::isfinite(pts[i + k * q]), Data, "point coordinates must be finite");
      mn = std::min(mn, pts[i + k * q]);
      mx = std::max(mx, pts[i + k * q]);
    }
    box_lo[k] = box_lo_in ? box_lo_in[k] : mn;
    box_hi[k] = box_hi_in ? box_hi_in[k] : mx;
    require(mn >= box_lo[k] && mx <= box_hi[k], Data, "bounding box does not cover the points");
  }
  for (std::int64_t i = 0; i < q; ++i) require(std::isfinite(vals[i]), Data, "point cloud values must be finite");
  for (int k = 0; k < d; ++k) {
    require(sizes[k] >= 2, Parameter, "grid sizes must be >= 2");
    require(glo[k] < ghi[k], Parameter, "grid intervals must be nondegenerate");
  }
  const int kn = neighbors > 0 ? neighbors : 2 * d + 2;
  require(power > 0.0, Parameter, "IDW power must be positive");
  const IdwIndex ix = idw_build_index(pts, q, d, box_lo.data(), box_hi.data(), sizes, glo, ghi);
  double cell_diag2 = 0.0;
  for (int k = 0; k < d; ++k) {
    const double h = (ghi[k] - glo[k]) / static_cast<double>(sizes[k] - 1);
    cell_diag2 += h * h;
  }
  const double hit_tol2 = 1e-24 * cell_diag2;
  bool covered = true;
  for (int k = 0; k < d; ++k)
    if (box_lo[k] < glo[k] || box_hi[k] > ghi[k]) covered = false;
  std::int64_t n_nodes = 1;
  for (int k = 0; k < d; ++k) n_nodes *= sizes[k];
  std::mutex mu;
  double max_nearest = 0.0;
  std::int64_t n_extra = 0;
  parallel_for(static_cast<std::size_t>(n_nodes), [&](std::size_t begin, std::size_t end) {
    std::vector<std::int64_t> midx(d), center(d);
    std::vector<double> y(d);
    double lmax = 0.0;
    std::int64_t lextra = 0;
    for (std::size_t node = begin; node < end; ++node) {
      std::int64_t rem = static_cast<std::int64_t>(node);
      for (int k = 0; k < d; ++k) {
        midx[k] = rem % sizes[k];
        rem /= sizes[k];
        y[k] = glo[k] + (ghi[k] - glo[k]) * static_cast<double>(midx[k]) /
                            static_cast<double>(sizes[k] - 1);
        center[k] = ix.bin_of(k, y[k]);
      }
      IdwHeap heap(static_cast<std::size_t>(kn));
      std::int64_t max_rho = 0;
      for (int k = 0; k < d; ++k)
        max_rho = std::max({max_rho, center[k], ix.nbins[k] - 1 - center[k]});
      for (std::int64_t rho = 0;; ++rho) {
        idw_for_ring(ix, center, rho, [&](const std::vector<std::int64_t>& c) {
          const std::int64_t b = ix.flat(c);
          for (std::uint32_t ii = ix.offsets[b]; ii < ix.offsets[b + 1]; ++ii) {
            const std::uint32_t id = ix.items[ii];
            double d2 = 0.0;
            for (int k = 0; k < d; ++k) {
              const double diff = pts[id + k * q] - y[k];
              d2 += diff * diff;
            }
            heap.push(d2, id);
          }
        });
        const double safe = static_cast<double>(rho) * ix.min_width;
        if (heap.full() && heap.worst() <= safe * safe) break;
        if (rho >= max_rho) break;
      }
      auto best = heap.heap.front();
      for (const auto& cand : heap.heap) best = std::min(best, cand);
      double value;
      if (best.first < hit_tol2) {
        value = vals[best.second];
      } else {
        double wsum = 0.0, vsum = 0.0;
        for (const auto& e : heap.heap) {
          const double w = power == 2.0 ? 1.0 / e.first : std::pow(e.first, -0.5 * power);
          wsum += w;
          vsum += w * vals[e.second];
        }
        value = vsum / wsum;
      }
      out[node] = value;
      if (nbr) {
        auto sorted = heap.heap;
        std::sort(sorted.begin(), sorted.end());
        for (int j = 0; j < kn; ++j)
          nbr[node * kn + j] = j < static_cast<int>(sorted.size()) ? sorted[j].second : 0xFFFFFFFFu;
      }
      const double nearest = std::sqrt(best.first);
      lmax = std::max(lmax, nearest);
      if (nearest > ix.bin_diag) ++lextra;
    }
    std::lock_guard<std::mutex> lk(mu);
    max_nearest = std::max(max_nearest, lmax);
    n_extra += lextra;
  });
  report[0] = covered ? 1.0 : 0.0;
  report[1] = max_nearest;
  report[2] = static_cast<double>(n_extra) / static_cast<double>(n_nodes);
}

}  // namespace

#define MODEL_ARGS                                                            \
  int d, const std::int64_t *ranks, const double *core, const int *family,    \
      const int *degree, const int *resolution, const double *lo,            \
      const double *hi, const std::uint32_t *nnz, const std::uint32_t *idx,  \
      const double *coeffs
#define MODEL_PASS d, ranks, core, family, degree, resolution, lo, hi, nnz, idx, coeffs

extern "C" {

const char* oracle_last_error() { return g_last_error.c_str(); }
void oracle_set_max_threads(int n) { g_max_threads.store(n > 0 ? n : 0); }
int oracle_max_threads() { return max_threads(); }

// --- RNG / transforms -------------------------------------------------------
std::uint64_t oracle_mix_seed(std::uint64_t seed, std::uint64_t tag) {
  return mix_seed(seed, tag);
}
std::uint64_t oracle_next_pow2(std::uint64_t n) { return next_pow2(n); }
int oracle_sample_without_replacement(std::uint64_t seed, std::uint64_t n,
                                      std::uint64_t k, std::uint64_t* out) {
  return guarded([&] {
    Rng rng(seed);
    const auto v = rng.sample_without_replacement(n, k);
    std::copy(v.begin(), v.end(), out);
  });
}
int oracle_make_plan(std::uint64_t q_w, std::uint64_t s, std::uint64_t seed,
                     double* signs, std::uint64_t* rows, double* scale) {
  return guarded([&] {
    const auto p = make_plan(q_w, s, seed);
    std::copy(p.signs.begin(), p.signs.end(), signs);
    std::copy(p.rows.begin(), p.rows.end(), rows);
    *scale = p.scale;
  });
}
int oracle_fft_pow2(double* x_interleaved, std::uint64_t n, int inverse) {
  return guarded([&] { fft_pow2(reinterpret_cast<cd*>(x_interleaved), n, inverse != 0); });
}
int oracle_unitary_fft(double* x_interleaved, std::uint64_t n, int inverse) {
  return guarded([&] { unitary_fft(reinterpret_cast<cd*>(x_interleaved), n, inverse != 0); });
}
int oracle_dct2(double* x, std::uint64_t n) {
  return guarded([&] { dct2_orthonormal(x, n); });
}
int oracle_interpolate_to_grid(const double* pts, const double* vals, std::int64_t q, int d,
                               const double* box_lo, const double* box_hi, const std::int64_t* sizes,
                               const double* glo, const double* ghi, int neighbors, double power,
                               double* out, double* report, std::uint32_t* nbr) {
  return guarded([&] {
    interpolate_to_grid(pts, vals, q, d, box_lo, box_hi, sizes, glo, ghi, neighbors, power, out,
                        report, nbr);
  });
}
int oracle_wht(double* x, std::uint64_t n) {
  return guarded([&] { wht_orthonormal(x, n); });
}

// --- basis ------------------------------------------------------------------
int oracle_legendre_values(int p, double t, double* out) {
  return guarded([&] { legendre_values(p, t, out); });
}
int oracle_gauss_legendre(int n, double* nodes, double* weights) {
  return guarded([&] {
    std::vector<double> a, b;
    gauss_legendre(n, a, b);
    std::copy(a.begin(), a.end(), nodes);
    std::copy(b.begin(), b.end(), weights);
  });
}
int oracle_mother_coords(int p, double* out) {  // 2(p+1) x (p+1) column-major
  return guarded([&] {
    const Mat& m = mother_wavelet(p);
    std::copy(m.a.begin(), m.a.end(), out);
  });
}
int oracle_eval_basis(int family, int degree, int resolution, double lo,
                      double hi, double x, double* out) {
  return guarded([&] {
    BasisSpec s{family, degree, resolution, lo, hi};
    eval_basis(s, x, out);
  });
}

// --- model ------------------------------------------------------------------
int oracle_validate_model(MODEL_ARGS) {
  return guarded([&] { (void)build_model(MODEL_PASS); });
}
int oracle_mode_values(MODEL_ARGS, int mode, double x, double* out) {
  return guarded([&] {
    const Model m = build_model(MODEL_PASS);
    const auto v = mode_values(m, mode, x);
    std::copy(v.begin(), v.end(), out);
  });
}
int oracle_evaluate(MODEL_ARGS, const double* y, int ny, double* out) {
  return guarded([&] {
    const Model m = build_model(MODEL_PASS);
    *out = evaluate(m, y, ny);
  });
}
int oracle_evaluate_batch(MODEL_ARGS, const double* pts, std::int64_t q,
                          int pd, double* out) {
  return guarded([&] {
    const Model m = build_model(MODEL_PASS);
    evaluate_batch(m, pts, q, pd, out);
  });
}
// randls.cpp:134-145 (Q x R column-major).
int oracle_build_design_rows(MODEL_ARGS, const double* pts, std::int64_t q,
                             int pd, double* w) {
  return guarded([&] {
    const Model m = build_model(MODEL_PASS);
    require(pd == m.d, Parameter, "points must have one column per mode");
    const auto tables = mode_value_tables(m, pts, q);
    for (std::int64_t ell = 0; ell < m.size(); ++ell)
      design_column(m, tables, q, ell, w + ell * q);
  });
}

// randls.cpp:147-184, public sketch(): seeds make_plan with cfg.seed directly.
// a: rows_out x r col-major with rows_out = S (2S for FFT); b: rows_out.
int oracle_sketch(const double* w, const double* u, std::int64_t q,
                  std::int64_t r, std::uint64_t seed, std::uint64_t sample_rows,
                  int transform, double* a, double* b, std::uint64_t* padded) {
  return guarded([&] {
    require(q >= 1, Parameter, "empty system");
    const std::uint64_t s = resolve_sample_rows(sample_rows, r);
    const SketchPlan plan = make_plan(static_cast<std::uint64_t>(q), s, seed);
    const bool fft = transform == Fft;
    const std::int64_t s_rows = static_cast<std::int64_t>(plan.rows.size());
    const std::int64_t lda = fft ? 2 * s_rows : s_rows;
    *padded = plan.q_pad;
    parallel_for(static_cast<std::size_t>(r) + 1, [&](std::size_t begin,
                                                      std::size_t end) {
      std::vector<double> scratch;
      std::vector<cd> cscratch;
      for (std::size_t c = begin; c < end; ++c) {
        if (c < static_cast<std::size_t>(r)) {
          const double* col = w + static_cast<std::int64_t>(c) * q;
          double* out = a + static_cast<std::int64_t>(c) * lda;
          sketch_column(plan, transform, static_cast<std::uint64_t>(q),
                        [&](std::uint64_t i) { return col[i]; }, scratch,
                        cscratch, out, fft ? out + s_rows : nullptr);
        } else {
          sketch_column(plan, transform, static_cast<std::uint64_t>(q),
                        [&](std::uint64_t i) { return u[i]; }, scratch,
                        cscratch, b, fft ? b + s_rows : nullptr);
        }
      }
    });
  });
}

// randls.cpp:186-225 (diagnostics): mixed = transform(D W), all padded rows.
int oracle_mixed_matrix(const double* w, std::int64_t q, std::int64_t r,
                        std::uint64_t seed, int transform, double* out) {
  return guarded([&] {
    require(q >= 1, Parameter, "empty matrix");
    const std::uint64_t q_pad = next_pow2(static_cast<std::uint64_t>(q));
    Rng rng(seed);
    std::vector<double> signs(q_pad);
    for (auto& x : signs) x = rng.sign();
    const bool fft = transform == Fft;
    const std::int64_t ld = fft ? 2 * static_cast<std::int64_t>(q_pad)
                                : static_cast<std::int64_t>(q_pad);
    parallel_for(static_cast<std::size_t>(r), [&](std::size_t begin,
                                                  std::size_t end) {
      std::vector<double> scratch;
      std::vector<cd> cscratch;
      for (std::size_t c = begin; c < end; ++c) {
        const double* col = w + static_cast<std::int64_t>(c) * q;
        double* o = out + static_cast<std::int64_t>(c) * ld;
        if (fft) {
          cscratch.assign(q_pad, {0.0, 0.0});
          for (std::int64_t i = 0; i < q; ++i) cscratch[i] = signs[i] * col[i];
          unitary_fft(cscratch.data(), q_pad, false);
          for (std::uint64_t i = 0; i < q_pad; ++i) {
            o[i] = cscratch[i].real();
            o[q_pad + i] = cscratch[i].imag();
          }
        } else {
          scratch.assign(q_pad, 0.0);
          for (std::int64_t i = 0; i < q; ++i) scratch[i] = signs[i] * col[i];
          if (transform == Dct)
            dct2_orthonormal(scratch.data(), q_pad);
          else
            wht_orthonormal(scratch.data(), q_pad);
          std::copy(scratch.begin(), scratch.end(), o);
        }
      }
    });
  });
}

// --- reestimate_core (randls.cpp:360-383), split in two calls so the caller
// can allocate the sketched system; the QR solve (Eigen ColPivHouseholderQR,
// :112-123) is done by the Python side with LAPACK dgeqp3 (oracle/oracle.py).
struct OracleRefitSizes {
  std::uint64_t sample_rows;   // S
  std::uint64_t working_rows;  // Q_w
  std::uint64_t padded_rows;   // q_pad
  std::uint64_t n_val;         // validation rows (== train size if !held_out)
  std::int64_t system_rows;    // S or 2S
  int held_out;
};

int oracle_refit_sizes(MODEL_ARGS, std::int64_t q, std::uint64_t seed,
                       std::uint64_t working_subset, std::uint64_t sample_rows,
                       int transform, double validation_fraction,
                       OracleRefitSizes* out) {
  return guarded([&] {
    const Model m = build_model(MODEL_PASS);
    const std::int64_t r_total = m.size();
    const std::uint64_t s = resolve_sample_rows(sample_rows, r_total);
    require(s > static_cast<std::uint64_t>(r_total), Parameter,
            "sample rows must exceed the core size");
    require(static_cast<std::uint64_t>(q) >= s, Parameter,
            "dataset smaller than the requested sketch");
    std::uint64_t n_val = 0;
    const auto uq = static_cast<std::uint64_t>(q);
    if (validation_fraction > 0.0) {
      n_val = static_cast<std::uint64_t>(
          std::llround(validation_fraction * static_cast<double>(uq)));
      n_val = std::min<std::uint64_t>(std::min(n_val, uq - 1), 100000);
    }
    const bool held = n_val >= 1;
    const std::uint64_t train = uq - (held ? n_val : 0);
    const std::uint64_t q_w =
        working_subset == 0 ? train : std::min<std::uint64_t>(working_subset, train);
    out->sample_rows = s;
    out->working_rows = q_w;
    out->padded_rows = transform == None ? q_w : next_pow2(q_w);
    out->n_val = held ? n_val : train;
    out->system_rows = transform == Fft ? 2 * static_cast<std::int64_t>(s)
                                        : static_cast<std::int64_t>(s);
    out->held_out = held ? 1 : 0;
  });
}

// Fills A (system_rows x R col-major), b, the sampled padded rows, and the
// validation row indices (into the dataset).
int oracle_refit_system(MODEL_ARGS, const double* pts, const double* vals,
                        std::int64_t q, int pd, std::uint64_t seed,
                        std::uint64_t working_subset, std::uint64_t sample_rows,
                        int transform, double validation_fraction, double* a,
                        double* b, std::uint64_t* rows_out,
                        std::uint64_t* val_index_out) {
  return guarded([&] {
    const Model m = build_model(MODEL_PASS);
    const std::int64_t r_total = m.size();
    const std::uint64_t s = resolve_sample_rows(sample_rows, r_total);
    require(s > static_cast<std::uint64_t>(r_total), Parameter,
            "sample rows must exceed the core size");
    require(static_cast<std::uint64_t>(q) >= s, Parameter,
            "dataset smaller than the requested sketch");
    SketchCfg cfg{seed, working_subset, sample_rows, transform,
                  validation_fraction};
    const Workspace ws = prepare(m, pts, vals, q, pd, cfg);
    const auto tables = mode_value_tables(m, ws.train_points.data(),
                                          static_cast<std::int64_t>(ws.q_w));
    // solve_sketched (:315-348)
    const SketchPlan plan = transform == None
                                ? make_plan_none(ws.q_w, s, mix_seed(seed, kSketchTag))
                                : make_plan(ws.q_w, s, mix_seed(seed, kSketchTag));
    const bool fft = transform == Fft;
    const std::int64_t s_rows = static_cast<std::int64_t>(plan.rows.size());
    const std::int64_t lda = fft ? 2 * s_rows : s_rows;
    const std::int64_t qw = static_cast<std::int64_t>(ws.q_w);
    parallel_for(static_cast<std::size_t>(r_total) + 1,
                 [&](std::size_t begin, std::size_t end) {
                   std::vector<double> scratch;
                   std::vector<cd> cscratch;
                   std::vector<double> col(static_cast<std::size_t>(qw));
                   for (std::size_t c = begin; c < end; ++c) {
                     if (c < static_cast<std::size_t>(r_total)) {
                       design_column(m, tables, qw, static_cast<std::int64_t>(c),
                                     col.data());
                       double* out = a + static_cast<std::int64_t>(c) * lda;
                       sketch_column(plan, transform, ws.q_w,
                                     [&](std::uint64_t i) { return col[i]; },
                                     scratch, cscratch, out,
                                     fft ? out + s_rows : nullptr);
                     } else {
                       sketch_column(plan, transform, ws.q_w,
                                     [&](std::uint64_t i) {
                                       return ws.train_values[i];
                                     },
                                     scratch, cscratch, b,
                                     fft ? b + s_rows : nullptr);
                     }
                   }
                 });
    std::copy(plan.rows.begin(), plan.rows.end(), rows_out);
    std::copy(ws.val_index.begin(), ws.val_index.end(), val_index_out);
  });
}

// Sketched columns at arbitrary indices (column r_total = the right-hand
// side b), plus the plan's sampled rows: full-size parity checks of single
// columns without forming A (randls.cpp:313-348, one column at a time).
int oracle_refit_column_set(MODEL_ARGS, const double* pts, const double* vals,
                            std::int64_t q, int pd, std::uint64_t seed,
                            std::uint64_t working_subset, std::uint64_t sample_rows,
                            int transform, double validation_fraction,
                            const std::int64_t* cols, std::int64_t ncols, double* a,
                            std::uint64_t* rows_out) {
  return guarded([&] {
    const Model m = build_model(MODEL_PASS);
    const std::int64_t r_total = m.size();
    const std::uint64_t s = resolve_sample_rows(sample_rows, r_total);
    SketchCfg cfg{seed, working_subset, sample_rows, transform,
                  validation_fraction};
    const Workspace ws = prepare(m, pts, vals, q, pd, cfg);
    const auto tables = mode_value_tables(m, ws.train_points.data(),
                                          static_cast<std::int64_t>(ws.q_w));
    const SketchPlan plan = make_plan(ws.q_w, s, mix_seed(seed, kSketchTag));
    const bool fft = transform == Fft;
    const std::int64_t s_rows = static_cast<std::int64_t>(plan.rows.size());
    const std::int64_t lda = fft ? 2 * s_rows : s_rows;
    const std::int64_t qw = static_cast<std::int64_t>(ws.q_w);
    parallel_for(static_cast<std::size_t>(ncols),
                 [&](std::size_t begin, std::size_t end) {
                   std::vector<double> scratch;
                   std::vector<cd> cscratch;
                   std::vector<double> col(static_cast<std::size_t>(qw));
                   for (std::size_t c = begin; c < end; ++c) {
                     const std::int64_t ell = cols[c];
                     require(ell >= 0 && ell <= r_total, Parameter, "column out of range");
                     double* out = a + static_cast<std::int64_t>(c) * lda;
                     if (ell < r_total) {
                       design_column(m, tables, qw, ell, col.data());
                       sketch_column(plan, transform, ws.q_w,
                                     [&](std::uint64_t i) { return col[i]; },
                                     scratch, cscratch, out, fft ? out + s_rows : nullptr);
                     } else {
                       sketch_column(plan, transform, ws.q_w,
                                     [&](std::uint64_t i) { return ws.train_values[i]; },
                                     scratch, cscratch, out, fft ? out + s_rows : nullptr);
                     }
                   }
                 });
    if (rows_out) std::copy(plan.rows.begin(), plan.rows.end(), rows_out);
  });
}

// Only the sketched columns in [col_begin, col_end) (and b when include_rhs):
// used by the CPU baseline to time a bounded sample of the transform stage.
int oracle_refit_columns(MODEL_ARGS, const double* pts, const double* vals,
                         std::int64_t q, int pd, std::uint64_t seed,
                         std::uint64_t working_subset, std::uint64_t sample_rows,
                         int transform, double validation_fraction,
                         std::int64_t col_begin, std::int64_t col_end, double* a) {
  return guarded([&] {
    const Model m = build_model(MODEL_PASS);
    const std::int64_t r_total = m.size();
    const std::uint64_t s = resolve_sample_rows(sample_rows, r_total);
    SketchCfg cfg{seed, working_subset, sample_rows, transform,
                  validation_fraction};
    const Workspace ws = prepare(m, pts, vals, q, pd, cfg);
    const auto tables = mode_value_tables(m, ws.train_points.data(),
                                          static_cast<std::int64_t>(ws.q_w));
    const SketchPlan plan = make_plan(ws.q_w, s, mix_seed(seed, kSketchTag));
    const bool fft = transform == Fft;
    const std::int64_t s_rows = static_cast<std::int64_t>(plan.rows.size());
    const std::int64_t lda = fft ? 2 * s_rows : s_rows;
    const std::int64_t qw = static_cast<std::int64_t>(ws.q_w);
    parallel_for(static_cast<std::size_t>(col_end - col_begin),
                 [&](std::size_t begin, std::size_t end) {
                   std::vector<double> scratch;
                   std::vector<cd> cscratch;
                   std::vector<double> col(static_cast<std::size_t>(qw));
                   for (std::size_t c = begin; c < end; ++c) {
                     const std::int64_t ell = col_begin + static_cast<std::int64_t>(c);
                     design_column(m, tables, qw, ell % r_total, col.data());
                     double* out = a + static_cast<std::int64_t>(c) * lda;
                     sketch_column(plan, transform, ws.q_w,
                                   [&](std::uint64_t i) { return col[i]; },
                                   scratch, cscratch, out,
                                   fft ? out + s_rows : nullptr);
                   }
                 });
  });
}

}  // extern "C"
