// fstk B200 library — multiwavelet bases.
//
// Host: Gauss-Legendre nodes and the Alpert-style mother multiwavelets of
// degree p (proj/src/basis.cpp:63-102, 116-189): the orthonormal complement of
// the degree-p polynomials in the split basis, canonically rotated so that
// wavelet m annihilates the moments x^{p+1} .. x^{p+m}, then sign-normalised.
// The result is unique up to rounding (independent of the QR implementation),
// so a plain Householder QR stands in for Eigen::HouseholderQR.
//
// Device: mode_general_kernel evaluates modes whose functions use wavelet
// (or several distinct) bases.  Per point it forms, for each distinct basis,
// the level-0 Legendre block and, per level, the active dyadic interval and
// its (p+1) scaled mother values (basis.cpp:226-253), then runs each
// function's sparse dot with an O(1) index -> (level, interval, m) lookup
// (inactive indices contribute c * 0, as the reference's dense phi does).
#include <cmath>
#include <map>
#include <mutex>
#include <vector>

#include "fstk_internal.h"

namespace fstk_gpu {

// ---------------------------------------------------------------- host ---
static void gauss_legendre(int n, std::vector<double>& nodes, std::vector<double>& weights) {
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

static void legendre_host(int p, double t, double* out) {  // basis.cpp:49-61
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

struct HMat {
  int r = 0, c = 0;
  std::vector<double> a;  // column-major
  HMat(int rr, int cc) : r(rr), c(cc), a(static_cast<size_t>(rr) * cc, 0.0) {}
  double& operator()(int i, int j) { return a[static_cast<size_t>(j) * r + i]; }
  double operator()(int i, int j) const { return a[static_cast<size_t>(j) * r + i]; }
};

// Full orthogonal factor of a Householder QR of A (m x n, m >= n).
static HMat householder_q(HMat A) {
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
  HMat Q(m, m);
  for (int i = 0; i < m; ++i) Q(i, i) = 1.0;
  for (int k = static_cast<int>(vs.size()) - 1; k >= 0; --k) {
    if (taus[k] == 0.0) continue;
    const auto& v = vs[k];
    for (int j = 0; j < m; ++j) {
      double d = 0.0;
      for (int i = k; i < m; ++i) d += v[i] * Q(i, j);
      d *= taus[k];
      for (int i = k; i < m; ++i) Q(i, j) -= d * v[i];
    }
  }
  return Q;
}

static HMat build_mother(int p) {
  const int n = p + 1;
  std::vector<double> qx, qw;
  gauss_legendre(2 * p + 4, qx, qw);
  const int nq = static_cast<int>(qx.size());
  HMat q(2 * n, n);
  std::vector<double> lg(n), lh(n);
  for (int side = 0; side < 2; ++side)
    for (int a = 0; a < nq; ++a) {
      const double t = qx[a];
      const double x = side == 0 ? 0.5 * (t - 1.0) : 0.5 * (t + 1.0);
      legendre_host(p, x, lg.data());
      legendre_host(p, t, lh.data());
      const double w = qw[a] * std::sqrt(2.0) / 4.0;
      for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) q(side * n + i, j) += w * lh[i] * lg[j];
    }
  const HMat full = householder_q(q);
  HMat comp(2 * n, n);
  for (int i = 0; i < 2 * n; ++i)
    for (int j = 0; j < n; ++j) comp(i, j) = full(i, n + j);
  HMat moments(n, n);
  for (int side = 0; side < 2; ++side)
    for (int a = 0; a < nq; ++a) {
      const double t = qx[a];
      const double x = side == 0 ? 0.5 * (t - 1.0) : 0.5 * (t + 1.0);
      legendre_host(p, t, lh.data());
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
  HMat mt(n, n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) mt(i, j) = moments(j, i);
  const HMat rot = householder_q(mt);
  HMat coords(2 * n, n);
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

// Device copies of the mother coordinates (2(p+1) x (p+1), column-major),
// pre-multiplied by sqrt(2) exactly as mother_values forms coords * s2
// (basis.cpp:207-210), cached per (device, p).
static std::mutex g_mw_mu;
static std::map<std::pair<int, int>, std::shared_ptr<DevBuf<double>>> g_mw;

std::shared_ptr<DevBuf<double>> mother_coords_device(int device, int p) {
  std::lock_guard<std::mutex> lk(g_mw_mu);
  auto key = std::make_pair(device, p);
  auto it = g_mw.find(key);
  if (it != g_mw.end()) return it->second;
  const HMat c = build_mother(p);
  const double s2 = std::sqrt(2.0);
  std::vector<double> h(c.a.size());
  for (size_t i = 0; i < h.size(); ++i) h[i] = c.a[i] * s2;
  auto buf = std::make_shared<DevBuf<double>>(h.size());
  FSTK_CUDA(cudaMemcpy(buf->p, h.data(), h.size() * 8, cudaMemcpyHostToDevice));
  g_mw[key] = buf;
  return buf;
}

// --------------------------------------------------------------- device ---
// Level scale 2^{(l-1)/2} as std::pow computes it (basis.cpp:250), l = 1..20,
// and the Legendre recurrence constants (as in fstk_eval.cu's c_leg).
struct WaveConst {
  double scale[24];
  double a[kMaxDegree + 1], b[kMaxDegree + 1], c[kMaxDegree + 1], rc[kMaxDegree + 1];
  double norm[kMaxDegree + 2];
};
__constant__ WaveConst c_w;
static std::once_flag g_wconst_once[64];

void upload_wavelet_constants(int device) {
  std::call_once(g_wconst_once[device & 63], [&] {
    WaveConst h;
    for (int l = 0; l < 24; ++l) h.scale[l] = l >= 1 ? std::pow(2.0, 0.5 * (l - 1)) : 1.0;
    for (int n = 0; n <= kMaxDegree; ++n) {
      h.a[n] = static_cast<double>(2 * n + 1);
      h.b[n] = static_cast<double>(n);
      h.c[n] = static_cast<double>(n + 1);
      h.rc[n] = 1.0 / static_cast<double>(n + 1);
    }
    for (int n = 0; n <= kMaxDegree + 1; ++n) h.norm[n] = std::sqrt(2.0 * n + 1.0);
    h.norm[1] = std::sqrt(3.0);
    FSTK_CUDA(cudaMemcpyToSymbol(c_w, &h, sizeof(h)));
  });
}

// Legendre values 0..p at t into v[0], v[stride], ... (basis.cpp:49-61, exact ops).
__device__ __forceinline__ void legendre_dev(int p, double t, double* v, int stride) {
  v[0] = 1.0;
  if (p >= 1) v[stride] = xmul(c_w.norm[1], t);
  double pm1 = 1.0, pm0 = t;
  for (int q = 1; q < p; ++q) {
    const double num = xsub(xmul(xmul(c_w.a[q], t), pm0), xmul(c_w.b[q], pm1));
    const double pn1 = xdiv_small(num, c_w.c[q], c_w.rc[q]);
    pm1 = pm0;
    pm0 = pn1;
    v[(q + 1) * stride] = xmul(c_w.norm[q + 1], pn1);
  }
}

template <bool EXACT>
__global__ void __launch_bounds__(64) mode_general_kernel(
    GenModeDev G, const double* __restrict__ xs, int64_t n, int64_t n_out,
    const int64_t* __restrict__ row_src, double* __restrict__ tk, int64_t ldt,
    unsigned long long* err_row) {
  extern __shared__ double V[];  // G.vtot x blockDim, column per thread
  const int tid = threadIdx.x, nt = blockDim.x;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * nt + tid;
  if (i >= n_out) return;
  int64_t src = i;
  bool valid = i < n;
  if (row_src) {
    src = i < n ? row_src[i] : -1;
    valid = src >= 0;
  }
  const ModeDev& md = G.md;
  if (!valid) {
    for (int j = 0; j < md.r; ++j) tk[j * ldt + i] = 0.0;
    return;
  }
  const double x = xs[src];
  double t;
  if (!(x >= md.lo - md.slack && x <= md.hi + md.slack)) {
    atomicMin(err_row, static_cast<unsigned long long>(i));
    t = 0.0;
  } else {
    const double cl = fmin(md.hi, fmax(md.lo, x));
    t = xadd(-1.0, __ddiv_rn(xmul(2.0, xsub(cl, md.lo)), md.span));
  }
  double* Vt = V + tid;
  // Per distinct basis: [L0 (p+1)] [tmp (p+1)] then per level [interval, (p+1) values].
  for (int sidx = 0; sidx < G.nspec; ++sidx) {
    const SpecDev& sp = G.sp[sidx];
    const int p = sp.p, n1 = p + 1;
    double* base = Vt + sp.voff * nt;
    legendre_dev(p, t, base, nt);
    if (sp.family == 0) continue;
    double* tmp = base + n1 * nt;
    for (int level = 1; level <= sp.s; ++level) {
      const int64_t n_int = int64_t(1) << (level - 1);
      const double h = 2.0 / static_cast<double>(n_int);
      int64_t iv = static_cast<int64_t>(floor(__ddiv_rn(xadd(t, 1.0), h)));
      if (iv < 0) iv = 0;
      if (iv > n_int - 1) iv = n_int - 1;
      const double a0 = xadd(-1.0, xmul(h, static_cast<double>(iv)));
      const double local = xsub(__ddiv_rn(xmul(2.0, xsub(t, a0)), h), 1.0);
      // mother_values (basis.cpp:201-213)
      const int side = local < 0.0 ? 0 : 1;
      const double l2 = side == 0 ? xadd(xmul(2.0, local), 1.0) : xsub(xmul(2.0, local), 1.0);
      legendre_dev(p, l2, tmp, nt);
      double* blk = base + (2 * n1 + (level - 1) * (n1 + 1)) * nt;
      blk[0] = static_cast<double>(iv);
      const double scale = c_w.scale[level];
      for (int m = 0; m < n1; ++m) {
        double v = 0.0;
        const double* cm = sp.coords + m * 2 * n1 + side * n1;  // (coords * sqrt2) column m
        for (int q = 0; q < n1; ++q) v = xadd(v, xmul(cm[q], tmp[q * nt]));
        blk[(m + 1) * nt] = xmul(scale, v);
      }
    }
  }
  // Sparse dots (model.cpp:86-88) with the basis value looked up by index.
  for (int j = 0; j < md.r; ++j) {
    const SpecDev& sp = G.sp[G.fn_spec[j]];
    const int n1 = sp.p + 1;
    const double* base = Vt + sp.voff * nt;
    double v = 0.0;
    const int e = md.rowptr[j + 1];
    for (int s2 = md.rowptr[j]; s2 < e; ++s2) {
      const uint32_t idx = md.idx[s2];
      double bval;
      if (sp.family == 0 || idx < static_cast<uint32_t>(n1)) {
        bval = base[idx * nt];
      } else {
        const uint32_t blockno = idx / n1;                 // >= 1
        const int level = 32 - __clz(blockno);             // floor(log2(blockno)) + 1
        const uint32_t off = idx - (static_cast<uint32_t>(n1) << (level - 1));
        const uint32_t iv = off / n1, m = off % n1;
        const double* blk = base + (2 * n1 + (level - 1) * (n1 + 1)) * nt;
        bval = (static_cast<double>(iv) == blk[0]) ? blk[(m + 1) * nt] : 0.0;
      }
      const double c = md.coef[s2];
      v = EXACT ? xadd(v, xmul(c, bval)) : fma(c, bval, v);
    }
    tk[j * ldt + i] = v;
  }
}

void launch_mode_general(const GenModeDev& G, const double* xs, int64_t n,
                         int64_t n_out, const int64_t* row_src, double* tk, int64_t ldt, bool exact,
                         unsigned long long* err_row, cudaStream_t s, int device) {
  static std::once_flag once[64];
  std::call_once(once[device & 63], [&] {
    FSTK_CUDA(cudaFuncSetAttribute(mode_general_kernel<true>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    FSTK_CUDA(cudaFuncSetAttribute(mode_general_kernel<false>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  });
  const int threads = 64;
  const size_t sm = static_cast<size_t>(G.vtot) * threads * sizeof(double);
  const unsigned blocks = static_cast<unsigned>(ceil_div(n_out, threads));
  if (exact)
    mode_general_kernel<true><<<blocks, threads, sm, s>>>(G, xs, n, n_out, row_src, tk, ldt, err_row);
  else
    mode_general_kernel<false><<<blocks, threads, sm, s>>>(G, xs, n, n_out, row_src, tk, ldt, err_row);
  check_launch("mode_general_kernel");
}

}  // namespace fstk_gpu
