// A^T A for the core refit on the int8 tensor cores (exact integer slicing).
//
// The Gram of the sketched system (randls.cpp:112-123 solves min ||A x - b||
// by QR; we form A^T A, Cholesky-factor it and refine against A itself) is
// S x R^2 / 2 fused multiply-adds: at C2 that is 1.4e14 fp64 FMAs, 7.6 s at
// the B200's measured DGEMM peak.  Here it runs as int8 x int8 -> int32
// tensor-core GEMMs instead, with no loss of fp64-class accuracy:
//
//  * Per row segment g (<= kseg rows) and column a, e_ga = exponent of
//    max_s |A[s][a]| so v = A * 2^-e_ga lies in (-1, 1).
//  * v is cut into ns signed digits by round-to-nearest:
//      d_1 = rint(64 v),  r = 64 v - d_1,  d_i = rint(128 r), r = 128 r - d_i
//    every step exact in fp64 (Sterbenz), |d_i| <= 64, and
//      v = sum_i d_i 2^(1-7i) + O(2^-7ns).
//  * v_a v_b = sum_t 2^(2-7t) C_t with C_t = sum_{i+j=t} d_i(a) d_j(b).  Each
//    C_t is ONE int8 GEMM: the digit planes of a column are stored
//    consecutively along K ([d_1..d_ns] in X, [d_ns..d_1] in Y), so rows
//    [0, (t-1)k) of X against rows [(ns-t+1)k, ns k) of Y pair exactly the
//    digits with i + j = t.  |C_t| <= (t-1) k 64^2 < 2^31: exact in int32.
//  * Terms with i + j > ns + 1 are dropped.  The fold kernel adds
//    2^(e_a+e_b) sum_t 2^(2-7t) C_t into the fp64 Gram.
//
// ns = 7 gives 49 bits per column-max-relative entry; the Gram is then as
// good a preconditioner as a DGEMM Gram and the iterative refinement against
// A (fp64, fstk_refit.cu) converges to the same least-squares solution.  The
// caller falls back to the native fp64 Gram whenever the sliced one is not
// positive definite or refinement stalls, so rank-deficient systems take the
// exact same path as before.
#include <cublasLt.h>

#include <atomic>
#include <cmath>
#include <string>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>
#include <type_traits>

#include <functional>

#include "fstk_common.cuh"
#include "fstk_crt.cuh"
#include "fstk_internal.h"

namespace fstk_gpu {

namespace {

constexpr int kDigitMax = 64;
constexpr int kDefaultSlices = 2;
constexpr int kMaxSlices = 7;
std::atomic<int> g_slices{-1};

int clamp_slices(int v) { return v <= 0 ? 0 : std::min(std::max(v, 2), kMaxSlices); }

struct LtState {
  cublasLtHandle_t lt = nullptr;
  std::mutex mu;  // guards algos
  std::map<std::tuple<int64_t, int64_t, int64_t, int64_t, int64_t>, cublasLtMatmulAlgo_t> algos;
};
std::mutex g_lt_mu;
std::map<int, LtState*> g_lt;

LtState& lt_state(int device) {
  std::lock_guard<std::mutex> lk(g_lt_mu);
  LtState*& st = g_lt[device];
  if (!st) {
    st = new LtState();
    if (cublasLtCreate(&st->lt) != CUBLAS_STATUS_SUCCESS) fail(FSTK_E_COMPUTE, "cublasLtCreate failed");
  }
  return *st;
}

// a * 2^s exactly for any column exponent: one power-of-two factor when it is
// a normal double, else two (a column max below ~2^-996 needs 2^s > 2^1023).
struct Pow2Scale {
  double f1, f2;
  __device__ explicit Pow2Scale(int s) {
    const int h = s / 2;
    f1 = (s > -1000 && s < 1000) ? ldexp(1.0, s) : ldexp(1.0, h);
    f2 = (s > -1000 && s < 1000) ? 1.0 : ldexp(1.0, s - h);
  }
  __device__ double operator()(double a) const { return (a * f1) * f2; }
};

// Column sources of the sliced Gram.  DenseSrc: a column-major fp64 matrix.
// DesignSrc: the rows of the transform="none" design matrix generated from
// the mode tables, A[r][a] = scale ((u0 u1) u2 ...)(row0 + r) -- the same
// product order as design_block_kernel (fstk_refit.cu), so the values are
// bit-identical and no fp64 A is ever written.
struct DenseSrc {
  const double* A;
  int64_t lda;
  struct Col {
    const double* p;
    __device__ double operator()(int64_t r) const { return p[r]; }
  };
  __device__ Col col(int a) const { return Col{A + static_cast<int64_t>(a) * lda}; }
};

struct DesignSrc {
  DesignSpec s;
  struct Col {
    const double* u[kMaxOrder];
    int d;
    double scale;
    __device__ double operator()(int64_t r) const {
      double v = u[0][r];
#pragma unroll
      for (int k = 1; k < kMaxOrder; ++k)
        if (k < d) v = xmul(v, u[k][r]);
      return xmul(scale, v);
    }
  };
  // (Loops unrolled over kMaxOrder so u[] stays in registers.)
  __device__ Col col(int a) const {
    Col c;
    c.d = s.d;
    c.scale = s.scale;
    int64_t rem = a;
#pragma unroll
    for (int k = 0; k < kMaxOrder; ++k) {
      c.u[k] = s.tables;
      if (k < s.d) {
        const int64_t jk = rem % s.ranks.v[k];
        rem /= s.ranks.v[k];
        c.u[k] = s.tables + s.toff.v[k] + jk * s.ldt + s.row0;
      }
    }
    return c;
  }
};

template <class SRC>
__global__ void col_exponent_kernel(const SRC src, int64_t s0, int64_t rows, int n,
                                    int* __restrict__ ex) {
  const int a = blockIdx.x;
  double m = 0.0;
  if (a < n) {
    const auto col = src.col(a);
    for (int64_t r = threadIdx.x; r < rows; r += blockDim.x) m = fmax(m, fabs(col(s0 + r)));
  }
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  __shared__ double wm[32];
  if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) m = fmax(m, wm[w]);
    int e = 0;
    if (m > 0.0) frexp(m, &e);
    ex[a] = e;
  }
}

// Thread per 4 consecutive rows of one column; X/Y column stride ld = ns*kp.
__global__ void slice_kernel(const double* __restrict__ A, int64_t lda, int64_t rows, int n,
                             int64_t kp, int ns, const int* __restrict__ ex,
                             int8_t* __restrict__ X, int8_t* __restrict__ Y) {
  const int a = blockIdx.x;  // column on grid.x (any n)
  const int64_t r0 = (static_cast<int64_t>(blockIdx.y) * blockDim.x + threadIdx.x) * 4;
  if (r0 >= kp) return;
  const Pow2Scale sc(6 - ex[a]);
  double v[4];
#pragma unroll
  for (int u = 0; u < 4; ++u)
    v[u] = (a < n && r0 + u < rows) ? sc(A[static_cast<int64_t>(a) * lda + r0 + u]) : 0.0;
  const int64_t ld = static_cast<int64_t>(ns) * kp;
  int8_t* xa = X + static_cast<int64_t>(a) * ld + r0;
  int8_t* ya = Y + static_cast<int64_t>(a) * ld + r0;
  for (int i = 0; i < ns; ++i) {
    int q[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double d = rint(v[u]);
      q[u] = static_cast<int>(d);
      v[u] = (v[u] - d) * 128.0;
    }
    const char4 c = make_char4(static_cast<signed char>(q[0]), static_cast<signed char>(q[1]),
                               static_cast<signed char>(q[2]), static_cast<signed char>(q[3]));
    *reinterpret_cast<char4*>(xa + i * kp) = c;
    *reinterpret_cast<char4*>(ya + (ns - 1 - i) * kp) = c;
  }
}

// 2^e as a double for |e| <= 1022 (exact; built from the exponent field).
__device__ __forceinline__ double pow2(int e) {
  return __longlong_as_double(static_cast<long long>(e + 1023) << 52);
}

// G[c0+i][c0+j] (+)= 2^(e_i+e_j) sum_{t>=t_lo} 2^(2-7t) C_t[i][j] for the valid rows
// i >= j of the column block (the lower triangle the solver reads).  The
// plane weights are exact powers of two, applied smallest first.
__global__ void __launch_bounds__(256) fold_kernel(const int32_t* __restrict__ C, int64_t cstride,
                                                   int ns, int t_lo, int64_t m, int w, int c0, int n,
                                                   const int* __restrict__ ex,
                                                   double* __restrict__ G, int accumulate) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int j = blockIdx.y;
  if (i >= m || j >= w || i < j || c0 + i >= n || c0 + j >= n) return;
  const int64_t e = i + static_cast<int64_t>(j) * m;
  const int32_t* c = C + e;
  double v = 0.0;
  for (int t = ns + 1; t >= t_lo; --t)
    v += static_cast<double>(__ldg(c + static_cast<int64_t>(t - t_lo) * cstride)) * pow2(2 - 7 * t);
  // e_i + e_j may leave the normal range only for absurd column scales.
  const int sc = ex[c0 + i] + ex[c0 + j];
  v = (sc > -1000 && sc < 1000) ? v * pow2(sc) : ldexp(v, sc);
  double* g = G + (c0 + i) + static_cast<int64_t>(c0 + j) * n;
  *g = accumulate ? *g + v : v;
}

// C (M x N, int32, col-major, ldc) = op(A)^T B with A: K x M int8 (lda),
// B: K x N int8 (ldb) -- the "TN" IMMA layout cuBLASLt runs on tensor cores.
void imma_tn(LtState& st, DevBuf<uint8_t>& ws, int64_t M, int64_t N, int64_t K, const int8_t* A, int64_t lda,
             const int8_t* B, int64_t ldb, int32_t* Cm, int64_t ldc, cudaStream_t s) {
  cublasLtMatmulDesc_t op = nullptr;
  cublasLtMatrixLayout_t la = nullptr, lb = nullptr, lc = nullptr;
  auto ok = [](cublasStatus_t x, const char* what) {
    if (x != CUBLAS_STATUS_SUCCESS) fail(FSTK_E_COMPUTE, std::string("cuBLASLt: ") + what);
  };
  ok(cublasLtMatmulDescCreate(&op, CUBLAS_COMPUTE_32I, CUDA_R_32I), "desc");
  const cublasOperation_t tA = CUBLAS_OP_T, tB = CUBLAS_OP_N;
  ok(cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSA, &tA, sizeof(tA)), "transa");
  ok(cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSB, &tB, sizeof(tB)), "transb");
  ok(cublasLtMatrixLayoutCreate(&la, CUDA_R_8I, K, M, lda), "layout A");
  ok(cublasLtMatrixLayoutCreate(&lb, CUDA_R_8I, K, N, ldb), "layout B");
  ok(cublasLtMatrixLayoutCreate(&lc, CUDA_R_32I, M, N, ldc), "layout C");
  const auto key = std::make_tuple(M, N, K, lda, ldc);
  cublasLtMatmulAlgo_t algo;
  {
  std::lock_guard<std::mutex> lk(st.mu);
  auto it = st.algos.find(key);
  if (it == st.algos.end()) {
    cublasLtMatmulPreference_t pref = nullptr;
    ok(cublasLtMatmulPreferenceCreate(&pref), "pref");
    const size_t wsz = ws.n;
    ok(cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &wsz,
                                            sizeof(wsz)),
       "pref ws");
    cublasLtMatmulHeuristicResult_t res{};
    int cnt = 0;
    const cublasStatus_t hs =
        cublasLtMatmulAlgoGetHeuristic(st.lt, op, la, lb, lc, lc, pref, 1, &res, &cnt);
    cublasLtMatmulPreferenceDestroy(pref);
    if (hs != CUBLAS_STATUS_SUCCESS || cnt == 0)
      fail(FSTK_E_COMPUTE, "cuBLASLt: no int8 TN algorithm for the sliced Gram");
    it = st.algos.emplace(key, res.algo).first;
  }
  algo = it->second;
  }
  const int32_t one = 1, zero = 0;
  const cublasStatus_t ms = cublasLtMatmul(st.lt, op, &one, A, la, B, lb, &zero, Cm, lc, Cm, lc,
                                           &algo, ws.p, ws.n, s);
  cublasLtMatrixLayoutDestroy(la);
  cublasLtMatrixLayoutDestroy(lb);
  cublasLtMatrixLayoutDestroy(lc);
  cublasLtMatmulDescDestroy(op);
  ok(ms, "matmul");
  count_launch();
}

// ------------------------------------------------------------- CRT scheme ---
// Same Gram, fewer int8 GEMMs (an Ozaki-II-style modular split).  Per segment
// and column, x = rint(A 2^(k-e)) is a k-bit integer (k = 7 ns - 1: the same
// column-max-relative accuracy as ns digit planes, with no dropped terms).
// Its symmetric residues modulo pairwise-coprime m_i <= 255 are int8, and
// C_i = R_i^T R_i (one int8 GEMM per modulus, K = segment rows, exact in
// int32) is sum_s x_a x_b mod m_i.  Garner's algorithm (one reduction per
// digit) rebuilds the exact integer sum in 128-bit arithmetic (|sum| < M/4,
// M = prod m_i), which is converted to fp64 once (exact whenever
// representable) and scaled by 2^(e_a + e_b - 2k).  At ns = 5 that is 11 GEMMs of K rows instead of the
// digit scheme's 15; at ns = 7, 15 instead of 28.

// Symmetric residue of x modulo a compile-time m (unrolled callers), in
// 32-bit arithmetic: x itself when it fits (k <= 30), else two 31-bit halves
// x = hi 2^31 + lo with |hi| < 2^31.
template <bool X32>
__device__ __forceinline__ int sym_mod(long long x, int m) {
  int r;
  if constexpr (X32) {
    r = static_cast<int>(x) % m;
  } else {
    const int hi = static_cast<int>(x >> 31);
    const int lo = static_cast<int>(x & 0x7fffffffll);
    const int p31 = static_cast<int>((1ll << 31) % m);
    r = ((hi % m) * p31 + lo % m) % m;
  }
  if (r > m / 2) r -= m;
  if (r < -(m - 1) / 2) r += m;
  return r;
}

// Thread per RPT consecutive rows of one column (RPT = 16 on the 32-bit
// path: 16 independent loads in flight and one 16-byte store per modulus,
// 4 on the 64-bit path); plane i at X + i * kp * np.  kp % RPT == 0.
template <bool X32>
constexpr int residue_rows() { return X32 ? 16 : 4; }
template <int NM, bool X32, class SRC>
__global__ void __launch_bounds__(128) residue_kernel(const SRC src, int64_t s0, int64_t rows, int n, int64_t kp,
                               int64_t np, int k, const int* __restrict__ ex,
                               int8_t* __restrict__ X) {
  constexpr int RPT = residue_rows<X32>();
  const int a = blockIdx.x;  // column (grid.x: any R; rows on grid.y)
  const int64_t r0 = (static_cast<int64_t>(blockIdx.y) * blockDim.x + threadIdx.x) * RPT;
  if (r0 >= kp) return;
  const Pow2Scale sc(k - ex[a]);
  int8_t* dst = X + static_cast<int64_t>(a) * kp + r0;
  if constexpr (X32) {
    // |x| <= 2^30: 32-bit conversion, and each residue as an unsigned
    // remainder of x + (a multiple of m above 2^30) -- no signed-division
    // fix-ups.  Same symmetric residues as sym_mod.
    int x[RPT];
#pragma unroll
    for (int u = 0; u < RPT; ++u) x[u] = 0;
    if (a < n) {
      const auto col = src.col(a);
      if constexpr (std::is_same<SRC, DenseSrc>::value) {
        // A streams through once per segment: 16-byte loads, no L1 allocation.
        const double* p = col.p + s0 + r0;
        if (r0 + RPT <= rows && (reinterpret_cast<uintptr_t>(p) & 15) == 0) {
#pragma unroll
          for (int u = 0; u < RPT; u += 2) {
            const double2 v = __ldcs(reinterpret_cast<const double2*>(p + u));
            x[u] = __double2int_rn(sc(v.x));
            x[u + 1] = __double2int_rn(sc(v.y));
          }
          goto residues;
        }
      }
      if (r0 + RPT <= rows) {
#pragma unroll
        for (int u = 0; u < RPT; ++u) x[u] = __double2int_rn(sc(col(s0 + r0 + u)));
      } else {
#pragma unroll
        for (int u = 0; u < RPT; ++u)
          if (r0 + u < rows) x[u] = __double2int_rn(sc(col(s0 + r0 + u)));
      }
    }
  residues:
#pragma unroll
    for (int i = 0; i < NM; ++i) {
      const unsigned m = static_cast<unsigned>(kmod(i));
      const unsigned off = ((1u << 30) / m + 1u) * m;
      uint32_t w[RPT / 4];
#pragma unroll
      for (int g = 0; g < RPT / 4; ++g) {
        uint32_t word = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          int v = static_cast<int>((static_cast<unsigned>(x[4 * g + b]) + off) % m);
          if (v > static_cast<int>(m / 2)) v -= static_cast<int>(m);
          word |= (static_cast<uint32_t>(v) & 0xFFu) << (8 * b);
        }
        w[g] = word;
      }
      *reinterpret_cast<uint4*>(dst + static_cast<int64_t>(i) * kp * np) = make_uint4(w[0], w[1], w[2], w[3]);
    }
    return;
  }
  long long x[4] = {0ll, 0ll, 0ll, 0ll};
  if (a < n) {
    const auto col = src.col(a);
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (r0 + u < rows) x[u] = __double2ll_rn(sc(col(s0 + r0 + u)));
  }
#pragma unroll
  for (int i = 0; i < NM; ++i) {
    const char4 c = make_char4(static_cast<signed char>(sym_mod<X32>(x[0], kmod(i))),
                               static_cast<signed char>(sym_mod<X32>(x[1], kmod(i))),
                               static_cast<signed char>(sym_mod<X32>(x[2], kmod(i))),
                               static_cast<signed char>(sym_mod<X32>(x[3], kmod(i))));
    *reinterpret_cast<char4*>(dst + static_cast<int64_t>(i) * kp * np) = c;
  }
}

template <int NM, class CT>
__global__ void __launch_bounds__(256) crt_fold_kernel(const CT* __restrict__ C,
                                                       int64_t cstride, int64_t m, int w, int c0,
                                                       int n, int k, const int* __restrict__ ex,
                                                       double* __restrict__ G, int64_t ldg,
                                                       int accumulate, int negate) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int j = blockIdx.y;
  if (i >= m || j >= w || i < j || c0 + i >= n || c0 + j >= n) return;
  const CT* c = C + i + static_cast<int64_t>(j) * m;
  int r[NM];
#pragma unroll
  for (int t = 0; t < NM; ++t) r[t] = static_cast<int>(__ldg(c + static_cast<int64_t>(t) * cstride));
  // C is the int32 sum (cuBLASLt engine) or its symmetric residue: congruent
  // mod m_t, so the Garner digits are identical.
  const double v0 = crt_scale(crt_value<NM, sizeof(CT) == 1>(r), ex[c0 + i] + ex[c0 + j] - 2 * k);
  const double v = negate ? -v0 : v0;
  double* g = G + (c0 + i) + static_cast<int64_t>(c0 + j) * ldg;
  *g = accumulate ? *g + v : v;
}

// Byte-residue fold (SYRK engine): four consecutive rows per thread -- one
// 4-byte load per plane, four independent Garner chains in flight, and the
// four G entries contiguous.  m % 4 == 0 (column blocks are 256-aligned).
template <int NM>
__global__ void __launch_bounds__(256) crt_fold4_kernel(const int8_t* __restrict__ C, int64_t cstride, int64_t m,
                                                        int w, int c0, int n, int k, const int* __restrict__ ex,
                                                        double* __restrict__ G, int64_t ldg, int accumulate,
                                                        int negate) {
  const int64_t i0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 4;
  const int j = blockIdx.y;
  if (i0 >= m || j >= w || i0 + 3 < j || c0 + j >= n) return;
  const int8_t* c = C + i0 + static_cast<int64_t>(j) * m;
  char4 rb[NM];
#pragma unroll
  for (int t = 0; t < NM; ++t) rb[t] = __ldg(reinterpret_cast<const char4*>(c + static_cast<int64_t>(t) * cstride));
  const int ej = ex[c0 + j];
  double* g = G + (c0 + i0) + static_cast<int64_t>(c0 + j) * ldg;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int64_t i = i0 + u;
    if (i < j || c0 + i >= n) continue;
    int r[NM];
#pragma unroll
    for (int t = 0; t < NM; ++t)
      r[t] = u == 0 ? rb[t].x : u == 1 ? rb[t].y : u == 2 ? rb[t].z : rb[t].w;
    const double v0 = crt_scale(crt_value<NM, true>(r), ex[c0 + i] + ej - 2 * k);
    const double v = negate ? -v0 : v0;
    g[u] = accumulate ? g[u] + v : v;
  }
}

// Moduli for k-bit integers summed over kp rows: M > 4 kp 2^(2k).
int crt_moduli(int k, int64_t kp) {
  const double need = 2.0 + std::log2(static_cast<double>(std::max<int64_t>(kp, 1))) + 2.0 * k;
  double have = 0.0;
  for (int i = 0; i < kMaxModuli; ++i) {
    have += std::log2(static_cast<double>(kmod(i)));
    if (have > need + 0.25) return i + 1;
  }
  return -1;
}

template <int NM, class SRC>
void launch_crt(const SRC& src, int64_t s0, int64_t kr, int n, int64_t kp, int64_t np, int k,
                const int* ex, int8_t* X, cudaStream_t s) {
  if (k <= 30) {
    dim3 g(static_cast<unsigned>(np), static_cast<unsigned>(ceil_div(kp / residue_rows<true>(), 128)));
    residue_kernel<NM, true, SRC><<<g, 128, 0, s>>>(src, s0, kr, n, kp, np, k, ex, X);
  } else {
    dim3 g(static_cast<unsigned>(np), static_cast<unsigned>(ceil_div(kp / residue_rows<false>(), 128)));
    residue_kernel<NM, false, SRC><<<g, 128, 0, s>>>(src, s0, kr, n, kp, np, k, ex, X);
  }
  check_launch("residue_kernel");
}
template <int NM, class CT>
void launch_crt_fold(const CT* C, int64_t cstride, int64_t m, int64_t wn, int64_t c0, int n,
                     int k, const int* ex, double* G, int64_t ldg, int acc, int neg, cudaStream_t s) {
  if constexpr (sizeof(CT) == 1) {
    if (m % 4 == 0 && cstride % 4 == 0) {
      dim3 fg(static_cast<unsigned>(ceil_div(m, 1024)), static_cast<unsigned>(wn));
      crt_fold4_kernel<NM><<<fg, 256, 0, s>>>(C, cstride, m, static_cast<int>(wn), static_cast<int>(c0), n, k,
                                             ex, G, ldg, acc, neg);
      check_launch("crt_fold4_kernel");
      return;
    }
  }
  dim3 fg(static_cast<unsigned>(ceil_div(m, 256)), static_cast<unsigned>(wn));
  crt_fold_kernel<NM, CT><<<fg, 256, 0, s>>>(C, cstride, m, static_cast<int>(wn), static_cast<int>(c0),
                                             n, k, ex, G, ldg, acc, neg);
  check_launch("crt_fold_kernel");
}

#define FSTK_CRT_SWITCH(NMV, CALL)                                              \
  switch (NMV) {                                                                \
    case 7: CALL(7); break;                                                     \
    case 8: CALL(8); break;                                                     \
    case 9: CALL(9); break;                                                     \
    case 10: CALL(10); break;                                                   \
    case 11: CALL(11); break;                                                   \
    case 12: CALL(12); break;                                                   \
    case 13: CALL(13); break;                                                   \
    case 14: CALL(14); break;                                                   \
    case 15: CALL(15); break;                                                   \
    case 16: CALL(16); break;                                                   \
    case 17: CALL(17); break;                                                   \
    default: fail(FSTK_E_COMPUTE, "internal: unsupported CRT modulus count");   \
  }

}  // namespace

// Bits per entry of a CRT Gram level.  Levels 4..7 carry the accuracy of that
// many 7-bit planes (k = 7 level - 1).  Levels 3 and 2 are defined from the
// other side: the most bits that 8 and 7 moduli carry over a segment (23 and
// 19 at 32,768 rows).  As preconditioners of a mixed sketch they keep the
// refinement's contraction per step below 2e-4 and 3e-3 at C2
// (tools/refine_time.py), well inside the 0.1 that escalates, for 8/9 and 7/9
// of level 4's int8 work.  Level 2 is the default (DESIGN 3.4).
int crt_level_bits(int level) { return level == 3 ? 23 : (level == 2 ? 19 : 7 * level - 1); }
int crt_low_level_moduli(int level) { return level == 3 ? 8 : 7; }
int crt_low_level_bits(int level, int64_t kp) {
  const int nm = crt_low_level_moduli(level);
  double have = 0.0;
  for (int i = 0; i < nm; ++i) have += std::log2(static_cast<double>(kmod(i)));
  const double room = have - 0.25 - 2.0 - std::log2(static_cast<double>(std::max<int64_t>(kp, 1)));
  return std::max(12, std::min(crt_level_bits(level), static_cast<int>(std::floor(room / 2.0 - 1e-9))));
}


namespace {
std::atomic<int> g_engine{-1};
}

int gram_engine() {
  int v = g_engine.load();
  if (v < 0) {
    const char* e = std::getenv("FSTK_GRAM_GEMM");
    v = (e && std::string(e) == "cublaslt") ? 2 : 1;
    g_engine.store(v);
  }
  return v;
}

int set_gram_engine(int engine) {
  const int prev = gram_engine();
  if (engine == 1 || engine == 2) g_engine.store(engine);
  return prev;
}

int gram_slices() {
  int v = g_slices.load();
  if (v < 0) {
    const char* e = std::getenv("FSTK_GRAM_SLICES");
    v = clamp_slices(e ? std::atoi(e) : kDefaultSlices);
    g_slices.store(v);
  }
  return v;
}

int set_gram_slices(int slices) {
  const int prev = gram_slices();
  g_slices.store(slices < 0 ? prev : clamp_slices(slices));
  return prev;
}

bool gram_sliced_applies(int64_t rows, int n) { return gram_slices() > 0 && n >= 256 && rows > 0; }

// gram (n x n, col-major, lower triangle) = beta * gram + A^T A over `rows`
// rows of A (col-major, lda).
double gram_accumulate_crt(const double* A, int64_t lda, int64_t rows, int n, double* gram,
                           double beta, int ns, cudaStream_t s, int device, GramScratch& sc);
bool gram_scheme_crt();

double gram_accumulate_sliced(const double* A, int64_t lda, int64_t rows, int n, double* gram,
                              double beta, int ns, int t_lo, cudaStream_t s, int device,
                              GramScratch& sc) {
  if (t_lo == 2 && gram_scheme_crt())
    return gram_accumulate_crt(A, lda, rows, n, gram, beta, ns, s, device, sc);
  double ops = 0.0;
  if (ns < 4) ns = 4;  // levels 2 and 3 exist in the CRT scheme only
  require(ns >= 4 && ns <= kMaxSlices, FSTK_E_PARAMETER, "sliced Gram: 4..7 digit planes");
  require(t_lo >= 2 && t_lo <= ns + 1, FSTK_E_PARAMETER, "sliced Gram: bad plane range");
  const int nt = ns + 2 - t_lo;  // plane sums t_lo..ns+1
  LtState& st = lt_state(device);
  const int64_t np = round_up(static_cast<int64_t>(n), 16);
  // Column blocks: C_t planes (ns of them, m x w int32) within ~4 GB; 2048
  // wide by default, so the wasted upper half of each diagonal block (the
  // GEMMs compute full m x w tiles) stays ~6% of the triangle.
  static const int64_t block_cap = [] {
    const char* e = std::getenv("FSTK_GRAM_BLOCK");
    return e ? std::max<int64_t>(256, std::atoll(e)) : int64_t(2048);
  }();
  int64_t w = std::max<int64_t>(256, (int64_t(4) << 30) / (np * nt * 4));
  w = std::min<int64_t>(round_up(std::min<int64_t>(w, np), 16), np);
  if (w > block_cap && np > block_cap) w = round_up(block_cap, 16);
  // Segment rows: int32-exact for any plane count, digit planes (X and Y)
  // within a third of the free memory (at most 24 GB), 16384 by default
  // (measured best at C2: longer K makes cuBLASLt pick slower kernels).  The
  // first call on a scratch fixes the segment length: the per-segment column
  // exponents, hence the digits, must be the same when a later call adds
  // more plane sums (the progressive upgrade in fstk_refit.cu).
  int64_t kmax = ((int64_t(1) << 31) - 1) / (int64_t(kDigitMax) * kDigitMax * kMaxSlices);
  kmax = std::min<int64_t>(kmax, 65536);
  size_t free_b = 0, total_b = 0;
  if (device_mem_info(&free_b, &total_b) != cudaSuccess) {
    cudaGetLastError();
    free_b = size_t(24) << 30;
  }
  const int64_t have = static_cast<int64_t>(sc.X.n + sc.Y.n);  // reusable scratch
  const int64_t plane_budget =
      std::min<int64_t>(int64_t(24) << 30, (static_cast<int64_t>(free_b) + have) / 3);
  kmax = std::min<int64_t>(kmax, std::max<int64_t>(1024, plane_budget / (2 * ns * np)));
  static const int64_t seg_cap = [] {
    const char* e = std::getenv("FSTK_GRAM_SEG");
    return e ? std::max<int64_t>(1024, std::atoll(e)) : int64_t(16384);
  }();
  kmax = std::min(kmax, seg_cap);
  kmax &= ~int64_t(15);
  if (sc.kp == 0) sc.kp = kmax;
  const int64_t kp = std::min<int64_t>(sc.kp, round_up(rows, 16));
  const int64_t ld = ns * kp;
  sc.X.ensure(static_cast<size_t>(ld * np));
  sc.Y.ensure(static_cast<size_t>(ld * np));
  sc.C.ensure(static_cast<size_t>(nt) * np * w);
  sc.ex.ensure(static_cast<size_t>(np));
  sc.ws.ensure(size_t(32) << 20);
  DevBuf<int8_t>& X = sc.X;
  DevBuf<int8_t>& Y = sc.Y;
  DevBuf<int32_t>& Cb = sc.C;
  DevBuf<int>& ex = sc.ex;
  bool first = true;
  for (int64_t s0 = 0; s0 < rows; s0 += kp) {
    const int64_t kr = std::min(kp, rows - s0);
    col_exponent_kernel<DenseSrc><<<static_cast<unsigned>(np), 256, 0, s>>>(DenseSrc{A, lda}, s0, kr, n,
                                                                           ex.p);
    check_launch("col_exponent_kernel");
    dim3 sg(static_cast<unsigned>(np), static_cast<unsigned>(ceil_div(kp / 4, 256)));
    slice_kernel<<<sg, 256, 0, s>>>(A + s0, lda, kr, n, kp, ns, ex.p, X.p, Y.p);
    check_launch("slice_kernel");
    for (int64_t c0 = 0; c0 < np; c0 += w) {
      const int64_t wn = std::min(w, np - c0);
      const int64_t m = np - c0;
      for (int t = t_lo; t <= ns + 1; ++t) {
        const int64_t K = (t - 1) * kp;
        ops += 2.0 * static_cast<double>(m) * static_cast<double>(wn) * static_cast<double>(K);
        imma_tn(st, sc.ws, m, wn, K, X.p + c0 * ld, ld, Y.p + c0 * ld + (ns - t + 1) * kp, ld,
                Cb.p + static_cast<int64_t>(t - t_lo) * m * wn, m, s);
      }
      dim3 fg(static_cast<unsigned>(ceil_div(m, 256)), static_cast<unsigned>(wn));
      const int acc = (!first || beta != 0.0) ? 1 : 0;
      fold_kernel<<<fg, 256, 0, s>>>(Cb.p, m * wn, ns, t_lo, m, static_cast<int>(wn),
                                     static_cast<int>(c0), n, ex.p, gram, acc);
      check_launch("fold_kernel");
    }
    first = false;
  }
  return ops;
}

bool gram_scheme_crt() {
  static const bool crt = [] {
    const char* e = std::getenv("FSTK_GRAM_SCHEME");
    return !(e && std::string(e) == "digits");
  }();
  return crt;
}

// CRT variant of gram_accumulate_sliced (whole Gram, t_lo = 2 semantics).
template <class SRC>
static double gram_accumulate_crt_src(const SRC& src, int64_t rows, int n, double* gram,
                                      double beta, int ns, cudaStream_t s, int device,
                                      GramScratch& sc, int64_t ldg = -1, bool negate = false,
                                      cudaEvent_t first_block_done = nullptr,
                                      const std::function<void()>* after_first_block = nullptr) {
  if (ldg < 0) ldg = n;
  require(ns >= 2 && ns <= 7, FSTK_E_PARAMETER, "CRT Gram: levels 2..7");
  int k = crt_level_bits(ns);
  // SYRK engine: 256-column tiles and 128-byte K blocks (zero padding).  It
  // folds each tile in its epilogue while the next tile's MMAs run, which
  // hides the fold only when a tile's K loop is long: short updates (the
  // blocked Cholesky's 2048-row trailing updates, outside the hot path) keep
  // the library GEMMs and the separate fold kernel.
  static const int64_t syrk_min_rows = [] {
    const char* e = std::getenv("FSTK_SYRK_MIN_ROWS");
    return e ? std::atoll(e) : int64_t(8192);
  }();
  // (The SYRK's band table covers up to 131,072 columns; wider Grams keep the
  // library engine.)
  const bool syrk = gram_engine() == 1 && rows >= syrk_min_rows && n <= 131072;
  const bool fused = syrk && syrk_fused() && ns > 2;  // the fused kernel is instantiated from 8 moduli
  const int64_t np = round_up(static_cast<int64_t>(n), syrk ? 256 : 16);
  const int64_t kalign = syrk ? 128 : 16;
  static const int64_t seg_cap = [] {
    const char* e = std::getenv("FSTK_GRAM_SEG");
    return e ? std::max<int64_t>(1024, std::atoll(e)) : int64_t(32768);
  }();
  // int32-exact: K * 127^2 < 2^31; residue planes within a third of free
  // memory (<= 24 GB).
  // (The SYRK engine's integer epilogue needs |sums| < 2^30: <= 65536 rows.)
  int64_t kmax = std::min<int64_t>(seg_cap, syrk ? int64_t(65536) : ((int64_t(1) << 31) - 1) / (127 * 127));
  size_t free_b = 0, total_b = 0;
  if (device_mem_info(&free_b, &total_b) != cudaSuccess) {
    cudaGetLastError();
    free_b = size_t(24) << 30;
  }
  // Sized per call for this call's modulus count (an escalation to a higher
  // level re-sizes; the CRT sums are exact per segment, so the segment length
  // does not change what a call computes beyond fp64 accumulation order).
  // Sizing for the level-7 count on every call shrank C4's segments to ~20k
  // rows next to its 137 GB sketch (Gram 2.8 s instead of 2.3 s).
  // Levels 2 and 3 are 7 and 8 moduli whatever the segment length; their bits
  // follow from kp below.
  const int nm_need = ns <= 3 ? crt_low_level_moduli(ns) : std::max(8, crt_moduli(k, kmax));
  const int64_t have = static_cast<int64_t>(sc.X.n);
  const int64_t budget = std::min<int64_t>(int64_t(24) << 30, (static_cast<int64_t>(free_b) + have) / 3);
  kmax = std::min<int64_t>(kmax, std::max<int64_t>(1024, budget / (nm_need * np)));
  kmax &= ~(kalign - 1);
  const int64_t kp = std::min<int64_t>(kmax, round_up(rows, kalign));
  if (ns <= 3) k = crt_low_level_bits(ns, kp);
  // (Short segments would need fewer; the kernels are instantiated from 7.)
  const int nm = std::max(ns <= 3 ? crt_low_level_moduli(ns) : 8, crt_moduli(k, kp));
  require(nm >= 7 && nm <= 17, FSTK_E_COMPUTE, "internal: CRT modulus count out of range");
  static const int64_t block_cap = [] {
    const char* e = std::getenv("FSTK_GRAM_BLOCK");
    return e ? std::max<int64_t>(256, std::atoll(e)) : int64_t(2048);
  }();
  const int64_t wal = syrk ? 256 : 16;
  int64_t w = std::max<int64_t>(256, (int64_t(4) << 30) / (np * nm * (syrk ? 1 : 4)));
  w = std::min<int64_t>(round_up(std::min<int64_t>(w, np), wal), np);
  if (w > block_cap && np > block_cap) w = round_up(block_cap, wal);
  sc.last_block_w = fused ? 0 : w;  // fused: no per-block order to hook into
  sc.X.ensure(static_cast<size_t>(nm) * kp * np);
  if (fused) {
    sc.C8.ensure(syrk_crt_scratch_bytes(nm, device));
  } else if (syrk) {
    sc.C8.ensure(static_cast<size_t>(nm) * np * w + 256);  // + the scheduler's task counter
  } else {
    sc.C.ensure(static_cast<size_t>(nm) * np * w);
    sc.ws.ensure(size_t(32) << 20);
  }
  sc.ex.ensure(static_cast<size_t>(np));
  double ops = 0.0;
  bool first = true;
  for (int64_t s0 = 0; s0 < rows; s0 += kp) {
    const int64_t kr = std::min(kp, rows - s0);
    col_exponent_kernel<SRC><<<static_cast<unsigned>(np), 256, 0, s>>>(src, s0, kr, n, sc.ex.p);
    check_launch("col_exponent_kernel");
#define FSTK_CRT_RES(NMV) launch_crt<NMV, SRC>(src, s0, kr, n, kp, np, k, sc.ex.p, sc.X.p, s)
    FSTK_CRT_SWITCH(nm, FSTK_CRT_RES)
#undef FSTK_CRT_RES
    const int acc = (!first || beta != 0.0) ? 1 : 0;
    if (fused) {
      // One persistent tcgen05 launch: the whole lower triangle, every
      // modulus, Garner fold in the epilogue.
      ops += syrk_crt_fold(sc.X.p, nm, kp, np, n, k, sc.ex.p, gram, ldg, acc != 0, negate, sc.C8.p,
                           device, s);
    } else if (syrk) {
      for (int64_t c0 = 0; c0 < np; c0 += w) {
        const int64_t wn = std::min(w, np - c0);
        const int64_t m = np - c0;
        int8_t* c8 = reinterpret_cast<int8_t*>(sc.C8.p);
        int* counter = reinterpret_cast<int*>(sc.C8.p + static_cast<size_t>(nm) * np * w);
        if (syrk_mode() == 0) {  // one launch per modulus (default: measured fastest)
          for (int t = 0; t < nm; ++t)
            ops += syrk_i8_residues_one(sc.X.p, nm, t, kp, np, c0, wn, m, c8 + t * m * wn, counter, device, s);
        } else {
          ops += syrk_i8_residues(sc.X.p, nm, kp, np, c0, wn, m, c8, m * wn, counter, device, s);
        }
#define FSTK_CRT_FOLD(NMV) \
  launch_crt_fold<NMV, int8_t>(c8, m * wn, m, wn, c0, n, k, sc.ex.p, gram, ldg, acc, negate ? 1 : 0, s)
        FSTK_CRT_SWITCH(nm, FSTK_CRT_FOLD)
#undef FSTK_CRT_FOLD
        if (first_block_done && c0 == 0 && s0 + kp >= rows) {
          FSTK_CUDA(cudaEventRecord(first_block_done, s));
          // The caller's dependent work is enqueued here, ahead of the other
          // blocks' launches: the launch queue is finite, and work issued after
          // this whole update would reach the GPU only as the update drains.
          if (after_first_block) (*after_first_block)();
        }
      }
    } else {
      LtState& st = lt_state(device);
      for (int64_t c0 = 0; c0 < np; c0 += w) {
        const int64_t wn = std::min(w, np - c0);
        const int64_t m = np - c0;
        for (int t = 0; t < nm; ++t) {
          const int8_t* Rt = sc.X.p + static_cast<int64_t>(t) * kp * np;
          ops += 2.0 * static_cast<double>(m) * static_cast<double>(wn) * static_cast<double>(kp);
          imma_tn(st, sc.ws, m, wn, kp, Rt + c0 * kp, kp, Rt + c0 * kp, kp,
                  sc.C.p + static_cast<int64_t>(t) * m * wn, m, s);
        }
#define FSTK_CRT_FOLD(NMV) \
  launch_crt_fold<NMV, int32_t>(sc.C.p, m * wn, m, wn, c0, n, k, sc.ex.p, gram, ldg, acc, negate ? 1 : 0, s)
        FSTK_CRT_SWITCH(nm, FSTK_CRT_FOLD)
#undef FSTK_CRT_FOLD
        if (first_block_done && c0 == 0 && s0 + kp >= rows) {
          FSTK_CUDA(cudaEventRecord(first_block_done, s));
          // The caller's dependent work is enqueued here, ahead of the other
          // blocks' launches: the launch queue is finite, and work issued after
          // this whole update would reach the GPU only as the update drains.
          if (after_first_block) (*after_first_block)();
        }
      }
    }
    first = false;
  }
  return ops;
}

double gram_accumulate_crt(const double* A, int64_t lda, int64_t rows, int n, double* gram,
                           double beta, int ns, cudaStream_t s, int device, GramScratch& sc) {
  return gram_accumulate_crt_src(DenseSrc{A, lda}, rows, n, gram, beta, ns, s, device, sc);
}

double gram_update_crt(const double* T, int64_t ldt, int64_t rows, int n, double* G, int64_t ldg,
                       int ns, cudaStream_t s, int device, GramScratch& sc,
                       cudaEvent_t first_block_done, int64_t* first_block_cols,
                       const std::function<void()>* after_first_block, int64_t need_cols) {
  // The first column block is min(2048, n) columns wide (block_cap) unless the
  // scratch budget narrows it; a caller overlapping work with the rest of the
  // update must wait for the whole update when the block is narrower than it needs.
  if (first_block_cols) *first_block_cols = 0;
  // The callback runs inside only when the first block will be wide enough
  // for the caller (block_cap columns unless the scratch budget narrows it:
  // known only inside, so the width is checked there through last_block_w).
  struct Gate {
    GramScratch& sc;
    const std::function<void()>* cb;
    int64_t need;
    bool fired = false;
  } gate{sc, after_first_block, need_cols};
  std::function<void()> gated = [&gate] {
    if (gate.cb && gate.sc.last_block_w >= gate.need) {
      (*gate.cb)();
      gate.fired = true;
    }
  };
  const double ops = gram_accumulate_crt_src(DenseSrc{T, ldt}, rows, n, G, 1.0, ns, s, device, sc, ldg, true,
                                             first_block_done, after_first_block ? &gated : nullptr);
  if (after_first_block && !gate.fired) sc.last_block_w = 0;  // tell the caller to wait for the whole update
  if (first_block_cols) *first_block_cols = sc.last_block_w;
  return ops;
}

double gram_accumulate_sliced_design(const DesignSpec& spec, int64_t rows, int n, double* gram,
                                     double beta, int ns, cudaStream_t s, int device,
                                     GramScratch& sc) {
  return gram_accumulate_crt_src(DesignSrc{spec}, rows, n, gram, beta, ns, s, device, sc);
}

}  // namespace fstk_gpu
