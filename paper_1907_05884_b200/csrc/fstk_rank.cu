// The reference's rank decision and minimum-norm fallback on the GPU
// (proj/src/randls.cpp:112-123):
//
//   Eigen::ColPivHouseholderQR<Matrix> qr(a);
//   if (qr.rank() == a.cols()) alpha = qr.solve(b);
//   else { rank_deficient = true; alpha = CompleteOrthogonalDecomposition(a).solve(b); }
//
// rank() counts |R_ii| > min(m, n) * eps * max_i |R_ii| (Eigen's default
// threshold).  Three pieces:
//
//  * QrStream -- streaming TSQR: the R factor of the augmented system [A b]
//    (n + 1 columns), folded row block by row block with cuSOLVER geqrf on an
//    (n1 + block) x n1 scratch.  A is never modified, so the sketch stays
//    available; R of [A b] carries c = Q^T b in its last column.  Row shards
//    (several GPUs, or several ranks) fold their own R and stack them
//    (fstk_gpu_qr_stack): column-pivoted QR is invariant under the orthogonal
//    Q, so pivoting R reproduces the pivoting of A itself.
//  * cpqr_* kernels -- Householder QR with column pivoting on that R, step by
//    step like Eigen's ColPivHouseholderQR::computeInPlace: pivot on the
//    largest updated column norm (first index on ties), Eigen's
//    makeHouseholderInPlace sign and scaling, applyHouseholderOnTheLeft on
//    the trailing columns (c included, never pivoted), and the LAPACK
//    lawn176 norm downdate with recomputation below sqrt(eps).
//  * the solve: full rank -> x = P R^{-1} c; deficient -> the COD's
//    minimum-norm solution of the rank-k system [R11 R12] P^T x = c_k, i.e.
//    x = P Q3 U^{-T} c_k from the QR of [R11 R12]^T = Q3 U.
//
// The refit only takes this path when its Cholesky route cannot certify
// full rank (fstk_refit.cu, refit_solve); the usual full-rank system is
// solved by Cholesky + refinement against A and certified by a cheap
// smallest-singular-value bound (chol_lambda_min_estimate).
#include <cublas_v2.h>
#include <cusolverDn.h>

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <condition_variable>
#include <deque>
#include <thread>
#include <vector>

#include "fstk_internal.h"

namespace fstk_gpu {

// ------------------------------------------------------------- kernels ---
// Zeroes the strictly lower triangle of the leading n1 x n1 block (the
// Householder vectors geqrf leaves there).
__global__ void zero_lower_kernel(double* __restrict__ W, int64_t ld, int n1) {
  const int j = blockIdx.y;
  for (int i = j + 1 + blockIdx.x * blockDim.x + threadIdx.x; i < n1; i += gridDim.x * blockDim.x)
    W[i + j * ld] = 0.0;
}

// vn1[j] = vn2[j] = ||M[:, j]|| (Eigen: m_qr.col(k).norm(), a plain sum of
// squares).  One warp per column.
__global__ void cpqr_colnorm_kernel(const double* __restrict__ M, int64_t ld, int m, int n,
                                    double* __restrict__ vn1, double* __restrict__ vn2) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= n) return;
  const double* c = M + static_cast<int64_t>(warp) * ld;
  double s = 0.0;
  for (int i = lane; i < m; i += 32) s = fma(c[i], c[i], s);
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) {
    vn1[warp] = sqrt(s);
    vn2[warp] = vn1[warp];
  }
}

constexpr int kPivThreads = 1024;

// Step k, part 1 (one CTA): pivot = argmax_{j in [k, n)} vn1[j] (first index
// on ties), swap it into column k, then the Householder reflector of
// M[k:m, k] in place (Eigen makeHouseholderInPlace): beta = -+sqrt(c0^2 +
// |tail|^2) with the sign opposite to c0 (c0 >= 0 -> negative), essential =
// tail / (c0 - beta), tau = (beta - c0) / beta; tail^2 <= DBL_MIN -> tau = 0.
__global__ void __launch_bounds__(kPivThreads) cpqr_pivot_kernel(
    double* __restrict__ M, int64_t ld, int m, int n, int k, double* __restrict__ vn1,
    double* __restrict__ vn2, int* __restrict__ perm, double* __restrict__ tau,
    double* __restrict__ diag) {
  __shared__ double sv[kPivThreads / 32];
  __shared__ int si[kPivThreads / 32];
  __shared__ int piv;
  __shared__ double ssum[kPivThreads / 32];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  double bv = -1.0;
  int bi = INT_MAX;
  for (int j = k + t; j < n; j += kPivThreads) {
    const double v = vn1[j];
    if (v > bv) {  // j increases per thread: strict > keeps the first index
      bv = v;
      bi = j;
    }
  }
  for (int o = 16; o; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > bv || (ov == bv && oi < bi)) {
      bv = ov;
      bi = oi;
    }
  }
  if (lane == 0) {
    sv[w] = bv;
    si[w] = bi;
  }
  __syncthreads();
  if (w == 0) {
    bv = lane < kPivThreads / 32 ? sv[lane] : -1.0;
    bi = lane < kPivThreads / 32 ? si[lane] : INT_MAX;
    for (int o = 16; o; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) {
        bv = ov;
        bi = oi;
      }
    }
    if (lane == 0) piv = (bi == INT_MAX) ? k : bi;
  }
  __syncthreads();
  const int p = piv;
  double* ck = M + static_cast<int64_t>(k) * ld;
  if (p != k) {
    double* cp = M + static_cast<int64_t>(p) * ld;
    for (int i = t; i < m; i += kPivThreads) {
      const double a = ck[i];
      ck[i] = cp[i];
      cp[i] = a;
    }
    if (t == 0) {
      double x = vn1[k]; vn1[k] = vn1[p]; vn1[p] = x;
      x = vn2[k]; vn2[k] = vn2[p]; vn2[p] = x;
      const int q = perm[k]; perm[k] = perm[p]; perm[p] = q;
    }
  }
  __syncthreads();
  double s = 0.0;
  for (int i = k + 1 + t; i < m; i += kPivThreads) s = fma(ck[i], ck[i], s);
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) ssum[w] = s;
  __syncthreads();
  if (t == 0) {
    double tail = 0.0;
    for (int i = 0; i < kPivThreads / 32; ++i) tail += ssum[i];
    ssum[0] = tail;
  }
  __syncthreads();
  const double tail = ssum[0];
  const double c0 = ck[k];
  double beta, tk, denom;
  if (tail <= DBL_MIN) {
    tk = 0.0;
    beta = c0;
    denom = 0.0;
  } else {
    beta = sqrt(c0 * c0 + tail);
    if (c0 >= 0.0) beta = -beta;
    tk = (beta - c0) / beta;
    denom = c0 - beta;
  }
  __syncthreads();  // every thread has read c0 before it is overwritten
  for (int i = k + 1 + t; i < m; i += kPivThreads) ck[i] = denom != 0.0 ? ck[i] / denom : 0.0;
  if (t == 0) {
    ck[k] = beta;
    tau[k] = tk;
    diag[k] = beta;
  }
}

constexpr int kApplyThreads = 256;

// Step k, part 2: one CTA per trailing column j in (k, ncols): the
// reflector applied from the left (tmp = v^T M[k:, j] with v = [1; essential];
// M[k:, j] -= tau v tmp), then, for pivot candidates j < n, Eigen's norm
// downdate: temp = (1 + a)(1 - a) with a = |M[k, j]| / vn1[j], clipped at 0;
// if temp (vn1/vn2)^2 <= sqrt(eps) recompute vn1 = vn2 = ||M[k+1:, j]||,
// else vn1 *= sqrt(temp).
__global__ void __launch_bounds__(kApplyThreads) cpqr_apply_kernel(
    double* __restrict__ M, int64_t ld, int m, int ncols, int n, int k,
    const double* __restrict__ tau, double* __restrict__ vn1, double* __restrict__ vn2) {
  __shared__ double red[kApplyThreads / 32];
  __shared__ double bc;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const double tk = tau[k];
  const double* v = M + static_cast<int64_t>(k) * ld;
  for (int j = k + 1 + blockIdx.x; j < ncols; j += gridDim.x) {
    double* c = M + static_cast<int64_t>(j) * ld;
    if (tk != 0.0) {
      double s = 0.0;
      for (int i = k + 1 + t; i < m; i += kApplyThreads) s = fma(v[i], c[i], s);
      for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) red[w] = s;
      __syncthreads();
      if (t == 0) {
        double tot = 0.0;
        for (int i = 0; i < kApplyThreads / 32; ++i) tot += red[i];
        bc = tot + c[k];
      }
      __syncthreads();
      const double tmp = bc;
      if (t == 0) c[k] -= tk * tmp;
      for (int i = k + 1 + t; i < m; i += kApplyThreads) c[i] -= (tk * v[i]) * tmp;
      __syncthreads();
    }
    if (j < n) {
      // Norm downdate (LAPACK lawn176, as Eigen's ColPivHouseholderQR).
      const double u = vn1[j];
      bool recompute = false;
      double scale = 1.0;
      if (u != 0.0) {
        double a = fabs(c[k]) / u;
        a = (1.0 + a) * (1.0 - a);
        a = a < 0.0 ? 0.0 : a;
        const double r = u / vn2[j];
        const double temp2 = a * r * r;
        recompute = temp2 <= 1.4901161193847656e-08;  // sqrt(DBL_EPSILON)
        scale = sqrt(a);
      }
      if (recompute) {
        double s = 0.0;
        for (int i = k + 1 + t; i < m; i += kApplyThreads) s = fma(c[i], c[i], s);
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) red[w] = s;
        __syncthreads();
        if (t == 0) {
          double tot = 0.0;
          for (int i = 0; i < kApplyThreads / 32; ++i) tot += red[i];
          vn1[j] = sqrt(tot);
          vn2[j] = vn1[j];
        }
        __syncthreads();
      } else if (t == 0 && u != 0.0) {
        vn1[j] = u * scale;
      }
    }
  }
}

// T (n x k, ld n) = [R11 R12]^T: T[j, i] = M[i, j] for j >= i, 0 above.
__global__ void trapezoid_transpose_kernel(const double* __restrict__ M, int64_t ld, int n, int k,
                                           double* __restrict__ T) {
  const int i = blockIdx.y;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x)
    T[j + static_cast<int64_t>(i) * n] = j >= i ? M[i + static_cast<int64_t>(j) * ld] : 0.0;
}

// x[perm[i]] = y[i].
__global__ void scatter_perm_kernel(const double* __restrict__ y, const int* __restrict__ perm,
                                    int n, double* __restrict__ x) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[perm[i]] = y[i];
}

__global__ void iota_kernel(int* __restrict__ p, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = i;
}

// ----------------------------------------------------------- QrStream ---
void QrStream::init(int n1_, int64_t bmax_, cudaStream_t s_, int device_) {
  n1 = n1_;
  bmax = std::max<int64_t>(bmax_, 1);
  s = s_;
  device = device_;
  ldw = n1 + bmax;
  W.alloc(static_cast<size_t>(ldw) * n1);
  FSTK_CUDA(cudaMemsetAsync(W.p, 0, static_cast<size_t>(ldw) * n1 * 8, s));
  tau.alloc(static_cast<size_t>(n1));
  info.alloc(1);
  cusolverDnHandle_t h = solver_handle(device);
  cusolverDnSetStream(h, s);
  if (!params && cusolverDnCreateParams(&params) != CUSOLVER_STATUS_SUCCESS)
    fail(FSTK_E_COMPUTE, "cusolverDnCreateParams failed");
  size_t dev_b = 0, host_b = 0;
  if (cusolverDnXgeqrf_bufferSize(h, params, ldw, n1, CUDA_R_64F, W.p, ldw, CUDA_R_64F, tau.p,
                                  CUDA_R_64F, &dev_b, &host_b) != CUSOLVER_STATUS_SUCCESS)
    fail(FSTK_E_COMPUTE, "geqrf_bufferSize failed");
  work.alloc(std::max<size_t>(dev_b, 8));
  work_bytes = std::max<size_t>(dev_b, 8);
  host_work.assign(std::max<size_t>(host_b, 8), 0);
  has_r = false;
}

QrStream::~QrStream() {
  if (params) cusolverDnDestroyParams(params);
}

void QrStream::fold(int64_t rows) {
  if (rows <= 0) return;
  require(rows <= bmax, FSTK_E_COMPUTE, "QrStream: block larger than its scratch");
  cusolverDnHandle_t h = solver_handle(device);
  cusolverDnSetStream(h, s);
  const int64_t m = n1 + rows;
  if (cusolverDnXgeqrf(h, params, m, n1, CUDA_R_64F, W.p, ldw, CUDA_R_64F, tau.p, CUDA_R_64F,
                       work.p, work_bytes, host_work.data(), host_work.size(), info.p) !=
      CUSOLVER_STATUS_SUCCESS)
    fail(FSTK_E_COMPUTE, "geqrf failed");
  dim3 g(static_cast<unsigned>(std::min<int64_t>(ceil_div(n1, 256), 64)), static_cast<unsigned>(n1));
  zero_lower_kernel<<<g, 256, 0, s>>>(W.p, ldw, n1);
  check_launch("zero_lower_kernel");
  count_launch();
  has_r = true;
}

void QrStream::fold_upper(const double* R2, int64_t ld2) {
  require(bmax >= n1, FSTK_E_COMPUTE, "QrStream: scratch too small to stack a factor");
  FSTK_CUDA(cudaMemcpy2DAsync(W.p + n1, ldw * 8, R2, ld2 * 8, static_cast<size_t>(n1) * 8, n1,
                              cudaMemcpyDeviceToDevice, s));
  fold(n1);
}

void QrStream::get_r(double* dst, int64_t ld) const {
  FSTK_CUDA(cudaMemcpy2DAsync(dst, ld * 8, W.p, ldw * 8, static_cast<size_t>(n1) * 8, n1,
                              cudaMemcpyDeviceToDevice, s));
}

// --------------------------------------------------- pivoted QR + solve ---
// Raug: the (n+1) x (n+1) upper R of [A b] (ld ldr).  diag_size = min(rows
// of A, n) for Eigen's threshold.  Writes x (n, device) and returns the rank.
int cpqr_solve(const double* Raug, int64_t ldr, int n, int64_t diag_size, double* x,
               bool* deficient, cudaStream_t s, int device) {
  const int ncols = n + 1;
  DevBuf<double> M(static_cast<size_t>(n) * ncols), vn1(n), vn2(n), tau(n), diag(n), y(n);
  DevBuf<int> perm(n);
  // Rows 0..n-1 of [R c] (the last row of Raug is the residual norm).
  FSTK_CUDA(cudaMemcpy2DAsync(M.p, static_cast<size_t>(n) * 8, Raug, ldr * 8,
                              static_cast<size_t>(n) * 8, ncols, cudaMemcpyDeviceToDevice, s));
  iota_kernel<<<static_cast<unsigned>(ceil_div(n, 256)), 256, 0, s>>>(perm.p, n);
  check_launch("iota_kernel");
  cpqr_colnorm_kernel<<<static_cast<unsigned>(ceil_div(n, 8)), 256, 0, s>>>(M.p, n, n, n, vn1.p,
                                                                             vn2.p);
  check_launch("cpqr_colnorm_kernel");
  const int steps = n;  // min(rows, cols) of the n x n factor
  for (int k = 0; k < steps; ++k) {
    cpqr_pivot_kernel<<<1, kPivThreads, 0, s>>>(M.p, n, n, n, k, vn1.p, vn2.p, perm.p, tau.p,
                                                diag.p);
    const int trailing = ncols - k - 1;
    if (trailing > 0) {
      const unsigned g = static_cast<unsigned>(std::min(trailing, 4 * 148));
      cpqr_apply_kernel<<<g, kApplyThreads, 0, s>>>(M.p, n, n, ncols, n, k, tau.p, vn1.p, vn2.p);
    }
  }
  check_launch("cpqr_kernels");
  count_launch(2 * static_cast<uint64_t>(steps));
  std::vector<double> hd(n);
  FSTK_CUDA(cudaMemcpyAsync(hd.data(), diag.p, static_cast<size_t>(n) * 8, cudaMemcpyDeviceToHost, s));
  FSTK_CUDA(cudaStreamSynchronize(s));
  double maxp = 0.0;
  for (double v : hd) maxp = std::max(maxp, std::fabs(v));
  const double thr = static_cast<double>(diag_size) * DBL_EPSILON * maxp;
  int rank = 0;
  for (double v : hd)
    if (std::fabs(v) > thr) ++rank;
  cublasHandle_t blas = blas_handle(device);
  cublasSetStream(blas, s);
  cusolverDnHandle_t sol = solver_handle(device);
  cusolverDnSetStream(sol, s);
  const double* cprime = M.p + static_cast<int64_t>(n) * n;  // Q2^T c (column n)
  *deficient = rank < n;
  if (rank == n) {
    FSTK_CUDA(cudaMemcpyAsync(y.p, cprime, static_cast<size_t>(n) * 8, cudaMemcpyDeviceToDevice, s));
    if (cublasDtrsv(blas, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, n, M.p, n,
                    y.p, 1) != CUBLAS_STATUS_SUCCESS)
      fail(FSTK_E_COMPUTE, "cublasDtrsv failed");
    count_launch();
  } else if (rank == 0) {
    FSTK_CUDA(cudaMemsetAsync(y.p, 0, static_cast<size_t>(n) * 8, s));
  } else {
    // Minimum-norm solution of [R11 R12] z = c_k (Eigen COD): QR of the
    // transpose, [R11 R12]^T = Q3 U, z = Q3 [U^{-T} c_k; 0].
    const int k = rank;
    DevBuf<double> T(static_cast<size_t>(n) * k), tau3(k);
    DevBuf<int> dinfo(1);
    dim3 g(static_cast<unsigned>(std::min<int64_t>(ceil_div(n, 256), 64)), static_cast<unsigned>(k));
    trapezoid_transpose_kernel<<<g, 256, 0, s>>>(M.p, n, n, k, T.p);
    check_launch("trapezoid_transpose_kernel");
    int lw = 0, lw2 = 0;
    if (cusolverDnDgeqrf_bufferSize(sol, n, k, T.p, n, &lw) != CUSOLVER_STATUS_SUCCESS)
      fail(FSTK_E_COMPUTE, "geqrf_bufferSize failed");
    FSTK_CUDA(cudaMemsetAsync(y.p, 0, static_cast<size_t>(n) * 8, s));
    FSTK_CUDA(cudaMemcpyAsync(y.p, cprime, static_cast<size_t>(k) * 8, cudaMemcpyDeviceToDevice, s));
    if (cusolverDnDormqr_bufferSize(sol, CUBLAS_SIDE_LEFT, CUBLAS_OP_N, n, 1, k, T.p, n, tau3.p,
                                    y.p, n, &lw2) != CUSOLVER_STATUS_SUCCESS)
      fail(FSTK_E_COMPUTE, "ormqr_bufferSize failed");
    DevBuf<double> wk(static_cast<size_t>(std::max(std::max(lw, lw2), 1)));
    if (cusolverDnDgeqrf(sol, n, k, T.p, n, tau3.p, wk.p, std::max(lw, 1), dinfo.p) !=
        CUSOLVER_STATUS_SUCCESS)
      fail(FSTK_E_COMPUTE, "geqrf failed");
    if (cublasDtrsv(blas, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_T, CUBLAS_DIAG_NON_UNIT, k, T.p, n, y.p,
                    1) != CUBLAS_STATUS_SUCCESS)
      fail(FSTK_E_COMPUTE, "cublasDtrsv failed");
    if (cusolverDnDormqr(sol, CUBLAS_SIDE_LEFT, CUBLAS_OP_N, n, 1, k, T.p, n, tau3.p, y.p, n, wk.p,
                         std::max(lw2, 1), dinfo.p) != CUSOLVER_STATUS_SUCCESS)
      fail(FSTK_E_COMPUTE, "ormqr failed");
    count_launch(3);
  }
  scatter_perm_kernel<<<static_cast<unsigned>(ceil_div(n, 256)), 256, 0, s>>>(y.p, perm.p, n, x);
  check_launch("scatter_perm_kernel");
  FSTK_CUDA(cudaStreamSynchronize(s));
  return rank;
}

// ------------------------------------------- Cholesky-side certificate ---
// X := (L L^T)^{-1} X for the lower factor L (n x n, ld n) and nrhs columns
// (ld ldx): 1024-wide diagonal TRSMs plus DGEMM panel updates streaming L.
void chol_solve_blocked_multi(cublasHandle_t h, const double* L, int n, double* X, int64_t ldx,
                              int nrhs) {
  constexpr int NB = 1024;
  const double one = 1.0, mone = -1.0;
  auto ok = [](cublasStatus_t st) {
    if (st != CUBLAS_STATUS_SUCCESS) fail(FSTK_E_COMPUTE, "blocked Cholesky solve failed");
  };
  const int lx = static_cast<int>(ldx);
  for (int i0 = 0; i0 < n; i0 += NB) {  // L Y = X
    const int nb = std::min(NB, n - i0);
    const double* Lii = L + static_cast<int64_t>(i0) * n + i0;
    ok(cublasDtrsm(h, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT,
                   nb, nrhs, &one, Lii, n, X + i0, lx));
    const int rest = n - i0 - nb;
    if (rest > 0)
      ok(cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, rest, nrhs, nb, &mone, Lii + nb, n, X + i0, lx,
                     &one, X + i0 + nb, lx));
  }
  for (int i1 = n; i1 > 0; i1 -= NB) {  // L^T Z = Y
    const int i0 = std::max(0, i1 - NB);
    const int nb = i1 - i0;
    const double* Lii = L + static_cast<int64_t>(i0) * n + i0;
    ok(cublasDtrsm(h, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, CUBLAS_DIAG_NON_UNIT,
                   nb, nrhs, &one, Lii, n, X + i0, lx));
    if (i0 > 0)
      ok(cublasDgemm(h, CUBLAS_OP_T, CUBLAS_OP_N, i0, nrhs, nb, &mone, L + i0, n, X + i0, lx, &one,
                     X, lx));
  }
  count_launch(4 * ((n + NB - 1) / NB));
}

// Column c of X (n x nv, ld n): norms[c] = ||X_c||, then X_c /= norms[c].
// One CTA per column; no host round trip, so a whole power iteration can be
// enqueued at once on a side stream.
__global__ void colnorm_scale_kernel(double* __restrict__ X, int n, double* __restrict__ norms) {
  __shared__ double red[32];
  double* x = X + static_cast<int64_t>(blockIdx.x) * n;
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s = fma(x[i], x[i], s);
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    s = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) red[0] = sqrt(s);
  }
  __syncthreads();
  const double nrm = red[0];
  const double inv = nrm > 0.0 ? 1.0 / nrm : 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) x[i] *= inv;
  if (threadIdx.x == 0) norms[blockIdx.x] = nrm;
}

// Block power iteration on (L L^T)^{-1} (4 seeded vectors, `iters` steps),
// enqueued on stream s without host synchronisation; result() returns an
// UPPER estimate of lambda_min(L L^T) (the largest growth factor is a lower
// bound of lambda_max((L L^T)^{-1})); callers apply a safety factor.
void LambdaMinEstimate::start(const double* L, int n_, int iters, cudaStream_t s_, int device_) {
  constexpr int NV = kVectors;
  n = n_;
  s = s_;
  device = device_;
  std::vector<double> h(static_cast<size_t>(n) * NV);
  uint64_t st = 0x9e3779b97f4a7c15ull;
  for (double& v : h) {  // splitmix64 -> uniform(-1, 1)
    st += 0x9e3779b97f4a7c15ull;
    uint64_t z = st;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    z ^= z >> 31;
    v = static_cast<double>(z >> 11) * (2.0 / 9007199254740992.0) - 1.0;
  }
  X.ensure(h.size());  // (kept across the factorisations of a session)
  norms.ensure(NV);
  FSTK_CUDA(cudaMemcpyAsync(X.p, h.data(), h.size() * 8, cudaMemcpyHostToDevice, s));
  FSTK_CUDA(cudaStreamSynchronize(s));  // h is a host temporary
  cublasHandle_t blas = blas_side_handle(device);
  cublasSetStream(blas, s);
  for (int it = 0; it < iters; ++it) {
    colnorm_scale_kernel<<<NV, 256, 0, s>>>(X.p, n, norms.p);
    check_launch("colnorm_scale_kernel");
    chol_solve_blocked_multi(blas, L, n, X.p, n, NV);
  }
  colnorm_scale_kernel<<<NV, 256, 0, s>>>(X.p, n, norms.p);  // growth of the last step
  check_launch("colnorm_scale_kernel");
  started = true;
}

// ---- side worker: one detached host thread running jobs in order ----
namespace {
struct SideWorker {
  std::mutex mu;
  std::condition_variable cv;
  std::deque<std::packaged_task<void()>> q;
  SideWorker() {
    std::thread([this] {
      for (;;) {
        std::packaged_task<void()> job;
        {
          std::unique_lock<std::mutex> lk(mu);
          cv.wait(lk, [this] { return !q.empty(); });
          job = std::move(q.front());
          q.pop_front();
        }
        job();  // exceptions land in the task's future
      }
    }).detach();
  }
};
}  // namespace

std::shared_future<void> side_worker_submit(std::function<void()> job) {
  static SideWorker* w = new SideWorker();  // leaked: no teardown-order hazards at exit
  std::packaged_task<void()> task(std::move(job));
  std::shared_future<void> f = task.get_future().share();
  {
    std::lock_guard<std::mutex> lk(w->mu);
    w->q.push_back(std::move(task));
  }
  w->cv.notify_one();
  return f;
}

void LambdaMinEstimate::start_async(const double* L, int n_, int iters, cudaStream_t s_, int device_) {
  wait_enqueued();
  s = s_;
  device = device_;
  enqueued = side_worker_submit([this, L, n_, iters, s_, device_] {
    FSTK_CUDA(cudaSetDevice(device_));
    start(L, n_, iters, s_, device_);
  });
}

void LambdaMinEstimate::wait_enqueued() {
  if (!enqueued.valid()) return;
  std::shared_future<void> f = enqueued;
  enqueued = std::shared_future<void>();
  f.get();
}

LambdaMinEstimate::~LambdaMinEstimate() {
  // Only the enqueue job is waited for here.  The stream may already be gone
  // (a session destroys its side stream, after synchronising it, before its
  // members): releasing X and norms synchronises the device like cudaFree.
  try {
    wait_enqueued();
  } catch (...) {
  }
}

double LambdaMinEstimate::result() {
  wait_enqueued();
  if (!started) return 0.0;
  double hn[kVectors];
  FSTK_CUDA(cudaMemcpyAsync(hn, norms.p, sizeof(hn), cudaMemcpyDeviceToHost, s));
  FSTK_CUDA(cudaStreamSynchronize(s));
  double growth = 0.0;
  for (double g : hn) growth = std::max(growth, g);
  return growth > 0 ? 1.0 / growth : 0.0;
}

double chol_lambda_min_estimate(const double* L, int n, int iters, cudaStream_t s, int device) {
  LambdaMinEstimate e;
  e.start(L, n, iters, s, device);
  return e.result();
}

}  // namespace fstk_gpu

// ------------------------------------------------------------- C-ABI ---
extern "C" {

// solve_system (randls.cpp:112-123) for a host matrix: streaming TSQR of
// [A b] in row blocks, pivoted QR of R, Eigen's rank rule, QR or COD solve.
int32_t fstk_gpu_solve_system(const double* a, int64_t m, int64_t n, const double* b, double* x,
                              int32_t* rank, int32_t* rank_deficient, fstk_gpu_error* err) {
  using namespace fstk_gpu;
  return guarded(err, [&] {
    require(a && b && x, FSTK_E_PARAMETER, "null argument");
    require(m >= 1 && n >= 1 && n < (int64_t(1) << 16), FSTK_E_SHAPE,
            "solve_system: need m >= 1 and 1 <= n < 65536");
    int device = 0;
    FSTK_CUDA(cudaGetDevice(&device));
    cudaStream_t s;
    FSTK_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    struct SG {
      cudaStream_t s;
      ~SG() { cudaStreamDestroy(s); }
    } sg{s};
    const int nn = static_cast<int>(n), n1 = nn + 1;
    // Row blocks of up to ~1 GB of scratch, at least n1 rows.
    const int64_t bmax = std::min<int64_t>(m, std::max<int64_t>(n1, (int64_t(1) << 27) / n1));
    QrStream qs;
    qs.init(n1, bmax, s, device);
    std::vector<double> blk(static_cast<size_t>(bmax) * n1);
    for (int64_t r0 = 0; r0 < m; r0 += bmax) {
      const int64_t rows = std::min(bmax, m - r0);
      for (int64_t j = 0; j < n; ++j)
        std::memcpy(&blk[static_cast<size_t>(j) * rows], a + j * m + r0, rows * 8);
      std::memcpy(&blk[static_cast<size_t>(n) * rows], b + r0, rows * 8);
      FSTK_CUDA(cudaMemcpy2DAsync(qs.block(), qs.ldw * 8, blk.data(), rows * 8, rows * 8, n1,
                                  cudaMemcpyHostToDevice, s));
      qs.fold(rows);
      FSTK_CUDA(cudaStreamSynchronize(s));
    }
    DevBuf<double> xd(n);
    bool def = false;
    const int rk = cpqr_solve(qs.W.p, qs.ldw, nn, std::min(m, n), xd.p, &def, s, device);
    FSTK_CUDA(cudaMemcpyAsync(x, xd.p, n * 8, cudaMemcpyDeviceToHost, s));
    FSTK_CUDA(cudaStreamSynchronize(s));
    if (rank) *rank = rk;
    if (rank_deficient) *rank_deficient = def ? 1 : 0;
  });
}

// top := R of [top; other] for two (n1 x n1, ld n1) upper-triangular device
// factors: the stacking step of a sharded TSQR.
int32_t fstk_gpu_qr_stack(double* top, const double* other, int64_t n1, int32_t device,
                          void* stream, fstk_gpu_error* err) {
  using namespace fstk_gpu;
  return guarded(err, [&] {
    require(top && other, FSTK_E_PARAMETER, "null argument");
    require(n1 >= 1 && n1 <= 65536, FSTK_E_SHAPE, "qr_stack: bad size");
    DeviceGuard dg(device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    QrStream qs;
    qs.init(static_cast<int>(n1), n1, s, device);
    qs.fold_upper(top, n1);
    qs.fold_upper(other, n1);
    qs.get_r(top, n1);
    FSTK_CUDA(cudaStreamSynchronize(s));
  });
}

}  // extern "C"
