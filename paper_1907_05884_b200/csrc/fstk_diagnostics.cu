// fstk B200 library — refit diagnostics.
//
// self_convergence (proj/src/randls.cpp:385-413): sketched solves over a
//   nondecreasing list of sample counts with one seed (nested sampled rows),
//   reporting ||a_{i+1} - a_i|| / ||a_{i+1}||.  Each solve runs the GPU refit
//   stages (sketch -> A^T A -> Cholesky + refinement).
// leverage_scores (randls.cpp:227-233): squared row norms of the thin left
//   singular vectors of W restricted to its numerical rank (cuSOLVER gesvd;
//   rank rule of Eigen's SVDBase: sigma_i > min(m,n) eps sigma_max).
#include <cublas_v2.h>
#include <cusolverDn.h>

#include <cmath>
#include <vector>

#include "fstk_internal.h"

using namespace fstk_gpu;

extern "C" {

int32_t fstk_gpu_self_convergence(const fstk_gpu_model* m, const double* points,
                                  const double* values, int64_t q, int32_t d,
                                  const fstk_sketch_cfg* cfg, const uint64_t* s_values,
                                  int32_t n_s, double* deltas, fstk_gpu_error* err) {
  return guarded(err, [&] {
    require(m && points && values && cfg && s_values && deltas, FSTK_E_PARAMETER, "null argument");
    require(n_s >= 2, FSTK_E_PARAMETER, "need at least two sample counts");
    for (int i = 0; i < n_s; ++i) {
      require(s_values[i] > static_cast<uint64_t>(m->R), FSTK_E_PARAMETER,
              "sample rows must exceed the core size");
      require(i == 0 || s_values[i] >= s_values[i - 1], FSTK_E_PARAMETER,
              "sample counts must be nondecreasing");
    }
    require(static_cast<uint64_t>(q) >= s_values[n_s - 1], FSTK_E_PARAMETER,
            "dataset smaller than the requested sketch");
    DeviceGuard dg(m->device);
    const int64_t R = m->R;
    std::vector<std::vector<double>> alphas;
    DevBuf<double> gram(static_cast<size_t>(R) * R), rhs(R);
    for (int i = 0; i < n_s; ++i) {
      fstk_sketch_cfg c = *cfg;
      c.sample_rows = s_values[i];
      fstk_gpu_refit* rf = nullptr;
      fstk_reestimate_info info{};
      int32_t rc = fstk_gpu_refit_begin(m, points, values, q, d, &c, 0, 1, &rf, &info, err);
      if (rc) throw Error{rc, err ? err->message : "refit failed"};
      std::vector<double> a(R);
      rc = fstk_gpu_refit_normal_equations(rf, gram.p, rhs.p, &info, err);
      if (!rc) rc = fstk_gpu_refit_solve(rf, gram.p, rhs.p, a.data(), &info, err);
      fstk_gpu_refit_end(rf);
      if (rc) throw Error{rc, err ? err->message : "refit failed"};
      alphas.push_back(std::move(a));
    }
    for (int i = 0; i + 1 < n_s; ++i) {
      double dn = 0.0, nn = 0.0;
      for (int64_t j = 0; j < R; ++j) {
        const double dl = alphas[i + 1][j] - alphas[i][j];
        dn += dl * dl;
        nn += alphas[i + 1][j] * alphas[i + 1][j];
      }
      const double denom = std::sqrt(nn), delta = std::sqrt(dn);
      deltas[i] = denom > 0.0 ? delta / denom : delta;
    }
  });
}

int32_t fstk_gpu_leverage_scores(const double* w, int64_t q, int64_t r, double* scores,
                                 int32_t* rank_out, fstk_gpu_error* err) {
  return guarded(err, [&] {
    require(w && scores, FSTK_E_PARAMETER, "null argument");
    require(q >= r, FSTK_E_PARAMETER, "leverage scores need at least as many rows as columns");
    require(r >= 1, FSTK_E_PARAMETER, "empty matrix");
    int dev = 0;
    FSTK_CUDA(cudaGetDevice(&dev));
    cusolverDnHandle_t h = solver_handle(dev);
    cudaStream_t s;
    FSTK_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    struct SG {
      cudaStream_t s;
      ~SG() { cudaStreamDestroy(s); }
    } sg{s};
    cusolverDnSetStream(h, s);
    const int M = static_cast<int>(q), N = static_cast<int>(r);
    DevBuf<double> A(static_cast<size_t>(q) * r), S(r), U(static_cast<size_t>(q) * r), VT(1);
    DevBuf<int> info(1);
    FSTK_CUDA(cudaMemcpyAsync(A.p, w, static_cast<size_t>(q) * r * 8, cudaMemcpyHostToDevice, s));
    int lwork = 0;
    if (cusolverDnDgesvd_bufferSize(h, M, N, &lwork) != CUSOLVER_STATUS_SUCCESS)
      fail(FSTK_E_COMPUTE, "gesvd_bufferSize failed");
    DevBuf<double> work(std::max(lwork, 1)), rwork(std::max(N, 1));
    if (cusolverDnDgesvd(h, 'S', 'N', M, N, A.p, M, S.p, U.p, M, VT.p, 1, work.p, lwork, rwork.p,
                         info.p) != CUSOLVER_STATUS_SUCCESS)
      fail(FSTK_E_COMPUTE, "gesvd failed");
    count_launch();
    std::vector<double> sv(r), u(static_cast<size_t>(q) * r);
    FSTK_CUDA(cudaMemcpyAsync(sv.data(), S.p, r * 8, cudaMemcpyDeviceToHost, s));
    FSTK_CUDA(cudaMemcpyAsync(u.data(), U.p, u.size() * 8, cudaMemcpyDeviceToHost, s));
    FSTK_CUDA(cudaStreamSynchronize(s));
    const double thr = static_cast<double>(std::min(q, r)) * 2.220446049250313e-16 * sv[0];
    int rank = 0;
    for (int64_t j = 0; j < r; ++j)
      if (sv[j] > thr) ++rank;
    for (int64_t i = 0; i < q; ++i) {
      double acc = 0.0;
      for (int j = 0; j < rank; ++j) acc += u[static_cast<size_t>(j) * q + i] * u[static_cast<size_t>(j) * q + i];
      scores[i] = acc;
    }
    if (rank_out) *rank_out = rank;
  });
}

}  // extern "C"
