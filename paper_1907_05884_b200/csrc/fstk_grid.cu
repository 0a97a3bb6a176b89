// fstk B200 library — tensor-product grid evaluation.
//
// reconstruct --grid (proj/src/pipeline.cpp:531-569) and slice (:571-696)
// evaluate every node of a Cartesian grid through evaluate_batch.  On the
// grid the model is separable: Y = G x_0 U_0 x_1 U_1 ... with U_k the mode
// values on mode k's grid line (I_k x r_k, mode-value kernel), so the whole
// grid is a chain of d mode products — one GEMM for mode 0 and strided-batched
// GEMMs for the others (cuBLAS DGEMM, plain library GEMMs).  At 256^3 with
// ranks 32^3 that is ~1.1 GFLOP instead of the 1.2 TFLOP of point-wise
// evaluation, and the output write (8 B per node) bounds it.
#include <cublas_v2.h>

#include <climits>
#include <vector>

#include "fstk_internal.h"

using namespace fstk_gpu;

extern "C" {

int32_t fstk_gpu_evaluate_grid(const fstk_gpu_model* m, const double* coords, const int64_t* sizes,
                               int32_t d, double* out, fstk_gpu_error* err) {
  return guarded(err, [&] {
    require(m && coords && sizes && out, FSTK_E_PARAMETER, "null argument");
    require(d == m->d, FSTK_E_PARAMETER, "grid needs one size per mode");
    int64_t total = 1, ncoord = 0;
    for (int k = 0; k < d; ++k) {
      require(sizes[k] >= 1, FSTK_E_PARAMETER, "grid sizes must be >= 1");
      total *= sizes[k];
      ncoord += sizes[k];
    }
    std::lock_guard<std::mutex> lk(m->mu);
    DeviceGuard dg(m->device);
    cudaStream_t s = m->chunk[0].stream;
    cublasHandle_t h = blas_handle(m->device);
    cublasSetStream(h, s);
    DevBuf<double> dc(ncoord);
    FSTK_CUDA(cudaMemcpyAsync(dc.p, coords, ncoord * 8, cudaMemcpyHostToDevice, s));
    // Mode values on every grid line: U_k is I_k x r_k (ld = I_k).
    std::vector<int64_t> uoff(d);
    int64_t utot = 0;
    for (int k = 0; k < d; ++k) {
      uoff[k] = utot;
      utot += sizes[k] * m->ranks[k];
    }
    DevBuf<double> U(utot);
    DevBuf<unsigned long long> derr(d);
    FSTK_CUDA(cudaMemsetAsync(derr.p, 0xff, d * 8, s));
    {
      int64_t co = 0;
      for (int k = 0; k < d; ++k) {
        launch_mode_table_one(m, k, dc.p + co, sizes[k], U.p + uoff[k], sizes[k], false,
                              derr.p + k, s);
        co += sizes[k];
      }
    }
    std::vector<unsigned long long> bad(d);
    FSTK_CUDA(cudaMemcpyAsync(bad.data(), derr.p, d * 8, cudaMemcpyDeviceToHost, s));
    FSTK_CUDA(cudaStreamSynchronize(s));
    {
      int64_t co = 0;
      for (int k = 0; k < d; ++k) {
        if (bad[k] != ULLONG_MAX) {
          Error e{FSTK_E_DOMAIN, "point outside basis domain"};
          e.mode = k;
          e.index = static_cast<int64_t>(bad[k]);  // node index along mode k
          e.value = coords[co + static_cast<int64_t>(bad[k])];
          throw e;
        }
        co += sizes[k];
      }
    }
    // T_0 = core (r_0 x r_1 x ...); after step k: (I_0..I_k, r_{k+1}..), mode-0 fastest.
    int64_t maxsz = m->R;
    {
      int64_t cur = m->R;
      for (int k = 0; k < d; ++k) {
        cur = cur / m->ranks[k] * sizes[k];
        maxsz = std::max(maxsz, cur);
      }
    }
    DevBuf<double> A(maxsz), B(maxsz);
    FSTK_CUDA(cudaMemcpyAsync(A.p, m->d_core.p, m->R * 8, cudaMemcpyDeviceToDevice, s));
    const double one = 1.0, zero = 0.0;
    int64_t P = 1, rest = m->R;
    for (int k = 0; k < d; ++k) {
      const int64_t rk = m->ranks[k], Ik = sizes[k];
      rest /= rk;
      if (P == 1) {
        // (I_k x rest) = U_k (I_k x r_k) * T (r_k x rest)
        if (cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, static_cast<int>(Ik), static_cast<int>(rest),
                        static_cast<int>(rk), &one, U.p + uoff[k], static_cast<int>(Ik), A.p,
                        static_cast<int>(rk), &zero, B.p, static_cast<int>(Ik)) != CUBLAS_STATUS_SUCCESS)
          fail(FSTK_E_COMPUTE, "cublasDgemm failed");
      } else {
        // per trailing index b: (P x I_k) = T_b (P x r_k) * U_k^T
        if (cublasDgemmStridedBatched(h, CUBLAS_OP_N, CUBLAS_OP_T, static_cast<int>(P),
                                      static_cast<int>(Ik), static_cast<int>(rk), &one, A.p,
                                      static_cast<int>(P), P * rk, U.p + uoff[k],
                                      static_cast<int>(Ik), 0, &zero, B.p, static_cast<int>(P),
                                      P * Ik, static_cast<int>(rest)) != CUBLAS_STATUS_SUCCESS)
          fail(FSTK_E_COMPUTE, "cublasDgemmStridedBatched failed");
      }
      count_launch();
      std::swap(A, B);  // whole buffers (pointer, count and block size) trade places
      P *= Ik;
    }
    FSTK_CUDA(cudaMemcpyAsync(out, A.p, total * 8, cudaMemcpyDeviceToHost, s));
    FSTK_CUDA(cudaStreamSynchronize(s));
  });
}

// reconstruct --grid: uniform nodes lo + (hi - lo) i / (I - 1) over each
// mode's domain (StructuredGrid::node, ingest.cpp:57-61; sizes >= 2, :70-80).
int32_t fstk_gpu_reconstruct_grid(const fstk_gpu_model* m, const int64_t* sizes, int32_t d,
                                  double* out, fstk_gpu_error* err) {
  std::vector<double> coords;
  int32_t rc = guarded(err, [&] {
    require(m && sizes && out, FSTK_E_PARAMETER, "null argument");
    require(d == m->d, FSTK_E_PARAMETER, "--grid needs one size per mode");
    for (int k = 0; k < d; ++k) {
      require(sizes[k] >= 2, FSTK_E_PARAMETER, "grid sizes must be >= 2");
      const double lo = m->modes[k].lo, hi = m->modes[k].hi;
      for (int64_t i = 0; i < sizes[k]; ++i)
        coords.push_back(lo + (hi - lo) * static_cast<double>(i) /
                                  static_cast<double>(sizes[k] - 1));
    }
  });
  if (rc) return rc;
  return fstk_gpu_evaluate_grid(m, coords.data(), sizes, d, out, err);
}

}  // extern "C"

// FPTC ingest: point-major (Q x d row-major, the file payload)
// -> SoA (column-major Q x d) on the device, coalesced through shared memory.
namespace fstk_gpu {
__global__ void point_major_to_soa_kernel(const double* __restrict__ in, int64_t q, int d,
                                          double* __restrict__ out) {
  __shared__ double tile[256 * 8];
  const int64_t base = static_cast<int64_t>(blockIdx.x) * 256;
  const int64_t nrow = (q - base) < 256 ? (q - base) : 256;
  for (int e = threadIdx.x; e < nrow * d; e += blockDim.x) tile[e] = in[base * d + e];
  __syncthreads();
  for (int e = threadIdx.x; e < nrow * d; e += blockDim.x) {
    const int k = e / static_cast<int>(nrow), i = e % static_cast<int>(nrow);
    out[k * q + base + i] = tile[i * d + k];
  }
}
}  // namespace fstk_gpu

extern "C" int32_t fstk_gpu_point_major_to_soa(const double* in, int64_t q, int32_t d, double* out,
                                               void* stream, fstk_gpu_error* err) {
  return guarded(err, [&] {
    require(in && out, FSTK_E_PARAMETER, "null argument");
    require(d >= 1 && d <= kMaxOrder, FSTK_E_SHAPE, "point cloud dimension must be in [1, 8]");
    if (q <= 0) return;
    point_major_to_soa_kernel<<<static_cast<unsigned>(ceil_div(q, 256)), 256, 0,
                                static_cast<cudaStream_t>(stream)>>>(in, q, d, out);
    check_launch("point_major_to_soa_kernel");
  });
}
