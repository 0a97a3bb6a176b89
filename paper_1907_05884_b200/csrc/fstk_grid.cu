// fstk B200 library — tensor-product grid evaluation.
//
// reconstruct --grid (proj/src/pipeline.cpp:531-569) and slice (:571-696)
// evaluate every node of a Cartesian grid through evaluate_batch.  On the
// grid the model is separable: Y = G x_0 U_0 x_1 U_1 ... with U_k the mode
// values on mode k's grid line (I_k x r_k, mode-value kernel), so the whole
// grid is a chain of d mode products (the reference's dense mode product,
// tensor.cpp:104-136) -- each one a batched GEMM with the tiny inner
// dimension r_k, run by mode_product_kernel on the fp64 tensor cores
// (DMMA m8n8k4, the contraction kernel's fragment layout).  At 256^3 with
// ranks 32^3 that is ~1.2 GFLOP instead of the 1.2 TFLOP of point-wise
// evaluation; the output write (8 B per node) bounds it.
#include <climits>
#include <vector>

#include "fstk_common.cuh"
#include "fstk_internal.h"

using namespace fstk_gpu;

namespace fstk_gpu {
namespace {

constexpr int kMpTile = 64;   // output tile: 64 rows (p) x 64 columns (i)
constexpr int kMpKC = 32;     // inner-dimension chunk staged at once

// One mode product in general strided form:
//   B[p sp + i si + b sb] = sum_{j < r} A[p ap + j aj + b ab] U[i + I j]
// for p < P, i < I, b < rest.  CTA: a 64 x 64 (p, i) tile of one b; its A
// and U slabs are staged in shared memory 32 j at a time (zero padded to a
// multiple of 4) and 8 warps each run 8 DMMA n-tiles per 4-wide j step.
__global__ void __launch_bounds__(256) mode_product_kernel(const double* __restrict__ A, const double* __restrict__ U,
                                                           double* __restrict__ B, int64_t P, int r, int64_t I,
                                                           int64_t rest, int64_t ap, int64_t aj, int64_t ab,
                                                           int64_t sp, int64_t si, int64_t sb) {
  __shared__ double As[kMpKC][kMpTile + 1];
  __shared__ double Us[kMpKC][kMpTile + 1];
  const int64_t p0 = static_cast<int64_t>(blockIdx.x) * kMpTile;
  const int64_t i0 = static_cast<int64_t>(blockIdx.y) * kMpTile;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  for (int64_t b = blockIdx.z; b < rest; b += gridDim.z) {
    double c[8][2];
#pragma unroll
    for (int n = 0; n < 8; ++n) c[n][0] = c[n][1] = 0.0;
    for (int j0 = 0; j0 < r; j0 += kMpKC) {
      const int jn = min(kMpKC, r - j0), j4 = (jn + 3) & ~3;
      __syncthreads();
      for (int e = threadIdx.x; e < j4 * kMpTile; e += blockDim.x) {
        const int j = e / kMpTile, q = e % kMpTile;
        const int64_t p = p0 + q, i = i0 + q;
        As[j][q] = (j < jn && p < P) ? A[p * ap + (j0 + j) * aj + b * ab] : 0.0;
        Us[j][q] = (j < jn && i < I) ? U[i + I * (j0 + j)] : 0.0;
      }
      __syncthreads();
      for (int kk = 0; kk < j4; kk += 4) {
        const double a = As[kk + t][warp * 8 + g];
#pragma unroll
        for (int n = 0; n < 8; ++n) dmma_8x8x4(c[n][0], c[n][1], a, Us[kk + t][n * 8 + g]);
      }
    }
    const int64_t p = p0 + warp * 8 + g;
    if (p < P) {
#pragma unroll
      for (int n = 0; n < 8; ++n) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int64_t i = i0 + n * 8 + 2 * t + h;
          if (i < I) B[p * sp + i * si + b * sb] = c[n][h];
        }
      }
    }
  }
}

void mode_product(const double* A, const double* U, double* B, int64_t P, int r, int64_t I, int64_t rest,
                  int64_t ap, int64_t aj, int64_t ab, int64_t sp, int64_t si, int64_t sb, cudaStream_t s) {
  require(r >= 1, FSTK_E_COMPUTE, "internal: grid mode product rank");
  dim3 grid(static_cast<unsigned>(ceil_div(P, kMpTile)), static_cast<unsigned>(ceil_div(I, kMpTile)),
            static_cast<unsigned>(std::min<int64_t>(rest, 65535)));
  require(ceil_div(P, kMpTile) < (int64_t(1) << 31) && ceil_div(I, kMpTile) <= 65535, FSTK_E_SHAPE,
          "grid too large");
  mode_product_kernel<<<grid, 256, 0, s>>>(A, U, B, P, r, I, rest, ap, aj, ab, sp, si, sb);
  check_launch("mode_product_kernel");
}

}  // namespace
}  // namespace fstk_gpu

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
    int64_t P = 1, rest = m->R;
    for (int k = 0; k < d; ++k) {
      const int64_t rk = m->ranks[k], Ik = sizes[k];
      rest /= rk;
      if (P == 1) {
        // (I_k x rest) = U_k (I_k x r_k) * T (r_k x rest): rows = the rest
        // index (larger), columns = grid nodes.
        mode_product(A.p, U.p + uoff[k], B.p, rest, static_cast<int>(rk), Ik, 1, rk, 1, 0, Ik, 1, 0, s);
      } else {
        // per trailing index b: (P x I_k) = T_b (P x r_k) * U_k^T
        mode_product(A.p, U.p + uoff[k], B.p, P, static_cast<int>(rk), Ik, rest, 1, P, P * rk, 1, P, P * Ik, s);
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
