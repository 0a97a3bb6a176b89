// fstk B200 library — scattered-to-grid IDW interpolation.
//
// Replaces interpolate_to_grid (proj/src/ingest.cpp:265-383), the upstream
// step that turns a point cloud into the structured grid ST-HOSVD factors:
//  * the uniform-binning spatial index (build_index, ingest.cpp:140-190) is
//    sized on the host exactly as the reference sizes it (~4 points per bin,
//    capped by the grid cells and 2^22 bins, box padded to the cloud), and
//    built on the GPU: per-point bin ids, a histogram, an exclusive scan and
//    a scatter that leaves every bin's points contiguous (SoA coordinates);
//  * one thread per grid node (mode-0 fastest, so a warp walks neighbouring
//    bins) scans Chebyshev rings of bins around the node's bin (for_ring,
//    :217-260: faces per axis, lower axes strict interior) with the
//    reference's stop rule (:337-340), keeping the k smallest (d2, id) pairs
//    under the reference's lexicographic order (NeighborHeap, :194-212) in a
//    register insertion array -- the retained set is insertion-order
//    invariant, so the neighbour sets equal the reference's;
//  * exact hits within 1e-24 cell-diagonal^2 take the sample's value, else
//    inverse-distance weights 1/d2 (power 2) or d2^(-p/2) (:343-357), summed
//    in ascending (d2, id) order (the reference sums in heap order: values
//    agree to rounding);
//  * the report (box coverage, max nearest distance, extrapolated fraction)
//    is reduced on the device.
// Distances are sums of separately rounded squares (no FMA), node
// coordinates lo + (hi - lo) i / (n - 1) and bin indices floor((x - lo) / w)
// are formed in the reference's operation order.
#include <cub/cub.cuh>

#include <math_constants.h>

#include <cmath>
#include <cstring>
#include <limits>
#include <vector>

#include "fstk_common.cuh"
#include "fstk_internal.h"

namespace fstk_gpu {
namespace {

constexpr int kIdwMaxK = 64;

struct IdwGrid {
  int d;
  int k;                // neighbours
  int pow2;             // power == 2
  double power;
  int64_t n_nodes;
  int64_t q;
  int64_t sizes[kMaxOrder];
  double glo[kMaxOrder], ghi[kMaxOrder];
  int64_t nbins[kMaxOrder];
  double lo[kMaxOrder], width[kMaxOrder];
  double min_width, bin_diag, hit_tol2;
};

// Order-preserving map of doubles to unsigned integers (for atomic min/max).
__device__ __forceinline__ unsigned long long ord(double x) {
  const unsigned long long u = static_cast<unsigned long long>(__double_as_longlong(x));
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__host__ __device__ inline double unord(unsigned long long u) {
  const unsigned long long v = (u >> 63) ? (u & 0x7fffffffffffffffull) : ~u;
  double x;
  memcpy(&x, &v, sizeof(x));
  return x;
}

// Per-mode min / max of the coordinates and a non-finite count (PointCloud::
// from_data / validate, ingest.cpp:19-49), grid-stride.
__global__ void box_kernel(const double* __restrict__ pts, int64_t q, int d,
                           unsigned long long* __restrict__ mn, unsigned long long* __restrict__ mx,
                           unsigned long long* __restrict__ bad) {
  for (int k = 0; k < d; ++k) {
    unsigned long long lmn = ~0ull, lmx = 0ull, lbad = 0ull;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < q;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
      const double x = pts[i + k * q];
      if (!isfinite(x)) {
        ++lbad;
        continue;
      }
      const unsigned long long o = ord(x);
      lmn = o < lmn ? o : lmn;
      lmx = o > lmx ? o : lmx;
    }
    for (int s = 16; s > 0; s >>= 1) {
      lmn = min(lmn, __shfl_xor_sync(0xffffffffu, lmn, s));
      lmx = max(lmx, __shfl_xor_sync(0xffffffffu, lmx, s));
      lbad += __shfl_xor_sync(0xffffffffu, lbad, s);
    }
    if ((threadIdx.x & 31) == 0) {
      atomicMin(mn + k, lmn);
      atomicMax(mx + k, lmx);
      if (lbad) atomicAdd(bad, lbad);
    }
  }
}

__global__ void nonfinite_kernel(const double* __restrict__ v, int64_t q, unsigned long long* bad) {
  unsigned long long lbad = 0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < q;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    if (!isfinite(v[i])) ++lbad;
  for (int s = 16; s > 0; s >>= 1) lbad += __shfl_xor_sync(0xffffffffu, lbad, s);
  if ((threadIdx.x & 31) == 0 && lbad) atomicAdd(bad, lbad);
}

// SpatialIndex::bin_of (ingest.cpp:129-132).
__device__ __forceinline__ int64_t bin_of(const IdwGrid& g, int k, double x) {
  const int64_t b = static_cast<int64_t>(floor(__ddiv_rn(__dsub_rn(x, g.lo[k]), g.width[k])));
  return min(g.nbins[k] - 1, max(int64_t(0), b));
}

__global__ void bin_kernel(const IdwGrid g, const double* __restrict__ pts, uint32_t* __restrict__ bin,
                           uint32_t* __restrict__ counts) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= g.q) return;
  int64_t f = 0;
#pragma unroll
  for (int k = kMaxOrder - 1; k >= 0; --k)
    if (k < g.d) f = f * g.nbins[k] + bin_of(g, k, pts[i + k * g.q]);
  bin[i] = static_cast<uint32_t>(f);
  atomicAdd(counts + f, 1u);
}

// Bins' points contiguous (order within a bin is irrelevant: the retained
// set is insertion-order invariant).
__global__ void scatter_kernel(const IdwGrid g, const double* __restrict__ pts, const uint32_t* __restrict__ bin,
                               uint32_t* __restrict__ cursor, double* __restrict__ ps, uint32_t* __restrict__ ids) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= g.q) return;
  const uint32_t pos = atomicAdd(cursor + bin[i], 1u);
#pragma unroll
  for (int k = 0; k < kMaxOrder; ++k)
    if (k < g.d) ps[pos + k * g.q] = pts[i + k * g.q];
  ids[pos] = static_cast<uint32_t>(i);
}

__device__ __forceinline__ bool lessp(double a, uint32_t ia, double b, uint32_t ib) {
  return a < b || (a == b && ia < ib);
}

template <int KT>
struct Best {
  double D[KT];
  uint32_t I[KT];
  int64_t pushed = 0;
  __device__ Best() {
#pragma unroll
    for (int j = 0; j < KT; ++j) {
      D[j] = CUDART_INF;
      I[j] = 0xFFFFFFFFu;
    }
  }
  // The KT smallest (d2, id) pairs seen so far, ascending.
  __device__ __forceinline__ void push(double d2, uint32_t id) {
    ++pushed;
    if (!lessp(d2, id, D[KT - 1], I[KT - 1])) return;
    D[KT - 1] = d2;
    I[KT - 1] = id;
#pragma unroll
    for (int j = KT - 1; j > 0; --j) {
      if (lessp(D[j], I[j], D[j - 1], I[j - 1])) {
        const double td = D[j];
        D[j] = D[j - 1];
        D[j - 1] = td;
        const uint32_t ti = I[j];
        I[j] = I[j - 1];
        I[j - 1] = ti;
      }
    }
  }
  __device__ __forceinline__ double kth(int k) const {  // D[k - 1]
    double w = D[0];
#pragma unroll
    for (int j = 1; j < KT; ++j)
      if (j == k - 1) w = D[j];
    return w;
  }
};

template <int D, int KT>
__device__ __forceinline__ void scan_bin(const IdwGrid& g, const int (&c)[D], const double (&y)[D],
                                         const uint32_t* __restrict__ offsets, const double* __restrict__ ps,
                                         const uint32_t* __restrict__ ids, Best<KT>& best) {
  int64_t f = 0;
#pragma unroll
  for (int k = D - 1; k >= 0; --k) f = f * g.nbins[k] + c[k];
  const uint32_t e = __ldg(offsets + f + 1);
  for (uint32_t ii = __ldg(offsets + f); ii < e; ++ii) {
    double d2 = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const double diff = __dsub_rn(__ldg(ps + ii + k * g.q), y[k]);
      d2 = __dadd_rn(d2, __dmul_rn(diff, diff));
    }
    best.push(d2, __ldg(ids + ii));
  }
}

template <int D, int KT>
__global__ void __launch_bounds__(128) idw_node_kernel(const IdwGrid g, const uint32_t* __restrict__ offsets,
                                                       const double* __restrict__ ps,
                                                       const uint32_t* __restrict__ ids,
                                                       const double* __restrict__ vals, double* __restrict__ out,
                                                       unsigned long long* __restrict__ stats,
                                                       uint32_t* __restrict__ nbr) {
  const int64_t node = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (node >= g.n_nodes) return;
  double y[D];
  int c[D];
  int64_t rem = node;
  int max_rho = 0;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    const int64_t m = rem % g.sizes[k];
    rem /= g.sizes[k];
    // StructuredGrid::node (ingest.cpp:57-61): lo + (hi - lo) * i / (n - 1).
    y[k] = __dadd_rn(g.glo[k], __ddiv_rn(__dmul_rn(__dsub_rn(g.ghi[k], g.glo[k]), static_cast<double>(m)),
                                         static_cast<double>(g.sizes[k] - 1)));
    c[k] = static_cast<int>(bin_of(g, k, y[k]));
    max_rho = max(max_rho, max(c[k], static_cast<int>(g.nbins[k]) - 1 - c[k]));
  }
  Best<KT> best;
  scan_bin<D, KT>(g, c, y, offsets, ps, ids, best);
  for (int rho = 1;; ++rho) {
    // Stop rule after ring rho - 1 (ingest.cpp:337-340).
    const double safe = static_cast<double>(rho - 1) * g.min_width;
    if (best.pushed >= g.k && best.kth(g.k) <= safe * safe) break;
    if (rho - 1 >= max_rho) break;
    // Ring rho: per axis and side, the face with lower axes restricted to
    // the strict interior (for_ring, ingest.cpp:217-260).
#pragma unroll 1
    for (int axis = 0; axis < D; ++axis) {
      int caxis = 0, naxis = 1;  // c[axis], nbins[axis] (static register indexing)
#pragma unroll
      for (int k = 0; k < D; ++k)
        if (k == axis) {
          caxis = c[k];
          naxis = static_cast<int>(g.nbins[k]);
        }
#pragma unroll 1
      for (int side = 0; side < 2; ++side) {
        const int fixed = caxis + (side == 0 ? -rho : rho);
        if (fixed < 0 || fixed >= naxis) continue;
        int lo[D], hi[D], cc[D];
        bool empty = false;
#pragma unroll
        for (int k = 0; k < D; ++k) {
          if (k == axis) {
            lo[k] = hi[k] = fixed;
          } else {
            const int r = k < axis ? rho - 1 : rho;
            lo[k] = max(0, c[k] - r);
            hi[k] = min(static_cast<int>(g.nbins[k]) - 1, c[k] + r);
            if (lo[k] > hi[k]) empty = true;
          }
          cc[k] = lo[k];
        }
        if (empty) continue;
        for (;;) {
          scan_bin<D, KT>(g, cc, y, offsets, ps, ids, best);
          bool carry = true;  // odometer over the axes other than `axis`
#pragma unroll
          for (int k = 0; k < D; ++k) {
            if (carry && k != axis) {
              if (++cc[k] > hi[k]) {
                cc[k] = lo[k];
              } else {
                carry = false;
              }
            }
          }
          if (carry) break;
        }
      }
    }
  }
  const int kk = static_cast<int>(best.pushed < g.k ? best.pushed : static_cast<int64_t>(g.k));
  double value;
  if (best.D[0] < g.hit_tol2) {
    value = __ldg(vals + best.I[0]);
  } else {
    double wsum = 0.0, vsum = 0.0;
#pragma unroll
    for (int j = 0; j < KT; ++j) {
      if (j < kk) {
        const double w = g.pow2 ? __ddiv_rn(1.0, best.D[j]) : pow(best.D[j], -0.5 * g.power);
        wsum = __dadd_rn(wsum, w);
        vsum = __dadd_rn(vsum, __dmul_rn(w, __ldg(vals + best.I[j])));
      }
    }
    value = __ddiv_rn(vsum, wsum);
  }
  out[node] = value;
  if (nbr) {
#pragma unroll
    for (int j = 0; j < KT; ++j)
      if (j < g.k) nbr[node * g.k + j] = j < kk ? best.I[j] : 0xFFFFFFFFu;
  }
  const double nearest = sqrt(best.D[0]);
  atomicMax(stats, ord(nearest));
  const unsigned active = __activemask();
  const unsigned extra = __ballot_sync(active, nearest > g.bin_diag);
  if (extra && (threadIdx.x & 31) == __ffs(active) - 1)
    atomicAdd(stats + 1, static_cast<unsigned long long>(__popc(extra)));
}

template <int D, int KT>
void launch_nodes(const IdwGrid& g, const uint32_t* offsets, const double* ps, const uint32_t* ids,
                  const double* vals, double* out, unsigned long long* stats, uint32_t* nbr, cudaStream_t s) {
  const unsigned blocks = static_cast<unsigned>(ceil_div(g.n_nodes, 128));
  idw_node_kernel<D, KT><<<blocks, 128, 0, s>>>(g, offsets, ps, ids, vals, out, stats, nbr);
  check_launch("idw_node_kernel");
}
template <int D>
void launch_nodes_k(const IdwGrid& g, const uint32_t* offsets, const double* ps, const uint32_t* ids,
                    const double* vals, double* out, unsigned long long* stats, uint32_t* nbr, cudaStream_t s) {
  if (g.k <= 8)
    launch_nodes<D, 8>(g, offsets, ps, ids, vals, out, stats, nbr, s);
  else if (g.k <= 16)
    launch_nodes<D, 16>(g, offsets, ps, ids, vals, out, stats, nbr, s);
  else if (g.k <= 32)
    launch_nodes<D, 32>(g, offsets, ps, ids, vals, out, stats, nbr, s);
  else
    launch_nodes<D, 64>(g, offsets, ps, ids, vals, out, stats, nbr, s);
}

// points / values / out / nbr are device pointers here.
void interpolate_device(const double* pts, const double* vals, int64_t q, int d, const double* box_lo,
                        const double* box_hi, const int64_t* sizes, const double* glo, const double* ghi,
                        int neighbors, double power, double* out, fstk_interp_report* report, uint32_t* nbr,
                        cudaStream_t s) {
  require(d >= 1 && d <= kMaxOrder, FSTK_E_SHAPE, "point cloud dimension must be in [1, 8]");
  require(q >= 1, FSTK_E_DATA, "point cloud is empty");
  require(q < (int64_t(1) << 32) - 1, FSTK_E_SHAPE, "point cloud too large (ids are 32-bit)");
  for (int k = 0; k < d; ++k) {
    require(sizes[k] >= 2, FSTK_E_PARAMETER, "grid sizes must be >= 2");
    require(glo[k] < ghi[k], FSTK_E_PARAMETER, "grid intervals must be nondegenerate");
  }
  const int kn = neighbors > 0 ? neighbors : 2 * d + 2;
  require(power > 0.0, FSTK_E_PARAMETER, "IDW power must be positive");
  require(kn <= kIdwMaxK, FSTK_E_PARAMETER, "IDW neighbours: at most 64 on the GPU");
  // Box and finiteness (PointCloud::from_data / validate).
  DevBuf<unsigned long long> red(2 * kMaxOrder + 4);
  std::vector<unsigned long long> init(2 * kMaxOrder + 4, 0ull);
  for (int k = 0; k < kMaxOrder; ++k) init[k] = ~0ull;
  FSTK_CUDA(cudaMemcpyAsync(red.p, init.data(), init.size() * 8, cudaMemcpyHostToDevice, s));
  const unsigned rb = static_cast<unsigned>(std::min<int64_t>(ceil_div(q, 256), 1184));
  box_kernel<<<rb, 256, 0, s>>>(pts, q, d, red.p, red.p + kMaxOrder, red.p + 2 * kMaxOrder);
  check_launch("box_kernel");
  nonfinite_kernel<<<rb, 256, 0, s>>>(vals, q, red.p + 2 * kMaxOrder + 1);
  check_launch("nonfinite_kernel");
  std::vector<unsigned long long> hr(2 * kMaxOrder + 4);
  FSTK_CUDA(cudaMemcpyAsync(hr.data(), red.p, hr.size() * 8, cudaMemcpyDeviceToHost, s));
  FSTK_CUDA(cudaStreamSynchronize(s));
  require(hr[2 * kMaxOrder] == 0, FSTK_E_DATA, "point coordinates must be finite");
  require(hr[2 * kMaxOrder + 1] == 0, FSTK_E_DATA, "point cloud values must be finite");
  double blo[kMaxOrder], bhi[kMaxOrder];
  for (int k = 0; k < d; ++k) {
    const double mn = unord(hr[k]), mx = unord(hr[kMaxOrder + k]);
    blo[k] = box_lo ? box_lo[k] : mn;
    bhi[k] = box_hi ? box_hi[k] : mx;
    require(mn >= blo[k] && mx <= bhi[k], FSTK_E_DATA, "bounding box does not cover the points");
  }
  // build_index sizing (ingest.cpp:140-175), on the host in the same order.
  IdwGrid g{};
  g.d = d;
  g.k = kn;
  g.power = power;
  g.pow2 = power == 2.0 ? 1 : 0;
  g.q = q;
  g.n_nodes = 1;
  const double per_mode = std::pow(std::max(1.0, static_cast<double>(q) / 4.0), 1.0 / d);
  int64_t total = 1;
  for (int k = 0; k < d; ++k) {
    g.sizes[k] = sizes[k];
    g.glo[k] = glo[k];
    g.ghi[k] = ghi[k];
    g.n_nodes *= sizes[k];
    g.nbins[k] = std::max<int64_t>(1, std::min<int64_t>(sizes[k] - 1, static_cast<int64_t>(std::llround(per_mode))));
    total *= g.nbins[k];
  }
  while (total > (int64_t(1) << 22)) {
    total = 1;
    for (int k = 0; k < d; ++k) {
      g.nbins[k] = std::max<int64_t>(1, g.nbins[k] / 2);
      total *= g.nbins[k];
    }
  }
  double min_w = std::numeric_limits<double>::infinity(), diag2 = 0.0, cell_diag2 = 0.0;
  bool covered = true;
  for (int k = 0; k < d; ++k) {
    g.lo[k] = std::min(glo[k], blo[k]);
    const double hi = std::max(ghi[k], bhi[k]);
    g.width[k] = (hi - g.lo[k]) / static_cast<double>(g.nbins[k]);
    if (g.width[k] <= 0.0) g.width[k] = 1.0;
    min_w = std::min(min_w, g.width[k]);
    diag2 += g.width[k] * g.width[k];
    const double h = (ghi[k] - glo[k]) / static_cast<double>(sizes[k] - 1);
    cell_diag2 += h * h;
    if (blo[k] < glo[k] || bhi[k] > ghi[k]) covered = false;
  }
  g.min_width = min_w;
  g.bin_diag = std::sqrt(diag2);
  g.hit_tol2 = 1e-24 * cell_diag2;
  // The index on the device: bin ids, histogram, scan, scatter.
  DevBuf<uint32_t> bin(q), counts(total + 1), offsets(total + 1), ids(q);
  DevBuf<double> ps(q * d);
  FSTK_CUDA(cudaMemsetAsync(counts.p, 0, (total + 1) * sizeof(uint32_t), s));
  const unsigned pb = static_cast<unsigned>(ceil_div(q, 256));
  bin_kernel<<<pb, 256, 0, s>>>(g, pts, bin.p, counts.p);
  check_launch("bin_kernel");
  size_t tmp_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, counts.p, offsets.p, static_cast<int>(total + 1), s);
  DevBuf<uint8_t> tmp(tmp_bytes + 16);
  cub::DeviceScan::ExclusiveSum(tmp.p, tmp_bytes, counts.p, offsets.p, static_cast<int>(total + 1), s);
  check_launch("cub::DeviceScan");
  FSTK_CUDA(cudaMemcpyAsync(counts.p, offsets.p, (total + 1) * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
  scatter_kernel<<<pb, 256, 0, s>>>(g, pts, bin.p, counts.p, ps.p, ids.p);
  check_launch("scatter_kernel");
  unsigned long long* stats = red.p + 2 * kMaxOrder + 2;
  FSTK_CUDA(cudaMemsetAsync(stats, 0, 2 * sizeof(unsigned long long), s));
  switch (d) {
    case 1: launch_nodes_k<1>(g, offsets.p, ps.p, ids.p, vals, out, stats, nbr, s); break;
    case 2: launch_nodes_k<2>(g, offsets.p, ps.p, ids.p, vals, out, stats, nbr, s); break;
    case 3: launch_nodes_k<3>(g, offsets.p, ps.p, ids.p, vals, out, stats, nbr, s); break;
    case 4: launch_nodes_k<4>(g, offsets.p, ps.p, ids.p, vals, out, stats, nbr, s); break;
    case 5: launch_nodes_k<5>(g, offsets.p, ps.p, ids.p, vals, out, stats, nbr, s); break;
    case 6: launch_nodes_k<6>(g, offsets.p, ps.p, ids.p, vals, out, stats, nbr, s); break;
    case 7: launch_nodes_k<7>(g, offsets.p, ps.p, ids.p, vals, out, stats, nbr, s); break;
    default: launch_nodes_k<8>(g, offsets.p, ps.p, ids.p, vals, out, stats, nbr, s); break;
  }
  unsigned long long hs[2];
  FSTK_CUDA(cudaMemcpyAsync(hs, stats, sizeof(hs), cudaMemcpyDeviceToHost, s));
  FSTK_CUDA(cudaStreamSynchronize(s));
  if (report) {
    report->box_covered = covered ? 1 : 0;
    report->max_nearest_distance = unord(hs[0]);
    report->extrapolated_fraction = static_cast<double>(hs[1]) / static_cast<double>(g.n_nodes);
  }
}

}  // namespace
}  // namespace fstk_gpu

using namespace fstk_gpu;

extern "C" {

int32_t fstk_gpu_interpolate_to_grid(const double* points, const double* values, int64_t q, int32_t d,
                                     const double* box_lo, const double* box_hi, const int64_t* sizes,
                                     const double* grid_lo, const double* grid_hi, int32_t neighbors,
                                     double power, double* out, fstk_interp_report* report,
                                     uint32_t* neighbor_ids, int32_t device, fstk_gpu_error* err) {
  return guarded(err, [&] {
    require(points && values && sizes && grid_lo && grid_hi && out, FSTK_E_PARAMETER, "null argument");
    require(d >= 1 && d <= kMaxOrder, FSTK_E_SHAPE, "point cloud dimension must be in [1, 8]");
    require(q >= 1, FSTK_E_DATA, "point cloud is empty");
    DeviceGuard dg(device);
    int64_t n_nodes = 1;
    for (int k = 0; k < d; ++k) n_nodes *= std::max<int64_t>(sizes[k], 0);
    const int kn = neighbors > 0 ? neighbors : 2 * d + 2;
    cudaStream_t s = nullptr;
    FSTK_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    struct StreamGuard {
      cudaStream_t s;
      ~StreamGuard() { cudaStreamDestroy(s); }
    } sg{s};
    DevBuf<double> dp(q * d), dv(q), dout(std::max<int64_t>(n_nodes, 1));
    DevBuf<uint32_t> dn(neighbor_ids ? std::max<int64_t>(n_nodes * kn, 1) : 1);
    FSTK_CUDA(cudaMemcpyAsync(dp.p, points, q * d * 8, cudaMemcpyHostToDevice, s));
    FSTK_CUDA(cudaMemcpyAsync(dv.p, values, q * 8, cudaMemcpyHostToDevice, s));
    interpolate_device(dp.p, dv.p, q, d, box_lo, box_hi, sizes, grid_lo, grid_hi, neighbors, power, dout.p,
                       report, neighbor_ids ? dn.p : nullptr, s);
    FSTK_CUDA(cudaMemcpyAsync(out, dout.p, n_nodes * 8, cudaMemcpyDeviceToHost, s));
    if (neighbor_ids)
      FSTK_CUDA(cudaMemcpyAsync(neighbor_ids, dn.p, n_nodes * kn * 4, cudaMemcpyDeviceToHost, s));
    FSTK_CUDA(cudaStreamSynchronize(s));
  });
}

int32_t fstk_gpu_interpolate_to_grid_device(const double* points, const double* values, int64_t q, int32_t d,
                                            const double* box_lo, const double* box_hi, const int64_t* sizes,
                                            const double* grid_lo, const double* grid_hi, int32_t neighbors,
                                            double power, double* out, fstk_interp_report* report,
                                            uint32_t* neighbor_ids, void* stream, fstk_gpu_error* err) {
  return guarded(err, [&] {
    require(points && values && sizes && grid_lo && grid_hi && out, FSTK_E_PARAMETER, "null argument");
    interpolate_device(points, values, q, d, box_lo, box_hi, sizes, grid_lo, grid_hi, neighbors, power, out,
                       report, neighbor_ids, static_cast<cudaStream_t>(stream));
  });
}

}  // extern "C"
