// Hand-written sm_100a int8 SYRK for the CRT Gram (fstk_gram.cu): the
// tensor-core stage of A^T A (randls.cpp:112-123 solves the sketched system
// whose normal equations these are; randls.cpp:315-348 builds it).
//
// For every modulus t of one row segment, C_t = R_t^T R_t where R_t is the
// kp x np int8 residue plane (column a contiguous along K).  Only the lower
// triangle of C_t is needed (G is symmetric), so only 256 x 256 tiles with
// tile row >= tile column are computed -- the library GEMMs this replaces
// computed whole rectangular column blocks.  The epilogue reduces each int32
// sum modulo m_t and stores the symmetric residue as one byte: the Garner
// fold (crt_fold_kernel) needs nothing more, so the C planes it streams are
// 4x smaller than int32 sums and the fold's arithmetic is unchanged.
//
// Structure (one persistent kernel for all moduli and tiles of a column block):
//  * CTA pairs (__cluster_dims__(2)) run tcgen05.mma.cta_group::2.kind::i8,
//    M = 256 (128 rows per CTA), N = 256, K = 32 per instruction; each CTA
//    TMA-loads (cp.async.bulk.tensor, 128B swizzle) its 128-row halves of
//    the A and B panels, 128 bytes of K per stage, 6 stages deep.
//  * warp 0: TMA producer; warp 1 (leader CTA): the single MMA-issuing
//    thread; warp 2: TMEM allocator; warps 4-7: epilogue.
//  * Accumulators live in TMEM (2 x 256 columns, double-buffered, so the
//    epilogue of tile i overlaps the MMAs of tile i+1) and are read back
//    with tcgen05.ld.
// Exactness: |C_t| <= kp * 127^2 < 2^31 for kp <= 133,152, so the int32
// accumulation is exact, as with the library GEMMs; the stored residues are
// congruent to the library's int32 sums modulo m_t, so the fold produces the
// identical Gram bit for bit.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <mutex>

#include "fstk_common.cuh"
#include "fstk_internal.h"

namespace fstk_gpu {

namespace {

constexpr int kTile = 256;                    // output tile edge (CTA pair)
constexpr int kHalf = 128;                    // rows per CTA
constexpr int kKB = 128;                      // K bytes per stage (one swizzle row)
constexpr int kStages = 6;
constexpr int kPanelBytes = kHalf * kKB;      // 16 KB: one operand half
constexpr int kStageBytes = 2 * kPanelBytes;  // A half + B half
constexpr int kThreads = 256;
constexpr int kAccCols = 256;                 // TMEM columns per accumulator
constexpr int kSmemBytes = kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;

struct SyrkParams {
  int nm;               // moduli (residue planes)
  int kblocks;          // kp / 128
  int np;               // columns per plane (rows of the tensor map per plane)
  int c0;               // first column of the block
  int ntj;              // tile columns of the block
  int nti;              // tile rows of the block
  int tri;              // ntj (ntj + 1) / 2: tiles of the diagonal band
  int per_mod;          // tiles per modulus
  int ntasks;           // nm * per_mod
  long long ldc;        // C rows (m)
  long long cstride;    // plane stride of C
  int8_t* C;
  int mod[kSyrkMaxModuli];
  double inv[kSyrkMaxModuli];
};

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of the same variable in CTA `rank` of the cluster.
__device__ __forceinline__ uint32_t map_rank(const void* p, uint32_t rank) {
  uint32_t out;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(out) : "r"(smem_u32(p)), "r"(rank));
  return out;
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// K-major operand tile of 128 rows x 128 bytes written by TMA with 128-byte
// swizzle: rows 128 B apart, 8-row groups 1024 B apart (SBO), descriptor
// version 1 (sm_100), layout SWIZZLE_128B.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>(1) << 16;           // LBO (unused for swizzled K-major)
  d |= static_cast<uint64_t>(1024 >> 4) << 32;   // SBO
  d |= static_cast<uint64_t>(1) << 46;           // version
  d |= static_cast<uint64_t>(2) << 61;           // SWIZZLE_128B
  return d;
}
// kind::i8 instruction descriptor: s8 x s8 -> s32, both K-major, M = 256, N = 256.
constexpr uint32_t kIdesc = (2u << 4) | (1u << 7) | (1u << 10) |
                            (static_cast<uint32_t>(kTile >> 3) << 17) |
                            (static_cast<uint32_t>(kTile >> 4) << 24);

__device__ __forceinline__ void tma_load_2sm(void* dst, const CUtensorMap* map, int x, int y,
                                             uint32_t bar_cluster) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_cluster), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(kIdesc), "r"(acc)
      : "memory");
}
// Arrive once on the mbarrier at this offset in both CTAs of the pair when
// every previously issued MMA of this thread has completed.
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"(static_cast<uint16_t>(3))
      : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, "
      "%30, %31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
        "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
        "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Task -> (modulus, tile row, tile column), tile row >= tile column: per
// modulus the diagonal band first (tile rows 0..ntj-1, triangular), then the
// full rows below it, tile columns fastest -- consecutive tasks (which run
// concurrently on neighbouring pairs) share their A and B panels in L2.
__device__ __forceinline__ void decode_task(const SyrkParams& p, int task, int& t, int& ti, int& tj) {
  t = task / p.per_mod;
  int r = task - t * p.per_mod;
  if (r < p.tri) {
    ti = 0;
    while ((ti + 1) * (ti + 2) / 2 <= r) ++ti;
    tj = r - ti * (ti + 1) / 2;
  } else {
    r -= p.tri;
    ti = p.ntj + r / p.ntj;
    tj = r - (ti - p.ntj) * p.ntj;
  }
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    syrk_i8_kernel(const __grid_constant__ CUtensorMap map, const SyrkParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const uint32_t rank = cluster_rank();
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int pair = blockIdx.x >> 1;
  const int npairs = gridDim.x >> 1;

  if (warp == 0 && lane == 0)
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map)) : "memory");
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 8);  // 4 epilogue warps x 2 CTAs
    }
    fence_mbar_init();
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(2 * kAccCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(tmem_slot);

  if (warp == 0) {
    if (lane == 0) {
      // ---- TMA producer (both CTAs): this CTA's 128-row halves of A and B.
      uint32_t stage = 0, phase = 0;
      for (int task = pair; task < p.ntasks; task += npairs) {
        int t, ti, tj;
        decode_task(p, task, t, ti, tj);
        const int base = t * p.np + p.c0 + static_cast<int>(rank) * kHalf;
        const int rowA = base + ti * kTile;
        const int rowB = base + tj * kTile;
        for (int kb = 0; kb < p.kblocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * kStageBytes;
          if (rank == 0) mbar_arrive_expect_tx(&full[stage], 2 * kStageBytes);
          const uint32_t bar = map_rank(&full[stage], 0);
          tma_load_2sm(sa, &map, kb * kKB, rowA, bar);
          tma_load_2sm(sa + kPanelBytes, &map, kb * kKB, rowB, bar);
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0 && lane == 0) {
      // ---- MMA issuer (leader CTA, one thread).
      uint32_t stage = 0, phase = 0, acc = 0, aphase = 0;
      for (int task = pair; task < p.ntasks; task += npairs) {
        mbar_wait(&tempty[acc], aphase ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + acc * kAccCols;
        for (int kb = 0; kb < p.kblocks; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * kStageBytes);
          const uint64_t da = sw128_desc(sa), db = sw128_desc(sa + kPanelBytes);
#pragma unroll
          for (int k = 0; k < kKB / 32; ++k)
            mma_i8(d, da + 2 * k, db + 2 * k, (kb | k) != 0 ? 1u : 0u);
          mma_commit_pair(&empty[stage]);
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        mma_commit_pair(&tfull[acc]);
        acc ^= 1;
        if (acc == 0) aphase ^= 1;
      }
    }
  } else if (warp >= 4) {
    // ---- Epilogue (both CTAs): TMEM lanes 32q..32q+31 = this warp's rows.
    const int q = warp & 3;
    const uint32_t tempty_leader0 = map_rank(&tempty[0], 0);
    const uint32_t tempty_leader1 = map_rank(&tempty[1], 0);
    uint32_t acc = 0, aphase = 0;
    for (int task = pair; task < p.ntasks; task += npairs) {
      int t, ti, tj;
      decode_task(p, task, t, ti, tj);
      const int mt = p.mod[t];
      const double inv = p.inv[t];
      const long long i = static_cast<long long>(ti) * kTile + rank * kHalf + q * 32 + lane;
      int8_t* crow = p.C + t * p.cstride + i + static_cast<long long>(tj) * kTile * p.ldc;
      mbar_wait(&tfull[acc], aphase);
      tc_fence_after();
      const uint32_t tbase = tmem + acc * kAccCols + (static_cast<uint32_t>(q * 32) << 16);
#pragma unroll 1
      for (int ch = 0; ch < kAccCols / 32; ++ch) {
        uint32_t v[32];
        tmem_ld32(tbase + ch * 32, v);
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          const int x = static_cast<int>(v[c]);
          // Symmetric residue: |x| < 2^31 is exact in fp64 and x/m is never
          // within 2^-21 of a half-integer unless it is one (then either
          // representative, |r| <= 127, is congruent).
          const int qq = static_cast<int>(rint(static_cast<double>(x) * inv));
          const int r = x - qq * mt;
          crow[static_cast<long long>(ch * 32 + c) * p.ldc] = static_cast<int8_t>(r);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        const uint32_t bar = acc ? tempty_leader1 : tempty_leader0;
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar)
                     : "memory");
      }
      acc ^= 1;
      if (acc == 0) aphase ^= 1;
    }
  }

  __syncwarp();
  tc_fence_before();
  cluster_sync_all();
  if (warp == 2)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(2 * kAccCols)
                 : "memory");
}

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !f) {
      cudaGetLastError();
      fail(FSTK_E_COMPUTE, "cuTensorMapEncodeTiled unavailable (driver too old for sm_100a TMA)");
    }
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  return fn;
}

}  // namespace

int syrk_i8_sm_count(int device) {
  static std::mutex mu;
  static int cached[64] = {0};
  std::lock_guard<std::mutex> lk(mu);
  if (device < 0 || device >= 64) device = 0;
  if (!cached[device]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device);
    cached[device] = v > 1 ? v : 2;
  }
  return cached[device];
}

double syrk_i8_residues(const int8_t* planes, int nm, int64_t kp, int64_t np, int64_t c0, int64_t wn,
                        int64_t m, const int* moduli, int8_t* C, int64_t cstride, int device,
                        cudaStream_t s) {
  require(nm >= 1 && nm <= kSyrkMaxModuli, FSTK_E_COMPUTE, "internal: SYRK modulus count");
  require(kp % kKB == 0 && kp > 0 && kp <= 133120, FSTK_E_COMPUTE, "internal: SYRK segment rows");
  require(np % kTile == 0 && c0 % kTile == 0 && wn % kTile == 0 && m % kTile == 0 && c0 + m == np,
          FSTK_E_COMPUTE, "internal: SYRK block shape");
  require(static_cast<int64_t>(nm) * np < (int64_t(1) << 31), FSTK_E_COMPUTE,
          "internal: SYRK plane rows exceed the tensor-map range");
  static std::once_flag attr_once;
  std::call_once(attr_once, [] {
    cudaFuncSetAttribute(syrk_i8_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
  });
  CUtensorMap map;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(kp), static_cast<cuuint64_t>(nm * np)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(kp)};
  const cuuint32_t box[2] = {kKB, kHalf};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult cr = tensor_map_encoder()(
      &map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<int8_t*>(planes), dims, strides, box, estr,
      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) fail(FSTK_E_COMPUTE, "cuTensorMapEncodeTiled failed for the SYRK planes");
  SyrkParams p{};
  p.nm = nm;
  p.kblocks = static_cast<int>(kp / kKB);
  p.np = static_cast<int>(np);
  p.c0 = static_cast<int>(c0);
  p.ntj = static_cast<int>(wn / kTile);
  p.nti = static_cast<int>(m / kTile);
  p.tri = p.ntj * (p.ntj + 1) / 2;
  p.per_mod = p.tri + (p.nti - p.ntj) * p.ntj;
  p.ntasks = nm * p.per_mod;
  p.ldc = m;
  p.cstride = cstride;
  p.C = C;
  for (int t = 0; t < nm; ++t) {
    p.mod[t] = moduli[t];
    p.inv[t] = 1.0 / static_cast<double>(moduli[t]);
  }
  const int pairs = std::max(1, std::min(p.ntasks, syrk_i8_sm_count(device) / 2));
  syrk_i8_kernel<<<2 * pairs, kThreads, kSmemBytes, s>>>(map, p);
  check_launch("syrk_i8_kernel");
  return 2.0 * static_cast<double>(p.ntasks) * kTile * kTile * static_cast<double>(kp);
}

}  // namespace fstk_gpu
