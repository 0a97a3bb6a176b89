// Hand-written sm_100a int8 SYRK (+ CRT fold) for the Gram of the sketched
// system (fstk_gram.cu): the tensor-core stage of A^T A (randls.cpp:112-123
// solves the sketched least-squares system whose normal equations these are;
// randls.cpp:315-348 builds it).
//
// For every modulus t of a row segment, C_t = R_t^T R_t on the int8 tensor
// cores (R_t = the kp x np residue plane t), lower-triangle 256 x 256 tiles
// only (the library GEMMs it replaces computed whole column blocks, ~6% of
// the upper triangle), each int32 sum reduced in the epilogue to its
// symmetric residue modulo m_t.  Garner's algorithm then rebuilds each exact
// integer sum and adds 2^(e_a+e_b-2k) times it into G.
//
// Common structure (CTA pairs, persistent, dynamic tile scheduler):
//  * __cluster_dims__(2): tcgen05.mma.cta_group::2.kind::i8, M = 256 (128
//    rows per CTA), N = 256, K = 32 per instruction, issued by one thread of
//    the leader CTA; each CTA TMA-loads (cp.async.bulk.tensor.2d.cta_group::2,
//    128B swizzle) its 128-row halves of the A and B panels, 128 bytes of K
//    per stage, 7 stages deep; tcgen05.commit multicast frees stages and
//    hands accumulators over in both CTAs.
//  * warp 0: TMA producer; warp 1 (leader CTA): the MMA-issuing thread;
//    warp 2: TMEM allocator; the epilogue warps read the two double-buffered
//    256-column int32 accumulators with tcgen05.ld.
//  * The leader's producer claims tasks with one atomicAdd and publishes them
//    through a ring of slots in both CTAs (remote st.shared::cluster +
//    mbarrier.arrive.release.cluster), so the concurrently active tiles stay
//    a contiguous window of the banded tile order however the pairs drift.
//  * Producer, MMA and epilogue waits are suspend-hinted mbarrier.try_wait.
//
// Variants ($FSTK_SYRK_MODE), all bit-identical:
//  * "permod" (default, syrk_res_kernel): one launch per column block and
//    modulus, byte residues to C (ld m), then crt_fold4_kernel -- like the
//    library GEMMs this keeps a 2,048-wide B block resident in L2 for the
//    whole launch; measured fastest (C2 Gram kernels 1.028 s vs 1.063 s for
//    the cuBLASLt engine on the same box);
//  * "block": the same kernel, every modulus of a column block in one launch;
//  * "fused" (syrk_crt_kernel): one launch per segment over the whole lower
//    triangle, all moduli of a tile on one pair, 8 epilogue warps keeping the
//    byte residues in an L2-resident per-CTA scratch and folding into G while
//    the next tile's MMAs run -- no fold kernel, but every modulus switch
//    re-reads the wave's panels (77% tensor-pipe activity against 90%).
// Exactness: |C_t| <= kp * 127^2 < 2^30 for kp <= 66,560, so the int32
// accumulation is exact; residues are congruent to the int32 sums, so the
// Garner digits -- and G -- equal the library engine's bit for bit.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <atomic>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "fstk_common.cuh"
#include "fstk_crt.cuh"
#include "fstk_internal.h"

namespace fstk_gpu {

namespace {

constexpr int kTile = 256;                    // output tile edge (CTA pair)
constexpr int kHalf = 128;                    // rows per CTA
constexpr int kKB = 128;                      // K bytes per stage (one swizzle row)
constexpr int kPanelBytes = kHalf * kKB;      // 16 KB: one operand half
constexpr int kStageBytes = 2 * kPanelBytes;  // A half + B half
constexpr int kEpiWarps = 8;   // two per TMEM lane quarter, 128 columns each
constexpr int kThreads = 32 * (4 + kEpiWarps);
constexpr int kStages = 7;
constexpr int kAccCols = 256;                 // TMEM columns per accumulator
constexpr int kTaskRing = 4;    // dynamic scheduler slots
constexpr int kSmemBytes = kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;

constexpr int kBandTilesDefault = 8;   // tile columns per band
constexpr int kMaxBands = 64;

struct SyrkParams {
  int kblocks;          // kp / 128
  int np;               // columns per plane (rows of the tensor map per plane)
  int nt;               // tiles per side (np / 256)
  int nbands;
  int band;             // tile columns per band
  int band_start[kMaxBands + 1];  // first task of each band
  int ntasks;
  int n;                // valid columns of G
  int k;                // integer bits (scale 2^-2k)
  int accumulate, negate;
  int hint;             // 0: none, 1: L2 evict_last, 2: evict_first (experiments)
  long long ldg;
  double* G;
  const int* ex;        // per-column exponents of this segment
  uint8_t* scratch;     // per CTA: NM x 128 x 256 residue bytes
  int lookahead;        // L2 prefetch distance in K blocks (0 = off)
  int* counter;         // dynamic tile scheduler: next task (zeroed before the launch)
  unsigned long long* dbg;  // optional wait-cycle counters ($FSTK_SYRK_DEBUG)
  unsigned sleep_ns;    // suspend hint of the epilogue's waits (0 = spin)
  unsigned pc_sleep;    // experiments: suspend hint of the producer / MMA waits
  int mod[kSyrkMaxModuli];
  unsigned p16[kSyrkMaxModuli];   // 2^16 mod m
  unsigned off[kSyrkMaxModuli];   // a multiple of m >= 2^22 (makes the folded value >= 0)
  unsigned magic[kSyrkMaxModuli]; // floor(2^32 / m)
};

// Symmetric residue of an int32 sum |x| < 2^30 modulo m <= 255 in integer
// ALU operations only (the epilogue shares the SM with the tensor pipe; fp64
// or conversion-pipe arithmetic here measured math-pipe-throttled):
// x = hi 2^16 + lo folds to y = hi (2^16 mod m) + lo + off in [0, 2^23),
// then Barrett with floor(2^32/m) gives q in {floor(y/m) - 1, floor(y/m)}.
__device__ __forceinline__ int sym_residue(int x, int m, unsigned p16, unsigned off, unsigned magic) {
  const unsigned y = static_cast<unsigned>((x >> 16) * static_cast<int>(p16)) +
                     static_cast<unsigned>(x & 0xFFFF) + off;
  const unsigned q = __umulhi(y, magic);
  int r = static_cast<int>(y - q * static_cast<unsigned>(m));
  if (r >= m) r -= m;
  if (r > (m >> 1)) r -= m;
  return r;
}

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
// Blocking wait with a hardware suspend hint: the waiting thread sleeps until
// the phase completes (or ~0.5 ms pass) instead of spinning on try_wait -- the
// epilogue warps wait ~100 us per tile and the kernel runs at the power cap,
// where issue slots spent spinning cost clock speed.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity, uint32_t hint_ns = 500000u) {
  uint32_t ok;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity), "r"(hint_ns)
        : "memory");
  } while (!ok);
}
// Cluster-scope acquire wait (task slots written by the peer CTA) and remote
// release-arrive on an mbarrier given by its shared::cluster address.
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!ok);
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t bar_cluster) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster) : "memory");
}
__device__ __forceinline__ void st_cluster_s32(uint32_t addr, int v) {
  asm volatile("st.shared::cluster.s32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
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
__device__ __forceinline__ void tma_load_2sm_hint(void* dst, const CUtensorMap* map, int x, int y,
                                                  uint32_t bar_cluster, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_cluster), "r"(x), "r"(y), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void tma_prefetch_l2(const CUtensorMap* map, int x, int y) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(x), "r"(y)
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

// Task -> (tile row, tile column), tile row >= tile column: bands of
// kBandTiles tile columns; in each band the diagonal triangle first, then the
// full rows below it, tile columns fastest.
__device__ __forceinline__ void decode_task(const SyrkParams& p, int task, int& ti, int& tj) {
  int b = 0;
  while (b + 1 < p.nbands && p.band_start[b + 1] <= task) ++b;
  int r = task - p.band_start[b];
  const int c0 = b * p.band;
  const int wb = min(p.band, p.nt - c0);
  const int tri = wb * (wb + 1) / 2;
  if (r < tri) {
    int a = 0;
    while ((a + 1) * (a + 2) / 2 <= r) ++a;
    ti = c0 + a;
    tj = c0 + r - a * (a + 1) / 2;
  } else {
    r -= tri;
    ti = c0 + wb + r / wb;
    tj = c0 + r % wb;
  }
}

__device__ __forceinline__ int sext_byte(uint32_t w, int b) {
  return static_cast<int>(w << (24 - 8 * b)) >> 24;
}

template <int NM>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    syrk_crt_kernel(const __grid_constant__ CUtensorMap map, const SyrkParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint64_t* tempty = tfull + 2;
  // Dynamic tile scheduler: the leader's producer claims tasks with one
  // atomic per task and publishes them through a ring of slots in both CTAs,
  // so the concurrently active tiles stay a contiguous window of the banded
  // order however the pairs' speeds drift (static round-robin let them
  // spread and tripled the panel re-reads from DRAM).
  uint64_t* task_full = tempty + 2;          // per slot, both CTAs: count 1
  uint64_t* task_empty = task_full + kTaskRing;  // per slot, leader: 1 + 2 kEpiWarps + 1
  int* task_slot = reinterpret_cast<int*>(task_empty + kTaskRing);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(task_slot + kTaskRing);

  const uint32_t rank = cluster_rank();
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0)
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map)) : "memory");
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 2 * kEpiWarps);  // epilogue warps x 2 CTAs
    }
    for (int r = 0; r < kTaskRing; ++r) {
      mbar_init(&task_full[r], 1);
      mbar_init(&task_empty[r], 2 + 2 * kEpiWarps);  // MMA + peer producer + epilogue warps
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
      uint64_t policy = 0;
      if (p.hint == 1) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(policy));
      if (p.hint == 2) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
      const uint32_t peer_slot0 = map_rank(&task_slot[0], 1);
      const uint32_t peer_full0 = map_rank(&task_full[0], 1);
      const uint32_t lead_empty0 = map_rank(&task_empty[0], 0);
      for (int n = 0;; ++n) {
        const int r = n % kTaskRing;
        const uint32_t rph = (n / kTaskRing) & 1;
        int task;
        if (rank == 0) {
          mbar_wait(&task_empty[r], rph ^ 1);
          task = atomicAdd(p.counter, 1);
          if (task >= p.ntasks) task = -1;
          task_slot[r] = task;
          st_cluster_s32(peer_slot0 + 4 * r, task);
          mbar_arrive(&task_full[r]);
          mbar_arrive_remote(peer_full0 + 8 * r);
        } else {
          mbar_wait_cluster(&task_full[r], rph);
          task = *reinterpret_cast<volatile int*>(&task_slot[r]);
          mbar_arrive_remote(lead_empty0 + 8 * r);
        }
        if (task < 0) break;
        int ti, tj;
        decode_task(p, task, ti, tj);
        for (int t = 0; t < NM; ++t) {
          const int base = t * p.np + static_cast<int>(rank) * kHalf;
          const int rowA = base + ti * kTile;
          const int rowB = base + tj * kTile;
          for (int kb = 0; kb < p.kblocks; ++kb) {
            // Steady L2 lookahead: the K block `lookahead` stages ahead of
            // this one (continuing into the next modulus's panels) is pulled
            // into L2, so the TMA loads meet L2 rather than DRAM latency --
            // the 7-stage shared-memory ring covers ~2.5 us.
            if (p.lookahead) {
              const int fk = kb + p.lookahead;
              if (fk < p.kblocks) {
                tma_prefetch_l2(&map, fk * kKB, rowA);
                tma_prefetch_l2(&map, fk * kKB, rowB);
              } else if (t + 1 < NM) {
                tma_prefetch_l2(&map, (fk - p.kblocks) * kKB, rowA + p.np);
                tma_prefetch_l2(&map, (fk - p.kblocks) * kKB, rowB + p.np);
              }
            }
            if (p.pc_sleep) mbar_wait_sleep(&empty[stage], phase ^ 1, p.pc_sleep); else mbar_wait(&empty[stage], phase ^ 1);
            uint8_t* sa = smem + stage * kStageBytes;
            if (rank == 0) mbar_arrive_expect_tx(&full[stage], 2 * kStageBytes);
            const uint32_t bar = map_rank(&full[stage], 0);
            if (p.hint) {
              tma_load_2sm_hint(sa, &map, kb * kKB, rowA, bar, policy);
              tma_load_2sm_hint(sa + kPanelBytes, &map, kb * kKB, rowB, bar, policy);
            } else {
              tma_load_2sm(sa, &map, kb * kKB, rowA, bar);
              tma_load_2sm(sa + kPanelBytes, &map, kb * kKB, rowB, bar);
            }
            if (++stage == kStages) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0 && lane == 0) {
      // ---- MMA issuer (leader CTA, one thread).
      uint32_t stage = 0, phase = 0, acc = 0, aphase = 0;
      unsigned long long w_empty = 0, w_full = 0, t_begin = clock64();
      for (int n = 0;; ++n) {
        const int r = n % kTaskRing;
        mbar_wait(&task_full[r], (n / kTaskRing) & 1);
        const int task = *reinterpret_cast<volatile int*>(&task_slot[r]);
        mbar_arrive(&task_empty[r]);
        if (task < 0) break;
        for (int t = 0; t < NM; ++t) {
          unsigned long long c0 = p.dbg ? clock64() : 0;
          if (p.pc_sleep) mbar_wait_sleep(&tempty[acc], aphase ^ 1, p.pc_sleep); else mbar_wait(&tempty[acc], aphase ^ 1);
          if (p.dbg) w_empty += clock64() - c0;
          tc_fence_after();
          const uint32_t d = tmem + acc * kAccCols;
          for (int kb = 0; kb < p.kblocks; ++kb) {
            if (p.dbg) c0 = clock64();
            if (p.pc_sleep) mbar_wait_sleep(&full[stage], phase, p.pc_sleep); else mbar_wait(&full[stage], phase);
            if (p.dbg) w_full += clock64() - c0;
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
      if (p.dbg) {
        atomicAdd(p.dbg + 0, w_empty);
        atomicAdd(p.dbg + 1, w_full);
        atomicAdd(p.dbg + 2, clock64() - t_begin);
      }
    }
  } else if (warp >= 4) {
    // ---- Epilogue (both CTAs): warp w reads TMEM lanes 32 (w % 4) .. +31
    // (this CTA's rows) and columns 128 ((w - 4) / 4) .. +127 of the tile.
    const int q = warp & 3;
    const int half = (warp - 4) >> 2;
    const int row = q * 32 + lane;  // row of this CTA's half tile
    const uint32_t tempty_leader0 = map_rank(&tempty[0], 0);
    const uint32_t tempty_leader1 = map_rank(&tempty[1], 0);
    // This thread's scratch row: modulus t at t * 128 * 256, 256 columns contiguous.
    uint8_t* srow = p.scratch + static_cast<size_t>(blockIdx.x) * NM * kHalf * kTile +
                    static_cast<size_t>(row) * kTile + half * (kTile / 2);
    uint32_t acc = 0, aphase = 0;
    const uint32_t lead_empty0 = map_rank(&task_empty[0], 0);
    for (int n = 0;; ++n) {
      const int r = n % kTaskRing;
      int task = 0;
      if (lane == 0) {
        mbar_wait_cluster(&task_full[r], (n / kTaskRing) & 1);
        task = *reinterpret_cast<volatile int*>(&task_slot[r]);
        mbar_arrive_remote(lead_empty0 + 8 * r);
      }
      task = __shfl_sync(0xffffffffu, task, 0);
      if (task < 0) break;
      int ti, tj;
      decode_task(p, task, ti, tj);
#pragma unroll 1
      for (int t = 0; t < NM; ++t) {
        const int mt = p.mod[t];
        const unsigned p16 = p.p16[t], off = p.off[t], magic = p.magic[t];
        if (p.sleep_ns)
          mbar_wait_sleep(&tfull[acc], aphase, p.sleep_ns);
        else
          mbar_wait(&tfull[acc], aphase);
        tc_fence_after();
        const uint32_t tbase =
            tmem + acc * kAccCols + half * (kAccCols / 2) + (static_cast<uint32_t>(q * 32) << 16);
        uint8_t* dst = srow + static_cast<size_t>(t) * kHalf * kTile;
#pragma unroll 1
        for (int ch = 0; ch < kAccCols / 64; ++ch) {
          uint32_t v[32];
          tmem_ld32(tbase + ch * 32, v);
          uint32_t w[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            uint32_t x = 0;
#pragma unroll
            for (int b = 0; b < 4; ++b) {
              const int r = sym_residue(static_cast<int>(v[4 * u + b]), mt, p16, off, magic);
              x |= (static_cast<uint32_t>(r) & 0xFFu) << (8 * b);
            }
            w[u] = x;
          }
          uint4* d4 = reinterpret_cast<uint4*>(dst + ch * 32);
          __stcg(d4, make_uint4(w[0], w[1], w[2], w[3]));
          __stcg(d4 + 1, make_uint4(w[4], w[5], w[6], w[7]));
        }
        // The accumulator is free as soon as its residues are out.
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
      // Fold the tile's NM residues of every entry of this thread's 128
      // columns into G while the MMAs of the next tile run.
      const int gi = ti * kTile + static_cast<int>(rank) * kHalf + row;
      const int ei = gi < p.n ? __ldg(p.ex + gi) : 0;
      const int gjb = tj * kTile + half * (kTile / 2);
#pragma unroll 1
      for (int ch = 0; ch < kTile / 64; ++ch) {
        const int gj0 = gjb + ch * 32;
        const int ej_lane = (gj0 + lane < p.n) ? __ldg(p.ex + gj0 + lane) : 0;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          uint4 wv[NM];
#pragma unroll
          for (int s2 = 0; s2 < NM; ++s2)
            wv[s2] = __ldcg(reinterpret_cast<const uint4*>(srow + static_cast<size_t>(s2) * kHalf * kTile +
                                                           ch * 32 + h * 16));
#pragma unroll
          for (int c = 0; c < 16; ++c) {
            const int cc = h * 16 + c;
            const int ej = __shfl_sync(0xffffffffu, ej_lane, cc);
            const int gj = gj0 + cc;
            if (gi >= gj && gi < p.n && gj < p.n) {
              int r[NM];
#pragma unroll
              for (int s2 = 0; s2 < NM; ++s2) {
                const uint32_t word = (c < 4) ? wv[s2].x : (c < 8) ? wv[s2].y : (c < 12) ? wv[s2].z : wv[s2].w;
                r[s2] = sext_byte(word, c & 3);
              }
              const double v0 = crt_scale(crt_value<NM, true>(r), ei + ej - 2 * p.k);
              const double val = p.negate ? -v0 : v0;
              double* g = p.G + gi + static_cast<long long>(gj) * p.ldg;
              *g = p.accumulate ? *g + val : val;
            }
          }
        }
      }
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

// ---- Unfused variants ("permod", "block"): one launch per column block
// [c0, c0 + wn) of the lower triangle, task = (modulus, tile) with the
// modulus outermost (the library GEMMs' order), symmetric residues stored
// as bytes into C (column-major, ld m, plane stride cstride); the Garner
// fold then runs as crt_fold_kernel<NM, int8_t> (fstk_gram.cu).
struct ResParams {
  int nm, kblocks, np, c0, ntj, nti, tri, per_mod, ntasks;
  int plane0;           // first plane (modulus) of this launch
  int* counter;         // dynamic tile scheduler (zeroed before the launch)
  unsigned long long* dbg;  // optional MMA-thread wait counters ($FSTK_SYRK_DEBUG)
  int hint_a, hint_b;   // L2 policy of the A / B panel loads: 0 none, 1 evict_last, 2 evict_first, 3 evict_normal
  long long ldc, cstride;
  int8_t* C;
  unsigned pc_sleep;
  int mod[kSyrkMaxModuli];
  unsigned p16[kSyrkMaxModuli], off[kSyrkMaxModuli], magic[kSyrkMaxModuli];
};

__device__ __forceinline__ void decode_res(const ResParams& p, int task, int& t, int& ti, int& tj) {
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

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 1)
    syrk_res_kernel(const __grid_constant__ CUtensorMap map, const ResParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint64_t* tempty = tfull + 2;
  uint64_t* task_full = tempty + 2;              // dynamic scheduler, as syrk_crt_kernel
  uint64_t* task_empty = task_full + kTaskRing;  // leader: MMA + peer producer + 8 epilogue warps
  int* task_slot = reinterpret_cast<int*>(task_empty + kTaskRing);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(task_slot + kTaskRing);
  const uint32_t rank = cluster_rank();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0)
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map)) : "memory");
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 8);
    }
    for (int r = 0; r < kTaskRing; ++r) {
      mbar_init(&task_full[r], 1);
      mbar_init(&task_empty[r], 2 + 8);
    }
    fence_mbar_init();
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
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
      uint32_t stage = 0, phase = 0;
      uint64_t pl = 0, pf = 0, pn = 0;
      asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pl));
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pf));
      asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pn));
      const uint64_t pol_a = p.hint_a == 1 ? pl : p.hint_a == 2 ? pf : pn;
      const uint64_t pol_b = p.hint_b == 1 ? pl : p.hint_b == 2 ? pf : pn;
      const uint32_t peer_slot0 = map_rank(&task_slot[0], 1);
      const uint32_t peer_full0 = map_rank(&task_full[0], 1);
      const uint32_t lead_empty0 = map_rank(&task_empty[0], 0);
      for (int n = 0;; ++n) {
        const int r = n % kTaskRing;
        const uint32_t rph = (n / kTaskRing) & 1;
        int task;
        if (rank == 0) {
          mbar_wait(&task_empty[r], rph ^ 1);
          task = atomicAdd(p.counter, 1);
          if (task >= p.ntasks) task = -1;
          task_slot[r] = task;
          st_cluster_s32(peer_slot0 + 4 * r, task);
          mbar_arrive(&task_full[r]);
          mbar_arrive_remote(peer_full0 + 8 * r);
        } else {
          mbar_wait_cluster(&task_full[r], rph);
          task = *reinterpret_cast<volatile int*>(&task_slot[r]);
          mbar_arrive_remote(lead_empty0 + 8 * r);
        }
        if (task < 0) break;
        int t, ti, tj;
        decode_res(p, task, t, ti, tj);
        const int base = (p.plane0 + t) * p.np + p.c0 + static_cast<int>(rank) * kHalf;
        for (int kb = 0; kb < p.kblocks; ++kb) {
          if (p.pc_sleep) mbar_wait_sleep(&empty[stage], phase ^ 1, p.pc_sleep); else mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * kStageBytes;
          if (rank == 0) mbar_arrive_expect_tx(&full[stage], 2 * kStageBytes);
          const uint32_t bar = map_rank(&full[stage], 0);
          if (p.hint_a) tma_load_2sm_hint(sa, &map, kb * kKB, base + ti * kTile, bar, pol_a);
          else tma_load_2sm(sa, &map, kb * kKB, base + ti * kTile, bar);
          if (p.hint_b) tma_load_2sm_hint(sa + kPanelBytes, &map, kb * kKB, base + tj * kTile, bar, pol_b);
          else tma_load_2sm(sa + kPanelBytes, &map, kb * kKB, base + tj * kTile, bar);
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0 && lane == 0) {
      uint32_t stage = 0, phase = 0, acc = 0, aphase = 0;
      unsigned long long w_empty = 0, w_full = 0, c0 = 0;
      const unsigned long long t_begin = clock64();
      for (int n = 0;; ++n) {
        const int r = n % kTaskRing;
        mbar_wait(&task_full[r], (n / kTaskRing) & 1);
        const int task = *reinterpret_cast<volatile int*>(&task_slot[r]);
        mbar_arrive(&task_empty[r]);
        if (task < 0) break;
        if (p.dbg) c0 = clock64();
        if (p.pc_sleep) mbar_wait_sleep(&tempty[acc], aphase ^ 1, p.pc_sleep); else mbar_wait(&tempty[acc], aphase ^ 1);
        if (p.dbg) w_empty += clock64() - c0;
        tc_fence_after();
        const uint32_t d = tmem + acc * kAccCols;
        for (int kb = 0; kb < p.kblocks; ++kb) {
          if (p.dbg) c0 = clock64();
          if (p.pc_sleep) mbar_wait_sleep(&full[stage], phase, p.pc_sleep); else mbar_wait(&full[stage], phase);
          if (p.dbg) w_full += clock64() - c0;
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * kStageBytes);
          const uint64_t da = sw128_desc(sa), db = sw128_desc(sa + kPanelBytes);
#pragma unroll
          for (int k = 0; k < kKB / 32; ++k) mma_i8(d, da + 2 * k, db + 2 * k, (kb | k) != 0 ? 1u : 0u);
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
      if (p.dbg) {
        atomicAdd(p.dbg + 0, w_empty);
        atomicAdd(p.dbg + 1, w_full);
        atomicAdd(p.dbg + 2, clock64() - t_begin);
      }
    }
  } else if (warp >= 4) {
    const int q = warp & 3;
    const uint32_t te0 = map_rank(&tempty[0], 0), te1 = map_rank(&tempty[1], 0);
    uint32_t acc = 0, aphase = 0;
    const uint32_t lead_empty0 = map_rank(&task_empty[0], 0);
    for (int n = 0;; ++n) {
      const int r = n % kTaskRing;
      int task = 0;
      if (lane == 0) {
        mbar_wait_cluster(&task_full[r], (n / kTaskRing) & 1);
        task = *reinterpret_cast<volatile int*>(&task_slot[r]);
        mbar_arrive_remote(lead_empty0 + 8 * r);
      }
      task = __shfl_sync(0xffffffffu, task, 0);
      if (task < 0) break;
      int t, ti, tj;
      decode_res(p, task, t, ti, tj);
      const int mt = p.mod[t];
      const unsigned p16 = p.p16[t], off = p.off[t], magic = p.magic[t];
      const long long i = static_cast<long long>(ti) * kTile + rank * kHalf + q * 32 + lane;
      int8_t* crow = p.C + t * p.cstride + i + static_cast<long long>(tj) * kTile * p.ldc;
      mbar_wait_sleep(&tfull[acc], aphase);
      tc_fence_after();
      const uint32_t tbase = tmem + acc * kAccCols + (static_cast<uint32_t>(q * 32) << 16);
#pragma unroll 1
      for (int ch = 0; ch < kAccCols / 32; ++ch) {
        uint32_t v[32];
        tmem_ld32(tbase + ch * 32, v);
#pragma unroll
        for (int c = 0; c < 32; ++c)
          crow[static_cast<long long>(ch * 32 + c) * p.ldc] =
              static_cast<int8_t>(sym_residue(static_cast<int>(v[c]), mt, p16, off, magic));
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0)
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(acc ? te1 : te0) : "memory");
      acc ^= 1;
      if (acc == 0) aphase ^= 1;
    }
  }
  __syncwarp();
  tc_fence_before();
  cluster_sync_all();
  if (warp == 2)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * kAccCols) : "memory");
}

// ---- Two CTA pairs per cluster ($FSTK_SYRK_CLUSTER=4): the pairs compute
// the tiles (2 rp, tj) and (2 rp + 1, tj), which share their B panel, so
// each CTA loads its A half (16 KB per stage) and half of its B half (8 KB)
// and multicasts the latter to the same-parity CTA of the other pair --
// 24 KB of L2-to-SM traffic per CTA and stage instead of 32.  Stage slots
// are written by both pairs, so every CTA's empty barrier waits for both
// pair leaders' MMA commits (multicast to all four CTAs).
__device__ __forceinline__ void tma_load_2sm_mc(void* dst, const CUtensorMap* map, int x, int y, uint32_t bar,
                                                uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      ".multicast::cluster [%0], [%1, {%4, %5}], [%2], %3;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "h"(mask), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void mma_commit_mask(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"(mask)
      : "memory");
}
__device__ __forceinline__ void cluster4_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// Cluster task -> (modulus, tile-row pair rp, tile column tj): per modulus,
// row pairs in order, columns tj < min(2 rp + 2, ntj) fastest.
__device__ __forceinline__ void decode_res4(const ResParams& p, int task, int& t, int& rp, int& tj) {
  t = task / p.per_mod;
  int r = task - t * p.per_mod;
  rp = 0;
  for (;;) {
    const int cnt = min(2 * rp + 2, p.ntj);
    if (r < cnt) break;
    r -= cnt;
    ++rp;
  }
  tj = r;
}

__global__ void __launch_bounds__(256, 1) syrk_res4_kernel(const __grid_constant__ CUtensorMap mapA,
                                                           const __grid_constant__ CUtensorMap mapB,
                                                           const ResParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint64_t* tempty = tfull + 2;
  uint64_t* task_full = tempty + 2;
  uint64_t* task_empty = task_full + kTaskRing;  // rank 0: 2 MMA + 3 producers + 16 epilogue warps
  int* task_slot = reinterpret_cast<int*>(task_empty + kTaskRing);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(task_slot + kTaskRing);
  const uint32_t crank = cluster_rank();  // 0..3
  const uint32_t pair = crank >> 1, prank = crank & 1, lead = crank & ~1u;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapB)) : "memory");
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 2);  // both pair leaders' commits
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 8);
    }
    for (int r = 0; r < kTaskRing; ++r) {
      mbar_init(&task_full[r], 1);
      mbar_init(&task_empty[r], 2 + 3 + 16);
    }
    fence_mbar_init();
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(2 * kAccCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster4_sync_all();
  tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(tmem_slot);
  const uint32_t lead_empty0 = map_rank(&task_empty[0], 0);
  if (warp == 0) {
    if (lane == 0) {
      uint32_t stage = 0, phase = 0;
      const uint16_t bmask = static_cast<uint16_t>((1u << prank) | (1u << (prank + 2)));
      for (int n = 0;; ++n) {
        const int r = n % kTaskRing;
        const uint32_t rph = (n / kTaskRing) & 1;
        int task;
        if (crank == 0) {
          mbar_wait(&task_empty[r], rph ^ 1);
          task = atomicAdd(p.counter, 1);
          if (task >= p.ntasks) task = -1;
          task_slot[r] = task;
          for (uint32_t q = 1; q < 4; ++q) st_cluster_s32(map_rank(&task_slot[r], q), task);
          mbar_arrive(&task_full[r]);
          for (uint32_t q = 1; q < 4; ++q) mbar_arrive_remote(map_rank(&task_full[r], q));
        } else {
          mbar_wait_cluster(&task_full[r], rph);
          task = *reinterpret_cast<volatile int*>(&task_slot[r]);
          mbar_arrive_remote(lead_empty0 + 8 * r);
        }
        if (task < 0) break;
        int t, rp, tj;
        decode_res4(p, task, t, rp, tj);
        int ti = 2 * rp + static_cast<int>(pair);
        if (ti >= p.nti) ti = 2 * rp;  // odd tile-row count: a duplicate tile, not stored
        const int plane = (p.plane0 + t) * p.np + p.c0;
        const int rowA = plane + ti * kTile + static_cast<int>(prank) * kHalf;
        const int rowB = plane + tj * kTile + static_cast<int>(prank) * kHalf + static_cast<int>(pair) * (kHalf / 2);
        for (int kb = 0; kb < p.kblocks; ++kb) {
          if (p.pc_sleep) mbar_wait_sleep(&empty[stage], phase ^ 1, p.pc_sleep); else mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * kStageBytes;
          if (prank == 0) mbar_arrive_expect_tx(&full[stage], 2 * kStageBytes);
          tma_load_2sm(sa, &mapA, kb * kKB, rowA, map_rank(&full[stage], lead));
          tma_load_2sm_mc(sa + kPanelBytes + pair * (kPanelBytes / 2), &mapB, kb * kKB, rowB,
                          smem_u32(&full[stage]) & 0xFEFFFFFFu, bmask);
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (prank == 0 && lane == 0) {
      uint32_t stage = 0, phase = 0, acc = 0, aphase = 0;
      const uint16_t pmask = static_cast<uint16_t>(3u << crank);
      for (int n = 0;; ++n) {
        const int r = n % kTaskRing;
        if (crank == 0) {
          mbar_wait(&task_full[r], (n / kTaskRing) & 1);
        } else {
          mbar_wait_cluster(&task_full[r], (n / kTaskRing) & 1);
        }
        const int task = *reinterpret_cast<volatile int*>(&task_slot[r]);
        if (crank == 0) mbar_arrive(&task_empty[r]); else mbar_arrive_remote(lead_empty0 + 8 * r);
        if (task < 0) break;
        if (p.pc_sleep) mbar_wait_sleep(&tempty[acc], aphase ^ 1, p.pc_sleep); else mbar_wait(&tempty[acc], aphase ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + acc * kAccCols;
        for (int kb = 0; kb < p.kblocks; ++kb) {
          if (p.pc_sleep) mbar_wait_sleep(&full[stage], phase, p.pc_sleep); else mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * kStageBytes);
          const uint64_t da = sw128_desc(sa), db = sw128_desc(sa + kPanelBytes);
#pragma unroll
          for (int k = 0; k < kKB / 32; ++k) mma_i8(d, da + 2 * k, db + 2 * k, (kb | k) != 0 ? 1u : 0u);
          mma_commit_mask(&empty[stage], static_cast<uint16_t>(0xF));
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        mma_commit_mask(&tfull[acc], pmask);
        acc ^= 1;
        if (acc == 0) aphase ^= 1;
      }
    }
  } else if (warp >= 4) {
    const int q = warp & 3;
    const uint32_t te0 = map_rank(&tempty[0], lead), te1 = map_rank(&tempty[1], lead);
    uint32_t acc = 0, aphase = 0;
    for (int n = 0;; ++n) {
      const int r = n % kTaskRing;
      int task = 0;
      if (lane == 0) {
        mbar_wait_cluster(&task_full[r], (n / kTaskRing) & 1);
        task = *reinterpret_cast<volatile int*>(&task_slot[r]);
        mbar_arrive_remote(lead_empty0 + 8 * r);
      }
      task = __shfl_sync(0xffffffffu, task, 0);
      if (task < 0) break;
      int t, rp, tj;
      decode_res4(p, task, t, rp, tj);
      const int ti = 2 * rp + static_cast<int>(pair);
      const bool store = ti < p.nti;
      const int mt = p.mod[t];
      const unsigned p16 = p.p16[t], off = p.off[t], magic = p.magic[t];
      const long long i = static_cast<long long>(ti) * kTile + prank * kHalf + q * 32 + lane;
      int8_t* crow = p.C + t * p.cstride + i + static_cast<long long>(tj) * kTile * p.ldc;
      mbar_wait_sleep(&tfull[acc], aphase);
      tc_fence_after();
      const uint32_t tbase = tmem + acc * kAccCols + (static_cast<uint32_t>(q * 32) << 16);
#pragma unroll 1
      for (int ch = 0; ch < kAccCols / 32; ++ch) {
        uint32_t v[32];
        tmem_ld32(tbase + ch * 32, v);
        if (store) {
#pragma unroll
          for (int c = 0; c < 32; ++c)
            crow[static_cast<long long>(ch * 32 + c) * p.ldc] =
                static_cast<int8_t>(sym_residue(static_cast<int>(v[c]), mt, p16, off, magic));
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0)
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(acc ? te1 : te0) : "memory");
      acc ^= 1;
      if (acc == 0) aphase ^= 1;
    }
  }
  __syncwarp();
  tc_fence_before();
  cluster4_sync_all();
  if (warp == 2)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * kAccCols) : "memory");
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

int sm_count(int device) {
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

template <int NM>
void launch_syrk(const CUtensorMap& map, const SyrkParams& p, int pairs, int device, cudaStream_t s) {
  static std::atomic<uint64_t> attr_set{0};
  const uint64_t bit = uint64_t(1) << (device & 63);
  if (!(attr_set.load() & bit)) {
    cudaFuncSetAttribute(syrk_crt_kernel<NM>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    attr_set.fetch_or(bit);
  }
  syrk_crt_kernel<NM><<<2 * pairs, kThreads, kSmemBytes, s>>>(map, p);
  check_launch("syrk_crt_kernel");
}

}  // namespace

// Variant of the tcgen05 SYRK ($FSTK_SYRK_MODE): 0 "permod" (default): one
// launch per column block and modulus, residues to C, separate byte fold;
// 1 "block": one launch per column block with every modulus; 2 "fused":
// one launch per segment with the fold in the epilogue.
int syrk_mode() {
  static const int mode = [] {
    const char* e = std::getenv("FSTK_SYRK_MODE");
    if (!e) return 0;
    const std::string v(e);
    return v == "fused" ? 2 : v == "block" ? 1 : 0;
  }();
  return mode;
}
bool syrk_fused() { return syrk_mode() == 2; }

static double syrk_res_launch(const int8_t* planes, int nm, int t0, int cnt, int64_t kp, int64_t np, int64_t c0,
                              int64_t wn, int64_t m, int8_t* C, int64_t cstride, int* counter, int device,
                              cudaStream_t s);
double syrk_i8_residues(const int8_t* planes, int nm, int64_t kp, int64_t np, int64_t c0, int64_t wn,
                        int64_t m, int8_t* C, int64_t cstride, int* counter, int device, cudaStream_t s) {
  return syrk_res_launch(planes, nm, 0, nm, kp, np, c0, wn, m, C, cstride, counter, device, s);
}
double syrk_i8_residues_one(const int8_t* planes, int nm, int t, int64_t kp, int64_t np, int64_t c0, int64_t wn,
                            int64_t m, int8_t* C, int* counter, int device, cudaStream_t s) {
  return syrk_res_launch(planes, nm, t, 1, kp, np, c0, wn, m, C, 0, counter, device, s);
}
static double syrk_res_launch(const int8_t* planes, int nm, int t0, int cnt, int64_t kp, int64_t np, int64_t c0,
                              int64_t wn, int64_t m, int8_t* C, int64_t cstride, int* counter, int device,
                              cudaStream_t s) {
  require(nm >= 1 && nm <= kSyrkMaxModuli, FSTK_E_COMPUTE, "internal: SYRK modulus count");
  require(kp % kKB == 0 && kp > 0 && kp <= 66560, FSTK_E_COMPUTE, "internal: SYRK segment rows");
  require(np % kTile == 0 && c0 % kTile == 0 && wn % kTile == 0 && m % kTile == 0 && c0 + m == np,
          FSTK_E_COMPUTE, "internal: SYRK block shape");
  static std::atomic<uint64_t> attr_set{0};
  const uint64_t bit = uint64_t(1) << (device & 63);
  if (!(attr_set.load() & bit)) {
    cudaFuncSetAttribute(syrk_res_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    attr_set.fetch_or(bit);
  }
  CUtensorMap map;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(kp), static_cast<cuuint64_t>(nm * np)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(kp)};
  const cuuint32_t box[2] = {kKB, kHalf};
  const cuuint32_t estr[2] = {1, 1};
  int promo = 2;
  ResParams p{};
  p.nm = cnt;
  p.kblocks = static_cast<int>(kp / kKB);
  p.np = static_cast<int>(np);
  p.c0 = static_cast<int>(c0);
  p.ntj = static_cast<int>(wn / kTile);
  p.nti = static_cast<int>(m / kTile);
  p.tri = p.ntj * (p.ntj + 1) / 2;
  p.per_mod = p.tri + (p.nti - p.ntj) * p.ntj;
  p.ntasks = cnt * p.per_mod;
  p.ldc = m;
  p.cstride = cstride;
  p.C = C;
  p.plane0 = t0;
  p.counter = counter;
  FSTK_CUDA(cudaMemsetAsync(counter, 0, sizeof(int), s));
  const char* e = std::getenv("FSTK_SYRK_PC_SLEEP");
  p.pc_sleep = e ? static_cast<unsigned>(std::atoi(e)) : 200000u;
  const char* hh = std::getenv("FSTK_SYRK_HINTS");
  if (hh && std::strlen(hh) >= 3) {
    p.hint_a = hh[0] - '0';
    p.hint_b = hh[2] - '0';
  }
  const char* pr = std::getenv("FSTK_SYRK_PROMO");
  promo = pr ? std::atoi(pr) : 2;
  for (int t = 0; t < cnt; ++t) {
    const unsigned mm = static_cast<unsigned>(kmod(t0 + t));
    p.mod[t] = kmod(t0 + t);
    p.p16[t] = 65536u % mm;
    p.off[t] = ((1u << 22) / mm + 1u) * mm;
    p.magic[t] = static_cast<unsigned>((uint64_t(1) << 32) / mm);
  }
  const CUtensorMapL2promotion promos[4] = {CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_64B,
                                             CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B};
  if (tensor_map_encoder()(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<int8_t*>(planes), dims, strides, box,
                           estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, promos[promo & 3],
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    fail(FSTK_E_COMPUTE, "cuTensorMapEncodeTiled failed for the SYRK planes");
  static const bool debug = std::getenv("FSTK_SYRK_DEBUG") != nullptr;
  static unsigned long long* dbg = nullptr;  // accumulated over launches; printed by the caller's tool
  if (debug && !dbg) {
    FSTK_CUDA(cudaMalloc(&dbg, 32));
    FSTK_CUDA(cudaMemset(dbg, 0, 32));
  }
  p.dbg = debug ? dbg : nullptr;
  static const int cluster = [] {
    const char* e = std::getenv("FSTK_SYRK_CLUSTER");
    return (e && std::atoi(e) == 4) ? 4 : 2;
  }();
  if (cluster == 4) {
    // Cluster tasks: tile-row pairs x tile columns (the two pairs share tj).
    int per = 0;
    for (int rp = 0; 2 * rp < p.nti; ++rp) per += std::min(2 * rp + 2, p.ntj);
    p.per_mod = per;
    p.ntasks = cnt * per;
    CUtensorMap mapB;
    const cuuint32_t boxB[2] = {kKB, kHalf / 2};
    if (tensor_map_encoder()(&mapB, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<int8_t*>(planes), dims, strides,
                             boxB, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, promos[promo & 3],
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      fail(FSTK_E_COMPUTE, "cuTensorMapEncodeTiled failed for the SYRK B planes");
    static std::atomic<uint64_t> attr4{0};
    const uint64_t bit = uint64_t(1) << (device & 63);
    if (!(attr4.load() & bit)) {
      cudaFuncSetAttribute(syrk_res4_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
      attr4.fetch_or(bit);
    }
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 4;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = kSmemBytes;
    cfg.stream = s;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    static int max_clusters[64] = {0};
    int& mc = max_clusters[device & 63];
    if (!mc) {
      cfg.gridDim = dim3(4 * (sm_count(device) / 4));
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, syrk_res4_kernel, &cfg) != cudaSuccess || n < 1) {
        cudaGetLastError();
        n = sm_count(device) / 4;
      }
      mc = n;
    }
    cfg.gridDim = dim3(4 * std::max(1, std::min(p.ntasks, mc)));
    FSTK_CUDA(cudaLaunchKernelEx(&cfg, syrk_res4_kernel, map, mapB, p));
    check_launch("syrk_res4_kernel");
    return 2.0 * static_cast<double>(p.ntasks) * 2 * kTile * kTile * static_cast<double>(kp);
  }
  const int pairs = std::max(1, std::min(p.ntasks, sm_count(device) / 2));
  syrk_res_kernel<<<2 * pairs, 256, kSmemBytes, s>>>(map, p);
  check_launch("syrk_res_kernel");
  if (debug && c0 + wn == np && t0 + cnt == nm) {  // last launch of a segment: report
    unsigned long long h[4];
    FSTK_CUDA(cudaMemcpyAsync(h, dbg, 32, cudaMemcpyDeviceToHost, s));
    FSTK_CUDA(cudaStreamSynchronize(s));
    std::fprintf(stderr, "syrk_res: MMA thread cycles %.3g, waiting tempty %.1f%%, waiting full %.1f%%\n",
                 double(h[2]), 100.0 * h[0] / double(h[2]), 100.0 * h[1] / double(h[2]));
    FSTK_CUDA(cudaMemsetAsync(dbg, 0, 32, s));
  }
  return 2.0 * static_cast<double>(p.ntasks) * kTile * kTile * static_cast<double>(kp);
}

size_t syrk_crt_scratch_bytes(int nm, int device) {
  return static_cast<size_t>(sm_count(device)) * nm * kHalf * kTile + 256;  // + the task counter
}

double syrk_crt_fold(const int8_t* planes, int nm, int64_t kp, int64_t np, int n, int k, const int* ex,
                     double* G, int64_t ldg, bool accumulate, bool negate, uint8_t* scratch, int device,
                     cudaStream_t s) {
  require(nm >= 8 && nm <= 17, FSTK_E_COMPUTE, "internal: SYRK modulus count");
  require(kp % kKB == 0 && kp > 0 && kp <= 66560, FSTK_E_COMPUTE, "internal: SYRK segment rows");
  require(np % kTile == 0 && np >= n && n > 0, FSTK_E_COMPUTE, "internal: SYRK plane shape");
  require(static_cast<int64_t>(nm) * np < (int64_t(1) << 31), FSTK_E_COMPUTE,
          "internal: SYRK plane rows exceed the tensor-map range");
  const int nt = static_cast<int>(np / kTile);
  static const int band = [] {
    const char* e = std::getenv("FSTK_SYRK_BAND");
    return e ? std::max(1, std::atoi(e)) : kBandTilesDefault;
  }();
  const int nbands = (nt + band - 1) / band;
  require(nbands <= kMaxBands && band <= 64, FSTK_E_COMPUTE, "internal: SYRK Gram too wide (> 131072 columns)");
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
  p.kblocks = static_cast<int>(kp / kKB);
  p.np = static_cast<int>(np);
  p.nt = nt;
  p.nbands = nbands;
  p.band = band;
  int task = 0;
  for (int b = 0; b < nbands; ++b) {
    p.band_start[b] = task;
    const int wb = std::min(band, nt - b * band);
    task += wb * (wb + 1) / 2 + (nt - b * band - wb) * wb;
  }
  p.band_start[nbands] = task;
  p.ntasks = task;
  p.n = n;
  p.k = k;
  p.accumulate = accumulate ? 1 : 0;
  p.negate = negate ? 1 : 0;
  static const int hint = [] {
    const char* e = std::getenv("FSTK_SYRK_HINT");
    return e ? std::atoi(e) : 0;
  }();
  p.hint = hint;
  p.ldg = ldg;
  p.G = G;
  p.ex = ex;
  p.scratch = scratch;
  static const int lookahead = [] {
    const char* e = std::getenv("FSTK_SYRK_LOOKAHEAD");
    return e ? std::atoi(e) : 0;
  }();
  p.lookahead = lookahead;
  p.counter = reinterpret_cast<int*>(scratch + static_cast<size_t>(sm_count(device)) * nm * kHalf * kTile);
  FSTK_CUDA(cudaMemsetAsync(p.counter, 0, sizeof(int), s));
  for (int t = 0; t < nm; ++t) {
    const unsigned m = static_cast<unsigned>(kmod(t));
    p.mod[t] = kmod(t);
    p.p16[t] = 65536u % m;
    p.off[t] = ((1u << 22) / m + 1u) * m;
    p.magic[t] = static_cast<unsigned>((uint64_t(1) << 32) / m);
  }
  static const bool debug = std::getenv("FSTK_SYRK_DEBUG") != nullptr;
  static const unsigned sleep_ns = [] {
    const char* e = std::getenv("FSTK_SYRK_SLEEP_NS");
    return e ? static_cast<unsigned>(std::atoi(e)) : 500000u;
  }();
  p.sleep_ns = sleep_ns;
  static const unsigned pc_sleep = [] {
    const char* e = std::getenv("FSTK_SYRK_PC_SLEEP");
    return e ? static_cast<unsigned>(std::atoi(e)) : 200000u;
  }();
  p.pc_sleep = pc_sleep;
  DevBuf<unsigned long long> dbg;
  if (debug) {
    dbg.alloc(4);
    FSTK_CUDA(cudaMemsetAsync(dbg.p, 0, 32, s));
    p.dbg = dbg.p;
  }
  const int pairs = std::max(1, std::min(p.ntasks, sm_count(device) / 2));
  switch (nm) {
    case 8: launch_syrk<8>(map, p, pairs, device, s); break;
    case 9: launch_syrk<9>(map, p, pairs, device, s); break;
    case 10: launch_syrk<10>(map, p, pairs, device, s); break;
    case 11: launch_syrk<11>(map, p, pairs, device, s); break;
    case 12: launch_syrk<12>(map, p, pairs, device, s); break;
    case 13: launch_syrk<13>(map, p, pairs, device, s); break;
    case 14: launch_syrk<14>(map, p, pairs, device, s); break;
    case 15: launch_syrk<15>(map, p, pairs, device, s); break;
    case 16: launch_syrk<16>(map, p, pairs, device, s); break;
    case 17: launch_syrk<17>(map, p, pairs, device, s); break;
    default: fail(FSTK_E_COMPUTE, "internal: unsupported CRT modulus count");
  }
  if (debug) {
    unsigned long long h[4];
    FSTK_CUDA(cudaMemcpyAsync(h, dbg.p, 32, cudaMemcpyDeviceToHost, s));
    FSTK_CUDA(cudaStreamSynchronize(s));
    std::fprintf(stderr, "syrk: MMA thread cycles total %.3g, waiting tempty %.1f%%, waiting full %.1f%%\n",
                 double(h[2]), 100.0 * h[0] / double(h[2]), 100.0 * h[1] / double(h[2]));
  }
  return 2.0 * static_cast<double>(p.ntasks) * nm * kTile * kTile * static_cast<double>(kp);
}

}  // namespace fstk_gpu

// Measurement entry (no reference counterpart): the unfused tcgen05 SYRK
// alone on device planes (nm planes of kp x np int8), whole lower triangle
// into C (np x np x nm bytes).
extern "C" int32_t fstk_gpu_debug_syrk(const int8_t* planes, int32_t nm, int64_t kp, int64_t np, int8_t* c,
                                       int32_t device, void* stream, fstk_gpu_error* err) {
  using namespace fstk_gpu;
  return guarded(err, [&] {
    DeviceGuard dg(device);
    DevBuf<int> counter(1);
    syrk_i8_residues(planes, nm, kp, np, 0, np, np, c, np * np, counter.p, device, static_cast<cudaStream_t>(stream));
    FSTK_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
  });
}
