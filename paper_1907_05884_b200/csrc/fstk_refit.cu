// fstk B200 library — randomized least-squares core refit (sm_100a).
//
// Replaces, on the GPU, reestimate_core (proj/src/randls.cpp:360-383):
//   prepare (:246-311)            host: bit-exact RNG bookkeeping (mt19937_64,
//                                 rng.cpp:11-61); device: gathers + mode tables
//                                 written directly in the mixing transform's
//                                 input order (Makhoul + bit-reversal for DCT,
//                                 bit-reversal for FFT, natural for WHT);
//   solve_sketched (:315-348)     device: per design column (and the rhs) the
//                                 value x_i = s_i * ((u0 u1) u2 ...) is generated
//                                 on the fly (W never exists), mixed by a
//                                 radix-2 transform that replays the reference
//                                 butterflies bit for bit (recurrence twiddles
//                                 transforms.cpp:36-46 replayed on the host, no
//                                 FMA contraction), in passes of <= 10 stages
//                                 held in shared memory, and only the S sampled
//                                 rows are written (scaled, DCT post-rotation
//                                 fused) into A;
//   solve_system (:112-123)       A^T A on the int8 tensor cores (exact CRT
//                                 residue products: the hand-written tcgen05
//                                 SYRK of fstk_syrk.cu with its Garner fold,
//                                 fstk_gram.cu; native fp64 DSYRK only as the
//                                 escalation fallback) and A^T b (DGEMV), a
//                                 Cholesky factor (blocked, int8 trailing
//                                 updates; timed separately) refined against A
//                                 itself to the least-squares solution; the
//                                 rank decision and minimum-norm solution of a
//                                 deficient system follow the reference's
//                                 ColPivHouseholderQR + COD (fstk_rank.cu);
//   relative_residual (:350-356)  device evaluation of the validation points.
#include <cublas_v2.h>
#include <cusolverDn.h>

#include <algorithm>
#include <chrono>
#include <climits>
#include <cmath>
#include <complex>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <numeric>
#include <random>
#include <thread>
#include <vector>

#include "fstk_internal.h"

namespace fstk_gpu {

// ------------------------------------------------------------- host RNG ---
// proj/include/fstk/rng.hpp:21-48, proj/src/rng.cpp:11-61 (std::mt19937_64
// is bit-exact by the C++ standard; the draws on top are spelled out).
struct Rng {
  std::mt19937_64 engine;
  explicit Rng(uint64_t seed) : engine(seed) {}
  uint64_t next_u64() { return engine(); }
  uint64_t uniform_index(uint64_t n) {
    require(n > 0, FSTK_E_PARAMETER, "uniform_index: n must be positive");
    // rng.cpp rejects x >= limit = UINT64_MAX - UINT64_MAX % n.  For n < 2^32
    // the limit exceeds 2^64 - 2^32, so a draw below that is accepted without
    // the second 64-bit division (all but one draw in 4e9): same decisions.
    if (n <= 0xffffffffull) {
      const uint64_t x0 = next_u64();
      if (x0 < 0xffffffff00000000ull) return x0 % n;
      const uint64_t limit0 = UINT64_MAX - UINT64_MAX % n;
      if (x0 < limit0) return x0 % n;
    }
    const uint64_t limit = UINT64_MAX - UINT64_MAX % n;
    uint64_t x;
    do {
      x = next_u64();
    } while (x >= limit);
    return x % n;
  }
  double sign() { return (next_u64() & 1ull) ? -1.0 : 1.0; }
  // rng.cpp sample_without_replacement: a partial Fisher-Yates shuffle of
  // [0, n) (swap i with i + uniform_index(n - i) for i < k), first k sorted.
  // Replayed with O(k) state -- positions [0, k) in a dense array, displaced
  // positions >= k in an open-addressing map -- so the same draws give the
  // same sample without materialising n indices; sorted by a bitmap over
  // [0, n) when that is cheaper than a comparison sort.
  std::vector<uint64_t> sample_without_replacement(uint64_t n, uint64_t k) {
    if (k >= n) {
      std::vector<uint64_t> all(n);
      std::iota(all.begin(), all.end(), 0);
      return all;
    }
    std::vector<uint64_t> pre(k);
    std::iota(pre.begin(), pre.end(), 0);
    int bits = 4;
    while ((uint64_t(1) << bits) < 2 * k) ++bits;
    const uint64_t cap = uint64_t(1) << bits, mask = cap - 1;
    constexpr uint64_t kEmpty = ~uint64_t(0);
    std::vector<std::pair<uint64_t, uint64_t>> tab(cap, {kEmpty, 0});
    auto home = [&](uint64_t key) { return (key * 0x9e3779b97f4a7c15ull) >> (64 - bits); };
    auto slot = [&](uint64_t key) -> std::pair<uint64_t, uint64_t>& {
      uint64_t h = home(key);
      while (tab[h].first != kEmpty && tab[h].first != key) h = (h + 1) & mask;
      return tab[h];
    };
    // The draws depend on the generator alone, not on the table: they are
    // made first, so the table slot (or dense entry) each swap will touch can
    // be prefetched a few swaps ahead.  The 2^21-entry table of a 2^20-row
    // working subset is 32 MB of random accesses: 47 -> 15 ms at C2.
    // Large samples: a second host thread makes the draws (generator and two
    // 64-bit divisions each) while this one applies the swaps behind it.
    std::vector<uint64_t> js(k);
    std::atomic<uint64_t> drawn{0};
    constexpr uint64_t kChunk = uint64_t(1) << 14;
    auto draw_all = [&] {
      for (uint64_t i = 0; i < k; ++i) {
        js[i] = i + uniform_index(n - i);
        if (((i + 1) & (kChunk - 1)) == 0) drawn.store(i + 1, std::memory_order_release);
      }
      drawn.store(k, std::memory_order_release);
    };
    std::thread drawer;
    if (k >= (uint64_t(1) << 17))
      drawer = std::thread(draw_all);
    else
      draw_all();
    struct Join {
      std::thread& t;
      ~Join() {
        if (t.joinable()) t.join();
      }
    } join{drawer};
    constexpr uint64_t kAhead = 16;
    uint64_t ready = 0;
    for (uint64_t i = 0; i < k; ++i) {
      // draws [0, ready) are published; the prefetch below looks kAhead ahead
      while (ready < std::min(k, i + kAhead + 1)) {
        ready = drawn.load(std::memory_order_acquire);
        if (ready < std::min(k, i + kAhead + 1)) std::this_thread::yield();
      }
      if (i + kAhead < k) {
        const uint64_t jn = js[i + kAhead];
        __builtin_prefetch(jn < k ? static_cast<const void*>(&pre[jn])
                                  : static_cast<const void*>(&tab[home(jn)]), 1);
      }
      const uint64_t j = js[i];
      const uint64_t vi = pre[i];
      uint64_t vj;
      if (j < k) {
        vj = pre[j];
        pre[j] = vi;
      } else {
        auto& e = slot(j);
        vj = e.first == kEmpty ? j : e.second;
        e = {j, vi};
      }
      pre[i] = vj;
    }
    if (n / 64 <= 16 * k) {
      std::vector<uint64_t> bm((n + 63) / 64, 0);
      for (const uint64_t v : pre) bm[v >> 6] |= uint64_t(1) << (v & 63);
      uint64_t o = 0;
      for (uint64_t w = 0; w < bm.size(); ++w)
        for (uint64_t b = bm[w]; b; b &= b - 1) pre[o++] = (w << 6) + __builtin_ctzll(b);
    } else {
      std::sort(pre.begin(), pre.end());
    }
    return pre;
  }
};

static uint64_t mix_seed(uint64_t seed, uint64_t tag) {  // rng.cpp:55-61
  uint64_t z = (seed ^ tag) + 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

constexpr uint64_t kValidationTag = 0x76616c69ull;  // randls.cpp:16
constexpr uint64_t kSubsetTag = 0x73756273ull;      // randls.cpp:17
constexpr uint64_t kSketchTag = 0x736b6574ull;      // randls.cpp:18

static uint64_t next_pow2(uint64_t n) {  // transforms.cpp:20-24
  uint64_t p = 1;
  while (p < n) p <<= 1;
  return p;
}

static uint64_t resolve_sample_rows(uint64_t sample_rows, int64_t r) {  // randls.cpp:125-130
  return sample_rows > 0 ? sample_rows
                         : static_cast<uint64_t>(std::ceil(2.5 * static_cast<double>(r)));
}

struct Plan {  // randls.cpp:54-75
  std::vector<double> signs;
  std::vector<uint64_t> rows;
  uint64_t q_pad = 0;
  double scale = 1.0;
};

static Plan make_plan(uint64_t q_w, uint64_t s, uint64_t seed, bool sample = true) {
  Plan plan;
  plan.q_pad = next_pow2(q_w);
  if (sample) {
    require(s >= 1, FSTK_E_PARAMETER, "sample rows must be positive");
    require(s <= plan.q_pad, FSTK_E_PARAMETER, "sample rows exceed the padded row count");
  }
  Rng rng(seed);
  plan.signs.resize(plan.q_pad);
  for (auto& x : plan.signs) x = rng.sign();
  if (sample) {
    plan.rows = rng.sample_without_replacement(plan.q_pad, s);
    plan.scale = std::sqrt(static_cast<double>(plan.q_pad) / static_cast<double>(s));
  }
  return plan;
}

// Extension (north_star literal estimator, not in the reference): S of the Q_w
// working rows sampled uniformly without replacement from the sketch stream,
// scaled by sqrt(Q_w / S), no mixing.  Bit-identical to oracle/fstk_oracle.cpp.
static Plan make_plan_none(uint64_t q_w, uint64_t s, uint64_t seed) {
  Plan plan;
  plan.q_pad = q_w;
  require(s >= 1, FSTK_E_PARAMETER, "sample rows must be positive");
  require(s <= q_w, FSTK_E_PARAMETER, "sample rows exceed the working subset");
  Rng rng(seed);
  plan.rows = rng.sample_without_replacement(q_w, s);
  plan.scale = std::sqrt(static_cast<double>(q_w) / static_cast<double>(s));
  return plan;
}

// ------------------------------------------------------ twiddle replay ---
// For stage len = 2^(s+1) the reference forms wlen = (cos, sin)(-2 pi / len)
// and multiplies w *= wlen once per butterfly (transforms.cpp:36-46).  The
// sequence w_0 = 1, w_{k+1} = w_k * wlen is replayed here with the same
// complex product (a c - b d, a d + b c), each operation rounded separately.
struct TwiddleKey {
  int device;
  uint64_t n;
  bool operator<(const TwiddleKey& o) const {
    return device < o.device || (device == o.device && n < o.n);
  }
};
static std::mutex g_tw_mu;
static std::map<TwiddleKey, std::shared_ptr<DevBuf<double2>>> g_tw;

#pragma GCC push_options
#pragma GCC optimize("fp-contract=off")
static void replay_twiddles(uint64_t n, std::vector<double2>& out) {
  out.assign(n > 1 ? n - 1 : 1, make_double2(1.0, 0.0));
  size_t off = 0;
  for (uint64_t len = 2; len <= n; len <<= 1) {
    const double ang = -2.0 * M_PI / static_cast<double>(len);
    const double wr = std::cos(ang), wi = std::sin(ang);
    double a = 1.0, b = 0.0;
    for (uint64_t k = 0; k < len / 2; ++k) {
      out[off + k] = make_double2(a, b);
      const double ac = a * wr, bd = b * wi, ad = a * wi, bc = b * wr;
      const double re = ac - bd, im = ad + bc;
      a = re;
      b = im;
    }
    off += len / 2;
  }
}
#pragma GCC pop_options

static std::shared_ptr<DevBuf<double2>> twiddles(int device, uint64_t n) {
  std::lock_guard<std::mutex> lk(g_tw_mu);
  auto it = g_tw.find({device, n});
  if (it != g_tw.end()) return it->second;
  std::vector<double2> h;
  replay_twiddles(n, h);
  auto buf = std::make_shared<DevBuf<double2>>(h.size());
  FSTK_CUDA(cudaMemcpy(buf->p, h.data(), h.size() * sizeof(double2), cudaMemcpyHostToDevice));
  g_tw[{device, n}] = buf;
  return buf;
}

// Twiddle rows of pair_pass2_kernel for n = 2^20: row lo holds, at local
// index (2^J - 1) + t' (J = 0..9, t' < 2^J), the replayed twiddle of stage
// 10 + J for k = lo + 1024 t', i.e. tw[(2^(10+J) - 1) + lo + 1024 t'].
static std::map<TwiddleKey, std::shared_ptr<DevBuf<double2>>> g_tw2;
static std::shared_ptr<DevBuf<double2>> warp_pass2_twiddles(int device, uint64_t n) {
  std::lock_guard<std::mutex> lk(g_tw_mu);
  auto it = g_tw2.find({device, n});
  if (it != g_tw2.end()) return it->second;
  std::vector<double2> h, rows(static_cast<size_t>(1024) * 1023);
  replay_twiddles(n, h);
  for (uint64_t lo = 0; lo < 1024; ++lo)
    for (int J = 0; J < 10; ++J)
      for (uint64_t t = 0; t < (uint64_t(1) << J); ++t)
        rows[lo * 1023 + (uint64_t(1) << J) - 1 + t] = h[(uint64_t(1) << (10 + J)) - 1 + lo + 1024 * t];
  auto buf = std::make_shared<DevBuf<double2>>(rows.size());
  FSTK_CUDA(cudaMemcpy(buf->p, rows.data(), rows.size() * sizeof(double2), cudaMemcpyHostToDevice));
  g_tw2[{device, n}] = buf;
  return buf;
}

// Whether the last pass of a sketch runs pair_pass2_kernel: complex
// transforms with q_pad = 2^20 (two passes of 10 stages), when
// FSTK_SKETCH_WARP2=1.  Off by default: it reads the intermediate once
// (4.36 GB per 256 columns) but takes 2.24-2.35 ms against 2.3 ms for
// transform_pass2_kernel (see the kernel's header).  Measured and dropped on
// the way (round 1/2): one class per warp (3.1 ms; each column re-reads the
// 16 MB of class twiddle rows), 4-class CTAs (3.4-5.0 ms), 8-class CTAs with
// the stage 15..19 twiddles in registers (2.67 ms at 8 warps per SM).
// build_inputs orders destination rows to match (class, then t).
static bool warp_last_pass(int kind, uint64_t n) {
  static const bool on = [] {
    const char* e = std::getenv("FSTK_SKETCH_WARP2");
    return e && std::atoi(e) == 1;
  }();
  return on && kind != FSTK_TRANSFORM_WHT && n == (uint64_t(1) << 20);
}

// ------------------------------------------------------ transform pass ---
enum SrcKind { SRC_TABLES = 0, SRC_DENSE = 1, SRC_BUFFER = 2 };

struct PassParams {
  int64_t n;          // q_pad
  int s0, L, G;       // stages [s0, s0+L), groups per CTA
  int kind;           // FSTK_TRANSFORM_*
  int src;            // SrcKind
  int last;           // write A/b instead of the buffer
  // design-column source
  const double* tables;
  Int64x8 toff;
  int64_t ldt;
  int d;
  int r[kMaxOrder];
  const double* sgn;        // per position sign (n)
  const int64_t* row_src;   // per position source row or -1 (n)
  const double* dense;      // SRC_DENSE: column-major q x R
  int64_t ldd;
  const double* rhs;        // rhs values indexed by row_src
  int64_t col0;             // first global column of the batch
  int64_t R;                // columns < R: design; == R: rhs
  const double2* tw;        // replayed twiddles (stage s at tw + 2^s - 1)
  double2* cbuf;            // complex intermediate, n per batch column
  double* rbuf;             // real intermediate (WHT)
  // last pass
  const int32_t* slot;      // per position destination row or -1
  const double* post_re;    // per destination row (DCT: cos; FFT/WHT unused)
  const double* post_im;    // per destination row (DCT: sin)
  const double* post_c;     // per destination row (DCT: c_k)
  double scale;             // plan.scale (sqrt(q_pad/S)) or 1
  double post_c0, post_ck;  // DCT normalisation c_0, c_k (dct_post; pair_pass2_kernel)
  double inv_sqrt_n;        // 1/sqrt(n) (FFT, WHT)
  int64_t row_lo, row_hi;   // destination rows owned by this shard
  int64_t im_off;           // FFT: rows of the Re block in A (Im block follows)
  double* A;
  int64_t lda;
  double* b;
  int prefetch;             // stage the next column with cp.async (see kernel)
  int stg_off;              // byte offset of the staging buffer in shared memory
  int compact;              // last pass: destination rows consecutive per CTA
  int list_off;             // byte offset of the per-CTA sampled-element list
  int ct_rounds;            // L == 10: compile-time stage rounds (radix_round_ct)
  int fuse_last;            // compact complex last pass: stage 9 evaluated in the store
  int swap;                 // staging in x's layout, alternating with x (see kernel)
  // pair_pass2_kernel (last pass of q_pad = 2^20): per-position-class twiddle
  // rows and the sampled elements of each class in destination-row order.
  const double2* tw2;       // 1024 rows of 1023 twiddles (warp_pass2_twiddles)
  const int32_t* lo_start;  // class lo owns destination rows [lo_start[lo], lo_start[lo+1])
  const uint16_t* t_list;   // per destination row: its element t (position t 1024 + lo)
  // Column-sharded sketch (fstk_gpu_refit_begin_columns): the last pass
  // writes sample row sl of column col straight into the all-to-all send
  // buffer A, packed per destination rank h (the owner of sl):
  // A[pk_base[h] + (col - c_lo) * ld_h + (sl - shard_lo[h]) (+ rows_h for Im)],
  // ld_h = fft2 * rows_h.
  int packed;
  int nshards;
  int fft2;
  int64_t S;
  int64_t c_lo;
  int64_t shard_lo[kMaxShards + 1];
  int64_t pk_base[kMaxShards];
};

__device__ __forceinline__ double* store_ptr(const PassParams& P, int64_t col, int64_t sl, bool im) {
  if (!P.packed) {
    double* out = (col == P.R) ? P.b : P.A + P.lda * col;
    return out + (sl - P.row_lo) + (im ? P.im_off : 0);
  }
  int h = static_cast<int>((sl * P.nshards) / P.S);
  while (h + 1 < P.nshards && P.shard_lo[h + 1] <= sl) ++h;
  while (h > 0 && P.shard_lo[h] > sl) --h;
  const int64_t rows_h = P.shard_lo[h + 1] - P.shard_lo[h];
  return P.A + P.pk_base[h] + (col - P.c_lo) * (P.fft2 * rows_h) + (sl - P.shard_lo[h]) +
         (im ? rows_h : 0);
}

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

__device__ __forceinline__ double2 cmul_x(double2 x, double2 w) {
  // (a + ib)(c + id) = (ac - bd) + i(ad + bc), separately rounded (GCC's
  // inline complex product on x86-64 without FMA).
  return make_double2(xsub(xmul(x.x, w.x), xmul(x.y, w.y)), xadd(xmul(x.x, w.y), xmul(x.y, w.x)));
}

__device__ __forceinline__ double source_value(const PassParams& P, int64_t col, int64_t p) {
  const int64_t src = P.row_src[p];
  if (src < 0) return 0.0;
  double v;
  if (col == P.R) {
    v = P.rhs[src];
  } else if (P.src == SRC_DENSE) {
    v = P.dense[src + P.ldd * col];
  } else {
    // design_column (randls.cpp:44-52): ((u0 * u1) * u2) * ..., mode-0 digit fastest.
    int64_t rem = col;
    const int j0 = static_cast<int>(rem % P.r[0]);
    rem /= P.r[0];
    v = P.tables[P.toff.v[0] + j0 * P.ldt + p];
    for (int k = 1; k < P.d; ++k) {
      const int jk = static_cast<int>(rem % P.r[k]);
      rem /= P.r[k];
      v = xmul(v, P.tables[P.toff.v[k] + jk * P.ldt + p]);
    }
  }
  return xmul(P.sgn[p], v);
}

// v2 pass: the CTA owns one set of G adjacent groups (E = 2^L elements each,
// stride 2^s0), keeps that set's replayed twiddles in shared memory and loops
// over columns; stages run three at a time in registers (radix-2^3 rounds of
// the very same radix-2 butterflies, so the result stays bit-identical).
static int pass_group(int s0) {
  // Groups per CTA in passes after the first (FSTK_SKETCH_G: 1 or 2).
  static const int g_later = [] {
    const char* e = std::getenv("FSTK_SKETCH_G");
    return (e && std::atoi(e) == 1) ? 1 : 2;
  }();
  return s0 == 0 ? 1 : g_later;
}
// Shared-memory slot of element e: one pad slot per 8 elements, so the 8
// consecutive elements a thread owns in the first radix round fall in
// distinct 16-byte bank groups.
__device__ __forceinline__ int spad(int e) { return e + (e >> 3); }

template <bool REAL, int NS, int G>
__device__ __forceinline__ void radix_round(typename std::conditional<REAL, double, double2>::type* x,
                                            const double2* tws, int nel, int j) {
  using T = typename std::conditional<REAL, double, double2>::type;
  constexpr int NV = 1 << NS;
  const int jstep = (1 << j) * G;         // element step between the NV values
  const int jmask = (1 << j) - 1;
  for (int blk = threadIdx.x; blk < (nel >> NS); blk += blockDim.x) {
    const int c = blk % G, q = blk / G;
    const int tb = ((q >> j) << (j + NS)) | (q & jmask);
    const int e0 = tb * G + c;
    T v[NV];
#pragma unroll
    for (int m = 0; m < NV; ++m) v[m] = x[spad(e0 + m * jstep)];
    if constexpr (REAL) {
#pragma unroll
      for (int jj = 0; jj < NS; ++jj) {
        const int half = 1 << jj;
#pragma unroll
        for (int a = 0; a < NV; ++a) {
          if (a & half) continue;
          const double u = v[a], w2 = v[a + half];
          v[a] = xadd(u, w2);
          v[a + half] = xsub(u, w2);
        }
      }
    } else {
      // Twiddle of stage jl = j + jj for lower element a: index
      // (2^jl - 1) G + ((tb & jmask) + (a mod 2^jj) 2^j) G + c.
      const int tw0 = (tb & jmask) * G + c;
#pragma unroll
      for (int jj = 0; jj < NS; ++jj) {
        const int half = 1 << jj;
        const double2* twj = tws + ((1 << (j + jj)) - 1) * G + tw0;
#pragma unroll
        for (int a = 0; a < NV; ++a) {
          if (a & half) continue;
          const double2 w = twj[(a & (half - 1)) * jstep];
          const double2 u = v[a];
          const double2 t2 = cmul_x(v[a + half], w);
          v[a] = make_double2(xadd(u.x, t2.x), xadd(u.y, t2.y));
          v[a + half] = make_double2(xsub(u.x, t2.x), xsub(u.y, t2.y));
        }
      }
    }
#pragma unroll
    for (int m = 0; m < NV; ++m) x[spad(e0 + m * jstep)] = v[m];
  }
}

// radix_round with the stage index J and the element count NEL known at
// compile time (the L = 10 passes of every q_pad >= 2^10): the NV shared
// addresses and the twiddle addresses of a block become one base plus
// immediate offsets, instead of an IMAD chain per access.  Same butterflies
// in the same order, so bit-identical to radix_round.
//   spad(e0 + m jstep) - spad(e0) == spad(m jstep) here: jstep is a multiple
//   of 8, or (J = 0) e0 mod 8 < G = jstep with m jstep < 8 G.
template <bool REAL, int NS, int G, int J, int NEL>
__device__ __forceinline__ void radix_round_ct(typename std::conditional<REAL, double, double2>::type* x,
                                               const double2* tws) {
  using T = typename std::conditional<REAL, double, double2>::type;
  constexpr int NV = 1 << NS;
  constexpr int jstep = (1 << J) * G;
  constexpr int jmask = (1 << J) - 1;
  static_assert(jstep % 8 == 0 || J == 0, "offset identity needs jstep % 8 == 0 or J == 0");
  for (int blk = threadIdx.x; blk < (NEL >> NS); blk += blockDim.x) {
    const int c = blk % G, q = blk / G;
    const int tb = ((q >> J) << (J + NS)) | (q & jmask);
    const int e0 = tb * G + c;
    T* xb = x + spad(e0);
    T v[NV];
#pragma unroll
    for (int m = 0; m < NV; ++m) v[m] = xb[spad(m * jstep)];
    if constexpr (REAL) {
#pragma unroll
      for (int jj = 0; jj < NS; ++jj) {
        const int half = 1 << jj;
#pragma unroll
        for (int a = 0; a < NV; ++a) {
          if (a & half) continue;
          const double u = v[a], w2 = v[a + half];
          v[a] = xadd(u, w2);
          v[a + half] = xsub(u, w2);
        }
      }
    } else {
      const double2* twb = tws + (tb & jmask) * G + c;
#pragma unroll
      for (int jj = 0; jj < NS; ++jj) {
        const int half = 1 << jj;
#pragma unroll
        for (int a = 0; a < NV; ++a) {
          if (a & half) continue;
          const double2 w = twb[((1 << (J + jj)) - 1) * G + (a & (half - 1)) * jstep];
          const double2 u = v[a];
          const double2 t2 = cmul_x(v[a + half], w);
          v[a] = make_double2(xadd(u.x, t2.x), xadd(u.y, t2.y));
          v[a + half] = make_double2(xsub(u.x, t2.x), xsub(u.y, t2.y));
        }
      }
    }
#pragma unroll
    for (int m = 0; m < NV; ++m) xb[spad(m * jstep)] = v[m];
  }
}

template <bool REAL, int G, int DT>  // DT: mode count when known at compile time (0 = runtime)
__global__ void __launch_bounds__(256, G == 2 ? 2 : 3) transform_pass2_kernel(const PassParams P, int ncols_batch) {
  using T = typename std::conditional<REAL, double, double2>::type;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int L = P.L, E = 1 << L, nel = E * G;
  T* x = reinterpret_cast<T*>(smem_raw);
  double2* tws = reinterpret_cast<double2*>(smem_raw + static_cast<size_t>(nel + nel / 8) * sizeof(T));
  // P.swap (complex intermediate source): the staging buffer has x's padded
  // layout, and the two alternate as the working buffer column by column.
  const bool swap = !REAL && P.src == SRC_BUFFER && P.prefetch && P.swap;
  T* const buf0 = x;
  T* const buf1 = reinterpret_cast<T*>(smem_raw + P.stg_off);
  int cur = 0;
  const int64_t stride = int64_t(1) << P.s0;
  const int64_t lo_blocks = stride / G;
  const int64_t bidx = blockIdx.x;
  const int64_t c0 = (bidx % lo_blocks) * G;
  const int64_t hi = bidx / lo_blocks;
  const int64_t base = hi * (stride << L) + c0;
  if constexpr (!REAL) {
    // twiddles of stages s0 .. s0+L-1 for this group set; stage j at (2^j - 1) G
    for (int e = threadIdx.x; e < (E - 1) * G; e += blockDim.x) {
      const int blk = e / G, c = e % G;
      const int j = 31 - __clz(blk + 1);
      const int m = blk + 1 - (1 << j);
      const int64_t k = c0 + c + static_cast<int64_t>(m) * stride;
      tws[e] = P.tw[(int64_t(1) << (P.s0 + j)) - 1 + k];
    }
  }
  // Prefetch (P.prefetch): the next column's inputs -- the intermediate's
  // 16-byte element pairs, or the DT mode-table segments of a design column
  // -- are copied into a shared staging buffer with cp.async while this
  // column's butterflies run, so the strided global reads no longer stall
  // the stages.  Data movement only: the arithmetic is unchanged.
  unsigned char* stg = smem_raw + P.stg_off;
  auto staged = [&](int cc) {
    return P.prefetch && cc < ncols_batch && (P.src == SRC_BUFFER || P.col0 + cc < P.R);
  };
  auto prefetch = [&](int cc, int into) {
    if (!staged(cc)) return;
    if (swap) {
      for (int e = threadIdx.x; e < nel; e += blockDim.x) {
        const int64_t p = base + (e % G) + static_cast<int64_t>(e / G) * stride;
        cp_async16((into ? buf1 : buf0) + spad(e), P.cbuf + static_cast<int64_t>(cc) * P.n + p);
      }
    } else if (P.src == SRC_BUFFER) {
      // G == 2: element pairs (e, e+1) are adjacent in global memory.
      const int nch = REAL ? nel / 2 : nel;
      for (int ch = threadIdx.x; ch < nch; ch += blockDim.x) {
        const int e = REAL ? 2 * ch : ch;
        const int64_t p = base + (e % G) + static_cast<int64_t>(e / G) * stride;
        const void* src = REAL ? static_cast<const void*>(P.rbuf + static_cast<int64_t>(cc) * P.n + p)
                               : static_cast<const void*>(P.cbuf + static_cast<int64_t>(cc) * P.n + p);
        cp_async16(stg + static_cast<size_t>(ch) * 16, src);
      }
    } else if constexpr (DT > 0) {
      // G == 1, stride 1: the CTA's positions are base .. base + nel - 1.
      // Mixed-radix digits in 32-bit arithmetic (columns < 2^31): a 64-bit
      // division per digit per column per thread was the pass's top cost.
      uint32_t rem = static_cast<uint32_t>(P.col0 + cc);
#pragma unroll
      for (int k = 0; k < DT; ++k) {
        const uint32_t rk = static_cast<uint32_t>(P.r[k]);
        const int64_t jk = rem % rk;
        rem /= rk;
        const double* t = P.tables + P.toff.v[k] + jk * P.ldt + base;
        for (int ch = threadIdx.x; ch < nel / 2; ch += blockDim.x)
          cp_async16(stg + (static_cast<size_t>(k) * nel + 2 * ch) * 8, t + 2 * ch);
      }
    }
    cp_async_commit();
  };
  // Compact last pass: destination rows are assigned in last-pass visit
  // order (build_inputs), so this CTA's sampled elements, in ascending e,
  // own the consecutive rows first, first + 1, ...  Collect their e once;
  // every column then stores only those (~S / q_pad of the elements) with
  // coalesced post-factor reads and A writes, instead of reloading slot[]
  // for all elements per column.
  uint16_t* elist = reinterpret_cast<uint16_t*>(smem_raw + P.list_off);
  __shared__ int s_wcnt[32];
  __shared__ int s_cnt;
  __shared__ int s_first;
  const bool use_list = P.last && P.compact;
  if (use_list) {
    if (threadIdx.x == 0) {
      s_cnt = 0;
      s_first = 0;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i0 = 0; i0 < nel; i0 += blockDim.x) {
      const int e = i0 + threadIdx.x;
      int sl = -1;
      if (e < nel) sl = P.slot[base + (e % G) + static_cast<int64_t>(e / G) * stride];
      const unsigned bal = __ballot_sync(0xffffffffu, sl >= 0);
      if (lane == 0) s_wcnt[warp] = __popc(bal);
      __syncthreads();
      int off = s_cnt;
      for (int w = 0; w < warp; ++w) off += s_wcnt[w];
      if (sl >= 0) {
        const int pos = off + __popc(bal & ((1u << lane) - 1));
        elist[pos] = static_cast<uint16_t>(e);
        if (pos == 0) s_first = sl;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        int tot = s_cnt;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) tot += s_wcnt[w];
        s_cnt = tot;
      }
      __syncthreads();
    }
  }
  // The DCT rotation of this CTA's first two sampled elements per thread,
  // the same for every column: kept in registers.
  double cre0 = 0.0, cim0 = 0.0, cre1 = 0.0, cim1 = 0.0;
  if (!REAL && use_list && P.kind == FSTK_TRANSFORM_DCT) {
    const int cnt = s_cnt;
    const int64_t first = s_first;
    if (static_cast<int>(threadIdx.x) < cnt) {
      cre0 = __ldg(P.post_re + first + threadIdx.x);
      cim0 = __ldg(P.post_im + first + threadIdx.x);
    }
    if (static_cast<int>(threadIdx.x + blockDim.x) < cnt) {
      cre1 = __ldg(P.post_re + first + threadIdx.x + blockDim.x);
      cim1 = __ldg(P.post_im + first + threadIdx.x + blockDim.x);
    }
  }
  prefetch(blockIdx.y, 0);
  for (int cc = blockIdx.y; cc < ncols_batch; cc += gridDim.y) {
    const int64_t col = P.col0 + cc;
    __syncthreads();
    // ---- load (generate the design column on the fly in the first pass)
    if (staged(cc)) {
      cp_async_wait_all();
      __syncthreads();
      if (swap) {
        x = cur ? buf1 : buf0;
      } else if (P.src == SRC_BUFFER) {
        const T* sv = reinterpret_cast<const T*>(stg);
        for (int e = threadIdx.x; e < nel; e += blockDim.x) x[spad(e)] = sv[e];
      } else if constexpr (DT > 0) {
        const double* sv = reinterpret_cast<const double*>(stg);
        for (int e = threadIdx.x; e < nel; e += blockDim.x) {
          // design_column (randls.cpp:44-52): ((u0 * u1) * u2) * ..., sign in u0.
          double v = sv[e];
#pragma unroll
          for (int k = 1; k < DT; ++k) v = xmul(v, sv[k * nel + e]);
          if constexpr (REAL)
            x[spad(e)] = v;
          else
            x[spad(e)] = make_double2(v, 0.0);
        }
      }
    } else if (P.src == SRC_BUFFER) {
#pragma unroll 4
      for (int e = threadIdx.x; e < nel; e += blockDim.x) {
        const int64_t p = base + (e % G) + static_cast<int64_t>(e / G) * stride;
        if constexpr (REAL)
          x[spad(e)] = P.rbuf[static_cast<int64_t>(cc) * P.n + p];
        else
          x[spad(e)] = P.cbuf[static_cast<int64_t>(cc) * P.n + p];
      }
    } else {
      constexpr int NTC = DT > 0 ? DT : kMaxOrder;
      const double* tc[NTC];
      const bool design = col < P.R;
      if (design && P.src == SRC_TABLES) {
        uint32_t rem = static_cast<uint32_t>(col);
#pragma unroll
        for (int k = 0; k < NTC; ++k) {
          if (DT > 0 || k < P.d) {
            const uint32_t rk = static_cast<uint32_t>(P.r[k]);
            const int64_t jk = rem % rk;
            rem /= rk;
            tc[k] = P.tables + P.toff.v[k] + jk * P.ldt;
          }
        }
      }
#pragma unroll 4
      for (int e = threadIdx.x; e < nel; e += blockDim.x) {
        const int64_t p = base + (e % G) + static_cast<int64_t>(e / G) * stride;
        double v = 0.0;
        if (design && P.src == SRC_TABLES) {
          // design_column (randls.cpp:44-52): ((u0 * u1) * u2) * ..., with the
          // sign already folded into u0 and zero rows at padded positions:
          // three independent loads, no gather.
          v = tc[0][p];
#pragma unroll
          for (int k = 1; k < NTC; ++k)
            if (DT > 0 || k < P.d) v = xmul(v, tc[k][p]);
        } else {
          const int64_t src = P.row_src[p];
          if (src >= 0) v = xmul(P.sgn[p], design ? P.dense[src + P.ldd * col] : P.rhs[src]);
        }
        if constexpr (REAL)
          x[spad(e)] = v;
        else
          x[spad(e)] = make_double2(v, 0.0);
      }
    }
    __syncthreads();
    prefetch(cc + gridDim.y, cur ^ 1);  // staging is free: this column now lives in x
    cur ^= 1;
    // ---- stages, three per register round
    // The compact last pass of a complex transform folds the tenth stage into
    // its store: only the sampled outputs (~S / q_pad of them) evaluate their
    // butterfly, saving a full shared-memory round trip of the tile.
    const bool fuse_last = !REAL && use_list && L == 10 && P.ct_rounds && P.fuse_last;
    if (L == 10 && P.ct_rounds) {
      constexpr int NE = 1024 * G;
      radix_round_ct<REAL, 3, G, 0, NE>(x, tws);
      __syncthreads();
      radix_round_ct<REAL, 3, G, 3, NE>(x, tws);
      __syncthreads();
      radix_round_ct<REAL, 3, G, 6, NE>(x, tws);
      __syncthreads();
      if (!fuse_last) {
        radix_round_ct<REAL, 1, G, 9, NE>(x, tws);
        __syncthreads();
      }
    } else
    for (int j = 0; j < L; j += 3) {
      const int ns = min(3, L - j);
      if (ns == 3)
        radix_round<REAL, 3, G>(x, tws, nel, j);
      else if (ns == 2)
        radix_round<REAL, 2, G>(x, tws, nel, j);
      else
        radix_round<REAL, 1, G>(x, tws, nel, j);
      __syncthreads();
    }
    // ---- store
    if (use_list) {
      const int cnt = s_cnt;
      const int64_t first = s_first;
      for (int idx = threadIdx.x; idx < cnt; idx += blockDim.x) {
        const int e = elist[idx];
        const int64_t sl = first + idx;
        if (sl < P.row_lo || sl >= P.row_hi) continue;
        if constexpr (REAL) {
          *store_ptr(P, col, sl, false) = xmul(P.scale, xmul(x[spad(e)], P.inv_sqrt_n));
        } else if (P.kind == FSTK_TRANSFORM_DCT) {
          double2 V;
          if (fuse_last) {
            // Stage 9 of the pass (radix_round_ct<..., 1, G, 9, ...>): the
            // class-local index i pairs with i ^ 512; lower u + w y, upper
            // u - w y, w = tws[(2^9 - 1) G + (i mod 512) G + c] -- the same
            // separately rounded operations.
            const int c = e % G, i = e / G, il = i & 511;
            const double2 u = x[spad(il * G + c)];
            const double2 t2 = cmul_x(x[spad((il + 512) * G + c)], tws[(511 + il) * G + c]);
            V = i < 512 ? make_double2(xadd(u.x, t2.x), xadd(u.y, t2.y))
                        : make_double2(xsub(u.x, t2.x), xsub(u.y, t2.y));
          } else {
            V = x[spad(e)];
          }
          const bool k0 = idx == static_cast<int>(threadIdx.x), k1 = idx == static_cast<int>(threadIdx.x + blockDim.x);
          const double re = k0 ? cre0 : (k1 ? cre1 : __ldg(P.post_re + sl));
          const double im = k0 ? cim0 : (k1 ? cim1 : __ldg(P.post_im + sl));
          const double val = xsub(xmul(re, V.x), xmul(im, V.y));
          // dct_post: c_0 at output position 0, c_k elsewhere
          const bool pos0 = base + (e % G) + static_cast<int64_t>(e / G) * stride == 0;
          *store_ptr(P, col, sl, false) = xmul(P.scale, xmul(pos0 ? P.post_c0 : P.post_ck, val));
        } else {
          double2 V;
          if (fuse_last) {
            const int c = e % G, i = e / G, il = i & 511;
            const double2 u = x[spad(il * G + c)];
            const double2 t2 = cmul_x(x[spad((il + 512) * G + c)], tws[(511 + il) * G + c]);
            V = i < 512 ? make_double2(xadd(u.x, t2.x), xadd(u.y, t2.y))
                        : make_double2(xsub(u.x, t2.x), xsub(u.y, t2.y));
          } else {
            V = x[spad(e)];
          }
          *store_ptr(P, col, sl, false) = xmul(P.scale, xmul(V.x, P.inv_sqrt_n));
          *store_ptr(P, col, sl, true) = xmul(P.scale, xmul(V.y, P.inv_sqrt_n));
        }
      }
      continue;
    }
#pragma unroll 4
    for (int e = threadIdx.x; e < nel; e += blockDim.x) {
      const int64_t p = base + (e % G) + static_cast<int64_t>(e / G) * stride;
      if (!P.last) {
        if constexpr (REAL)
          P.rbuf[static_cast<int64_t>(cc) * P.n + p] = x[spad(e)];
        else
          P.cbuf[static_cast<int64_t>(cc) * P.n + p] = x[spad(e)];
        continue;
      }
      const int32_t sl = P.slot[p];
      if (sl < 0 || sl < P.row_lo || sl >= P.row_hi) continue;
      if constexpr (REAL) {
        *store_ptr(P, col, sl, false) = xmul(P.scale, xmul(x[spad(e)], P.inv_sqrt_n));
      } else if (P.kind == FSTK_TRANSFORM_DCT) {
        const double2 V = x[spad(e)];
        const double val = xsub(xmul(P.post_re[sl], V.x), xmul(P.post_im[sl], V.y));
        *store_ptr(P, col, sl, false) = xmul(P.scale, xmul(P.post_c[sl], val));
      } else {
        const double2 V = x[spad(e)];
        *store_ptr(P, col, sl, false) = xmul(P.scale, xmul(V.x, P.inv_sqrt_n));
        *store_ptr(P, col, sl, true) = xmul(P.scale, xmul(V.y, P.inv_sqrt_n));
      }
    }
  }
}

// ------------------------------------------- warp-level first pass (K3a) ---
// Stages 0..9 of a q_pad >= 2^11 complex (DCT/FFT) sketch, one 1024-point
// block of one design column per warp, held in registers: no CTA barrier.
// Lane a first owns elements 32a + b (b = 0..31, register index) and runs
// stages 0..4 (len 2..32) in registers; one warp-private shared-memory
// exchange (33-element rows: conflict-free both ways) gives lane b' the
// elements 32a + b' for stages 5..9 (len 64..1024); the block is stored as
// 32 coalesced 512-byte rows.  The butterflies are transforms.cpp:36-46's,
// each a separately rounded (ac - bd, ad + bc) product and sum, with two
// value-preserving shortcuts: the k = 0 twiddle of every stage is the exact
// (1, 0) the recurrence starts from, and a product by it returns its operand
// (up to the sign of an exact zero), so it is skipped; stage 0's inputs are
// real, so its imaginary sums (+0 +- +0 = +0) are written directly.
// Stages 0..4 use twiddles 0..30, passed by value (constant-bank operands);
// stages 5..9 read twiddles 31..1022 from one shared copy per CTA.  The
// twiddles of these stages do not depend on q_pad.
struct WarpPass1Params {
  int64_t n;          // q_pad
  int nblk;           // n / 1024
  int ncols;          // columns in this batch
  int64_t col0;       // first global column of the batch
  int64_t R;          // columns < R: design; == R: rhs
  const double* tables;
  Int64x8 toff;
  int64_t ldt;
  int r[kMaxOrder];
  const double* sgn;
  const int64_t* row_src;
  const double* rhs;
  const double2* tw;  // replayed twiddles (global)
  double2* cbuf;      // complex intermediate, n per batch column
  double2 tw5[31];    // twiddles of stages 0..4
};

constexpr int kWp1Row = 33;                    // padded 32-element row
constexpr int kWp1Buf = 32 * kWp1Row;          // double2 per warp
constexpr int kWp1Tw = 992;                    // twiddles 31..1022

template <int DT, int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 1) warp_pass1_kernel(const WarpPass1Params P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* tws = reinterpret_cast<double2*>(smem_raw);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double2* X = tws + kWp1Tw + warp * kWp1Buf;
  double* Xr = reinterpret_cast<double*>(X);  // real inputs, rows of 33 doubles
  for (int i = threadIdx.x; i < kWp1Tw; i += blockDim.x) tws[i] = P.tw[31 + i];
  __syncthreads();
  const int64_t units = static_cast<int64_t>(P.ncols) * P.nblk;
  const int64_t nw = static_cast<int64_t>(gridDim.x) * WARPS;
  for (int64_t u = static_cast<int64_t>(blockIdx.x) * WARPS + warp; u < units; u += nw) {
    // Column fastest: concurrently running warps share the block's u1, u2
    // segments across consecutive columns (mode-0 digit fastest).
    const int64_t hb = u / P.ncols;
    const int cc = static_cast<int>(u - hb * P.ncols);
    const int64_t base = hb * 1024;
    const int64_t col = P.col0 + cc;
    // ---- inputs: design column x_p = ((s u0) u1) u2 ... (randls.cpp:44-52,
    // sign folded into u0), coalesced pairs, into the warp's buffer.
    __syncwarp();
    if (col < P.R) {
      const double* tc[DT];
      uint32_t rem = static_cast<uint32_t>(col);
#pragma unroll
      for (int k = 0; k < DT; ++k) {
        const uint32_t rk = static_cast<uint32_t>(P.r[k]);
        tc[k] = P.tables + P.toff.v[k] + static_cast<int64_t>(rem % rk) * P.ldt + base;
        rem /= rk;
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        double2 t[DT][8];
#pragma unroll
        for (int j = 0; j < 8; ++j)
#pragma unroll
          for (int k = 0; k < DT; ++k)
            t[k][j] = __ldg(reinterpret_cast<const double2*>(tc[k] + 64 * (8 * h + j) + 2 * lane));
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          double v0 = t[0][j].x, v1 = t[0][j].y;
#pragma unroll
          for (int k = 1; k < DT; ++k) {
            v0 = xmul(v0, t[k][j].x);
            v1 = xmul(v1, t[k][j].y);
          }
          const int e = 64 * (8 * h + j) + 2 * lane;
          Xr[e + (e >> 5)] = v0;
          Xr[e + 1 + (e >> 5)] = v1;
        }
      }
    } else {
      for (int e = lane; e < 1024; e += 32) {
        const int64_t p = base + e;
        const int64_t src = P.row_src[p];
        Xr[e + (e >> 5)] = src < 0 ? 0.0 : xmul(P.sgn[p], P.rhs[src]);
      }
    }
    __syncwarp();
    double2 v[32];
    // ---- stage 0 (len 2, twiddle (1, 0)): real inputs, staged as doubles
#pragma unroll
    for (int b = 0; b < 32; b += 2) {
      const double a0 = Xr[lane * kWp1Row + b], a1 = Xr[lane * kWp1Row + b + 1];
      v[b] = make_double2(xadd(a0, a1), 0.0);
      v[b + 1] = make_double2(xsub(a0, a1), 0.0);
    }
    // ---- stages 1..4 (len 4..32)
#pragma unroll
    for (int s = 1; s < 5; ++s) {
      const int half = 1 << s;
#pragma unroll
      for (int b = 0; b < 32; ++b) {
        if (b & half) continue;
        const int k = b & (half - 1);
        const double2 uu = v[b];
        const double2 t2 = k == 0 ? v[b + half] : cmul_x(v[b + half], P.tw5[half - 1 + k]);
        v[b] = make_double2(xadd(uu.x, t2.x), xadd(uu.y, t2.y));
        v[b + half] = make_double2(xsub(uu.x, t2.x), xsub(uu.y, t2.y));
      }
    }
    // ---- exchange: lane b' gets elements 32 a + b'
    __syncwarp();
#pragma unroll
    for (int b = 0; b < 32; ++b) X[lane * kWp1Row + b] = v[b];
    __syncwarp();
#pragma unroll
    for (int a = 0; a < 32; ++a) v[a] = X[a * kWp1Row + lane];
    // ---- stages 5..9 (len 64..1024): k = b' + 32 (a mod 2^i)
#pragma unroll
    for (int i = 0; i < 5; ++i) {
      const int half = 1 << i;  // in rows of 32
#pragma unroll
      for (int m = 0; m < half; ++m) {
        const double2 w = tws[32 * half - 32 + lane + 32 * m];
#pragma unroll
        for (int a = m; a < 32; a += 2 * half) {
          const double2 uu = v[a];
          const double2 t2 = cmul_x(v[a + half], w);
          v[a] = make_double2(xadd(uu.x, t2.x), xadd(uu.y, t2.y));
          v[a + half] = make_double2(xsub(uu.x, t2.x), xsub(uu.y, t2.y));
        }
      }
    }
    double2* out = P.cbuf + static_cast<int64_t>(cc) * P.n + base + lane;
#pragma unroll
    for (int a = 0; a < 32; ++a) __stcg(out + 32 * a, v[a]);
  }
}

// ------------------------------------------- warp-level last pass (K3b) ---
// Stages 10..19 of a q_pad = 2^20 complex sketch without a CTA barrier.
// A CTA owns the two adjacent position classes lo0, lo0 + 1 (positions
// t 1024 + lo, t < 1024: 32-byte runs of the intermediate), keeps their 2 x
// 1023 replayed twiddles in shared memory, and its kPp2Pairs warp pairs work
// on kPp2Pairs different columns at once: the twiddles are shared by every
// warp and no warp waits on another column's data.
// Warp h of a pair first takes the half t = 512 h + (0..511) of both classes:
// Loads: lane l reads t = 512 h + 16 l + b (b = 0..15) with 256-bit loads,
// one whole 32-byte sector (both classes' elements) per lane and load.  (With
// 16-byte loads at this 16 KB stride the small L1 left beside the shared
// memory caps the requests in flight: 1.8 TB/s against 4.7 TB/s, measured by
// tools/stride_read2.cu.)
// Phase A: stages 10..13 (len 2^11..2^14) over b, in registers, both classes.
// A warp-private 32 x 32 transpose (XOR-swizzled rows: conflict-free both
// ways) gives lane (class, b) the 32 elements a = t bits 4..8 for
// Phase B: stages 14..18.  The result is parked in the warp's buffer; after
// a 64-thread named barrier warp h takes class lo0 + h from both buffers,
// lane (c', b) the elements with t bit 4 = c' of both halves, for
// Phase C: stage 19 in registers.  Register j of lane l is then output
// t = 32 j + l of the class; destination rows are assigned class by class in
// ascending t (build_inputs), so a ballot over each register's sampled flags
// compacts the sampled outputs (~S / q_pad of them) into consecutive
// shared-memory slots, from which they are post-rotated (DCT) or split (FFT)
// and stored row-contiguously; the next column's loads are issued after them
// (a spill reload behind the 16 outstanding sector loads waits for DRAM).
// Same butterflies and epilogue as transform_pass2_kernel, in the same order,
// so A is bit-identical.
// Measured at C2 (profiles/ncu_sketch_r02.txt): 2.2-2.35 ms per 256 columns
// against 2.3 ms for transform_pass2_kernel (C2 sketch 0.443 s against
// 0.445 s), so it stays opt-in (FSTK_SKETCH_WARP2=1): with 10-12 warps per SM
// (168 registers; 12 warps fill 224 KB once the DCT rotations are read from
// L2 instead of a shared copy) the three shared-memory round trips and the
// pair / cluster barriers leave the fp64 pipe at 37%.
constexpr int kPp2Pairs = 6;                   // columns in flight per CTA
constexpr int kPp2Warps = 2 * kPp2Pairs;
constexpr int kPp2Buf = 1024;                  // double2 per warp
// CTAs of kPp2Cluster adjacent class pairs form a cluster and stay within one
// column of each other (split cluster barrier), so the 128-byte lines they
// share are fetched from DRAM once and hit in L2 for the others.
constexpr int kPp2Cluster = 4;
constexpr int kPp2Cap = 0;                     // sampled elements per class with DCT rotations cached in shared memory (0: read from L2)
constexpr size_t kPp2Smem = (2 * 1023 + kPp2Warps * kPp2Buf) * sizeof(double2) +
                            2 * kPp2Cap * 2 * sizeof(double) + 64 * sizeof(uint32_t);

__device__ __forceinline__ void pair_barrier(int pair) {
  asm volatile("bar.sync %0, 64;" ::"r"(pair + 1) : "memory");
}

// One 32-byte sector: the elements of classes lo0 and lo0 + 1 at one t.
// One 32-byte sector: the elements of classes lo0 and lo0 + 1 at one t.  Normal
// L2 eviction priority: the neighbouring class pairs of the cluster take the
// rest of the 128-byte line from L2 (evict_first re-fetched it from DRAM).
__device__ __forceinline__ void ld_sector(const double2* p, double2& c0, double2& c1) {
  asm volatile("ld.global.L1::no_allocate.L2::evict_normal.v4.b64 {%0,%1,%2,%3}, [%4];"
               : "=d"(c0.x), "=d"(c0.y), "=d"(c1.x), "=d"(c1.y)
               : "l"(p));
}

__device__ __forceinline__ void butterfly(double2& lo, double2& hi, const double2 w) {
  const double2 uu = lo;
  const double2 t2 = cmul_x(hi, w);
  lo = make_double2(xadd(uu.x, t2.x), xadd(uu.y, t2.y));
  hi = make_double2(xsub(uu.x, t2.x), xsub(uu.y, t2.y));
}

__device__ __forceinline__ void cluster_arrive_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.aligned;" ::: "memory"); }

__global__ void __cluster_dims__(kPp2Cluster, 1, 1) __launch_bounds__(kPp2Warps * 32, 1)
pair_pass2_kernel(const PassParams P, int ncols_batch) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int pair = warp >> 1, h = warp & 1;
  double2* tw = reinterpret_cast<double2*>(smem_raw);              // [2][1023]
  double2* Xall = tw + 2 * 1023;
  double2* X = Xall + warp * kPp2Buf;                              // this warp's buffer
  const double2* X0 = Xall + (2 * pair) * kPp2Buf;                 // t < 512 half of the pair
  const double2* X1 = X0 + kPp2Buf;                                // t >= 512 half
  double* cre_all = reinterpret_cast<double*>(Xall + kPp2Warps * kPp2Buf);
  double* cim_all = cre_all + 2 * kPp2Cap;
  uint32_t* mask_all = reinterpret_cast<uint32_t*>(cim_all + 2 * kPp2Cap);  // [2][32]
  const int lo0 = 2 * static_cast<int>(blockIdx.x);
  const bool dct = P.kind == FSTK_TRANSFORM_DCT;
  for (int i = threadIdx.x; i < 2 * 1023; i += blockDim.x) tw[i] = P.tw2[static_cast<int64_t>(lo0) * 1023 + i];
  if (threadIdx.x < 64) mask_all[threadIdx.x] = 0;
  __syncthreads();
  // Sampled flags of both classes: bit j of mask[class][l] is t = 32 j + l.
  {
    const int f0 = P.lo_start[lo0], f2 = P.lo_start[lo0 + 2], f1 = P.lo_start[lo0 + 1];
    for (int i = f0 + threadIdx.x; i < f2; i += blockDim.x) {
      const int cl = i >= f1 ? 1 : 0;
      const int t = P.t_list[i];
      atomicOr(mask_all + 32 * cl + (t & 31), 1u << (t >> 5));
      const int k = i - (cl ? f1 : f0);
      if (dct && k < kPp2Cap) {
        cre_all[cl * kPp2Cap + k] = P.post_re[i];
        cim_all[cl * kPp2Cap + k] = P.post_im[i];
      }
    }
  }
  __syncthreads();
  const double2* src0 = P.cbuf + lo0 + static_cast<int64_t>(512 * h + 16 * lane) * 1024;
  // Output coordinates: warp h stores class lo0 + h.
  const int lo = lo0 + h;
  const int first = P.lo_start[lo], cnt = P.lo_start[lo + 1] - first;
  // rows [row_lo, row_hi) of this shard within the class's rows first + [0, cnt)
  const int ilo = static_cast<int>(max(int64_t(0), min(int64_t(cnt), P.row_lo - first)));
  const int ihi = static_cast<int>(max(int64_t(0), min(int64_t(cnt), P.row_hi - first)));
  const uint32_t M = mask_all[32 * h + lane];
  const uint32_t lt = (1u << lane) - 1u;
  const bool zero_first = lo == 0 && cnt > 0 && (M & 1u) && lane == 0;  // t = 0 of class 0: dct_post(k = 0)
  const double2* twh = tw + 1023 * h;
  const double* cre = cre_all + h * kPp2Cap;
  const double* cim = cim_all + h * kPp2Cap;
  const int pc = lane >> 4, pb = lane & 15;  // phase B/C lane coordinates
  const double2* twc = tw + 1023 * pc;
  const int cstep = static_cast<int>(gridDim.y) * kPp2Pairs;
  int cc = static_cast<int>(blockIdx.y) * kPp2Pairs + pair;
  // Every warp of the cluster runs the same number of rounds (the cluster
  // barrier counts all of them); a pair without a column left idles through.
  const int rounds = (ncols_batch - static_cast<int>(blockIdx.y) * kPp2Pairs + cstep - 1) / cstep;
  double2 v[32];
  if (cc < ncols_batch) {
    const double2* src = src0 + static_cast<int64_t>(cc) * P.n;
#pragma unroll
    for (int b = 0; b < 16; ++b) ld_sector(src + static_cast<int64_t>(b) * 1024, v[b], v[16 + b]);
  }
  cluster_arrive_relaxed();
  for (int rnd = 0; rnd < rounds; ++rnd, cc += cstep) {
    if (cc >= ncols_batch) {
      cluster_wait();
      cluster_arrive_relaxed();
      continue;
    }
    const int64_t col = P.col0 + cc;
    // ---- phase A, stages 10..13: registers (class, b), k = lo + 1024 (b mod 2^j)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int half = 1 << j;
#pragma unroll
      for (int cl = 0; cl < 2; ++cl) {
#pragma unroll
        for (int b = 0; b < 16; ++b) {
          if (b & half) continue;
          butterfly(v[16 * cl + b], v[16 * cl + b + half], tw[1023 * cl + half - 1 + (b & (half - 1))]);
        }
      }
    }
    // ---- transpose: register r = 16 class + b of lane a  ->  register a of lane r.
    // Element (a, r) lives at 32 a + (r ^ a).
    __syncwarp();
#pragma unroll
    for (int r = 0; r < 32; ++r) X[32 * lane + (r ^ lane)] = v[r];
    __syncwarp();
#pragma unroll
    for (int a2 = 0; a2 < 32; ++a2) v[a2] = X[32 * a2 + (lane ^ a2)];
    // ---- phase B, stages 14..18: k = lo + 1024 (b + 16 (a mod 2^i))
#pragma unroll
    for (int i = 0; i < 5; ++i) {
      const int half = 1 << i;
#pragma unroll
      for (int m = 0; m < half; ++m) {
        const double2 w = twc[(16 << i) - 1 + 16 * m + pb];
#pragma unroll
        for (int a2 = m; a2 < 32; a2 += 2 * half) butterfly(v[a2], v[a2 + half], w);
      }
    }
    __syncwarp();
#pragma unroll
    for (int a2 = 0; a2 < 32; ++a2) X[32 * a2 + (lane ^ a2)] = v[a2];
    pair_barrier(pair);  // both halves parked
    // ---- phase C: class lo0 + h; lane (c', b) takes a = 2 a4 + c' of both halves
#pragma unroll
    for (int a4 = 0; a4 < 16; ++a4) {
      const int a2 = 2 * a4 + pc;
      const int idx = 32 * a2 + ((16 * h + pb) ^ a2);
      v[a4] = X0[idx];
      v[16 + a4] = X1[idx];
    }
    pair_barrier(pair);  // both buffers read: free for the compaction and the next column
    // stage 19: k = lo + 1024 (32 a4 + lane)
#pragma unroll
    for (int a4 = 0; a4 < 16; ++a4) butterfly(v[a4], v[16 + a4], twh[511 + 32 * a4 + lane]);
    // ---- compaction: register j is t = 32 j + lane; ascending t = ballot order
    {
      int base = 0;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const bool on = (M >> j) & 1u;
        const uint32_t bal = __ballot_sync(0xffffffffu, on);
        if (on) X[base + __popc(bal & lt)] = v[j];
        base += __popc(bal);
      }
    }
    __syncwarp();
    auto prefetch = [&] {
      cluster_wait();  // every CTA of the cluster has issued this round's loads
      if (cc + cstep < ncols_batch) {
        const double2* src = src0 + static_cast<int64_t>(cc + cstep) * P.n;
#pragma unroll
        for (int b = 0; b < 16; ++b) ld_sector(src + static_cast<int64_t>(b) * 1024, v[b], v[16 + b]);
      }
      cluster_arrive_relaxed();
    };
    // ---- sampled outputs of class lo: consecutive destination rows
    if (!P.packed) {
      double* out = ((col == P.R) ? P.b : P.A + P.lda * col) + (first - P.row_lo);
      if (dct) {
#pragma unroll 4
        for (int i = ilo + lane; i < ihi; i += 32) {
          const double2 V = X[i];
          const bool cached = i < kPp2Cap;
          const double re = cached ? cre[i] : __ldg(P.post_re + first + i);
          const double im = cached ? cim[i] : __ldg(P.post_im + first + i);
          const double val = xsub(xmul(re, V.x), xmul(im, V.y));
          const double cf = (zero_first && i == 0) ? P.post_c0 : P.post_ck;  // dct_post(k = t 1024 + lo)
          out[i] = xmul(P.scale, xmul(cf, val));
        }
      } else {
#pragma unroll 4
        for (int i = ilo + lane; i < ihi; i += 32) {
          const double2 V = X[i];
          out[i] = xmul(P.scale, xmul(V.x, P.inv_sqrt_n));
          out[i + P.im_off] = xmul(P.scale, xmul(V.y, P.inv_sqrt_n));
        }
      }
    } else {
      // column-sharded sketch: rows go to their owners' packed send blocks
      for (int i = ilo + lane; i < ihi; i += 32) {
        const int64_t sl = first + i;
        const double2 V = X[i];
        if (dct) {
          const double val = xsub(xmul(__ldg(P.post_re + sl), V.x), xmul(__ldg(P.post_im + sl), V.y));
          const double cf = (zero_first && i == 0) ? P.post_c0 : P.post_ck;
          *store_ptr(P, col, sl, false) = xmul(P.scale, xmul(cf, val));
        } else {
          *store_ptr(P, col, sl, false) = xmul(P.scale, xmul(V.x, P.inv_sqrt_n));
          *store_ptr(P, col, sl, true) = xmul(P.scale, xmul(V.y, P.inv_sqrt_n));
        }
      }
    }
    prefetch();
  }
  cluster_wait();
}

// u0[p] *= s_p for every function (sign folded into the mode-0 table: since
// s = +-1 and IEEE products are sign-symmetric, ((s u0) u1) u2 == s ((u0 u1) u2)
// bit for bit, which is what sketch_column feeds the transform).
__global__ void fold_sign_kernel(double* __restrict__ t0, int64_t ldt, int r0,
                                 const double* __restrict__ sgn, int64_t n) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double s = sgn[i];
  for (int j = 0; j < r0; ++j) t0[j * ldt + i] = xmul(s, t0[j * ldt + i]);
}

// transform = none (north_star K5): rows of A generated on the fly from the
// mode tables of the sampled points, block by block, so A never exists whole.
// W[i, ell] = scale * ((u0 u1) u2 ...)[row0 + i] (design_column order,
// randls.cpp:44-52, then plan.scale as sketch_column applies it).
template <int DT>
__global__ void __launch_bounds__(256) design_block_kernel(
    const double* __restrict__ tables, Int64x8 toff, int64_t ldt, int d, Int64x8 ranks,
    int64_t row0, int64_t nrows, int64_t R, double scale, double* __restrict__ W, int64_t ldw) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  constexpr int NTC = DT > 0 ? DT : kMaxOrder;
  for (int64_t ell = blockIdx.y; ell < R; ell += gridDim.y) {
    if (i >= nrows) continue;
    int64_t rem = ell;
    double v = 0.0;
#pragma unroll
    for (int k = 0; k < NTC; ++k) {
      if (DT > 0 || k < d) {
        const int64_t jk = rem % ranks.v[k];
        rem /= ranks.v[k];
        const double u = tables[toff.v[k] + jk * ldt + row0 + i];
        v = k == 0 ? u : xmul(v, u);
      }
    }
    W[ell * ldw + i] = xmul(scale, v);
  }
}

__global__ void scaled_gather_kernel(const double* __restrict__ vals, const int64_t* __restrict__ src,
                                     int64_t n, double scale, double* __restrict__ out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[i] = xmul(scale, vals[src[i]]);
}

// True when no entry is Inf/NaN (exponent field all ones); host threads.
static bool all_finite(const double* a, size_t n) {
  const unsigned hw = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  const size_t per = std::max<size_t>(size_t(1) << 20, (n + hw - 1) / hw);
  const size_t nt = (n + per - 1) / per;
  std::vector<char> bad(nt, 0);
  auto work = [&](size_t t) {
    const uint64_t* u = reinterpret_cast<const uint64_t*>(a);
    const size_t lo = t * per, hi = std::min(n, lo + per);
    uint64_t acc = 0;
    for (size_t i = lo; i < hi; ++i) acc |= static_cast<uint64_t>(((u[i] >> 52) & 0x7ff) == 0x7ff);
    bad[t] = acc != 0;
  };
  std::vector<std::thread> th;
  for (size_t t = 1; t < nt; ++t) th.emplace_back(work, t);
  if (nt > 0) work(0);
  for (auto& x : th) x.join();
  for (char b : bad)
    if (b) return false;
  return true;
}

// fn(lo, hi) over [0, n) in contiguous chunks on the host cores (independent
// per element; results do not depend on the split).
template <class F>
static void parallel_chunks(uint64_t n, F&& fn, uint64_t min_chunk = uint64_t(1) << 15) {
  const unsigned hw = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  const uint64_t nt = std::max<uint64_t>(1, std::min<uint64_t>(hw, n / std::max<uint64_t>(min_chunk, 1)));
  if (nt <= 1) {
    fn(uint64_t(0), n);
    return;
  }
  std::vector<std::thread> th;
  for (uint64_t t = 1; t < nt; ++t) th.emplace_back([&, t] { fn(n * t / nt, n * (t + 1) / nt); });
  fn(uint64_t(0), n / nt);
  for (auto& x : th) x.join();
}

__global__ void finite_check_kernel(const double* __restrict__ a, int64_t n, int* flag) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    if (!isfinite(a[i])) atomicExch(flag, 1);
}

__global__ void gather_points_kernel(const double* __restrict__ pts, int64_t ldp, int d,
                                     const int64_t* __restrict__ idx, int64_t n,
                                     double* __restrict__ out, int64_t ldo,
                                     const double* __restrict__ vals, double* __restrict__ vout) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t s = idx[i];
  for (int k = 0; k < d; ++k) out[k * ldo + i] = pts[k * ldp + s];
  if (vals) vout[i] = vals[s];
}

// --------------------------------------------------------- the sketcher ---
// Runs the transform over all columns [0, ncols) (ncols = R + 1 with the rhs)
// for a prepared input ordering.
struct SketchJob {
  int kind;
  uint64_t n;           // q_pad
  int src;              // SRC_TABLES or SRC_DENSE
  const double* tables;
  int64_t toff[kMaxOrder];
  int64_t ldt;
  int d;
  int r[kMaxOrder];
  const double* dense;
  int64_t ldd;
  const double* rhs;
  int64_t R;            // design columns
  bool with_rhs;
  const double* sgn;
  const int64_t* row_src;
  const int32_t* slot;
  const double* post_re;
  const double* post_im;
  const double* post_c;
  double scale;
  int64_t row_lo, row_hi, im_off;
  double* A;
  int64_t lda;
  double* b;
  bool compact = false;  // slot = last-pass visit order (build_inputs compact)
  const int32_t* lo_start = nullptr;  // warp_last_pass order (build_inputs)
  const uint16_t* t_list = nullptr;
  // Column range [col_lo, col_hi) of the R (+rhs) columns (col_hi < 0: all)
  // and the packed all-to-all layout (see PassParams::packed).
  int64_t col_lo = 0, col_hi = -1;
  bool packed = false;
  int nshards = 1;
  int64_t S = 0;
  int64_t shard_lo[kMaxShards + 1] = {0};
  int64_t pk_base[kMaxShards] = {0};
};

static int ilog2(uint64_t n) {
  int l = 0;
  while ((uint64_t(1) << l) < n) ++l;
  return l;
}

static void dct_post(uint64_t k, uint64_t n, double* re, double* im, double* c);

static void run_sketch(int device, const SketchJob& J, cudaStream_t s) {
  const int LOG = ilog2(J.n);
  const bool real = J.kind == FSTK_TRANSFORM_WHT;
  auto tw = real ? nullptr : twiddles(device, J.n);
  // Twiddles 0..30 (stages 0..4; independent of n) for warp_pass1_kernel.
  double2 tw_host[31];
  if (!real && J.n >= 32) {
    std::vector<double2> h;
    replay_twiddles(32, h);
    for (int i = 0; i < 31; ++i) tw_host[i] = h[i];
  }
  const int64_t ncols = J.R + (J.with_rhs ? 1 : 0);
  // The pass kernels decompose column indices in 32-bit arithmetic.
  require(ncols < (int64_t(1) << 31), FSTK_E_PARAMETER, "too many design columns");
  const size_t elem = real ? 8 : 16;
  const int npass = LOG == 0 ? 1 : (LOG + 9) / 10;
  // Column batches of ~FSTK_SKETCH_BATCH_MB (default 4 GB) of inter-pass
  // intermediate: big enough that each pass's grid fills the GPU many times
  // over (smaller batches measured slower; running consecutive batches on two
  // streams gained nothing, since full grids only overlap at their tails).
  // Measured at C2 (tools/sketch_time.py, 3 repetitions): 4 GB batches with
  // 64 columns per CTA 0.71 s vs 2 GB / 8 columns 0.78 s -- each CTA loads its
  // twiddle set once per launch and amortises it over more columns.  Capped
  // at a quarter of the free memory.
  int64_t batch_mb = 4096;
  {
    size_t fr = 0, tot = 0;
    if (device_mem_info(&fr, &tot) == cudaSuccess)
      batch_mb = std::max<int64_t>(64, std::min<int64_t>(batch_mb, static_cast<int64_t>(fr >> 22)));
    else
      cudaGetLastError();
  }
  if (const char* e = std::getenv("FSTK_SKETCH_BATCH_MB")) batch_mb = std::max(1, std::atoi(e));
  int64_t nb = ncols;
  if (npass > 1) nb = std::max<int64_t>(1, std::min<int64_t>(ncols, (batch_mb << 20) /
                                                                        static_cast<int64_t>(J.n * elem)));
  DevBuf<double2> cbuf;
  DevBuf<double> rbuf;
  if (npass > 1) {
    if (real)
      rbuf.alloc(static_cast<size_t>(nb) * J.n);
    else
      cbuf.alloc(static_cast<size_t>(nb) * J.n);
  }
  static std::once_flag attr_once[64];
  std::call_once(attr_once[device & 63], [&] {
    auto attr = [](const void* f) {
      FSTK_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
      // One carveout for every pass kernel: the passes alternate hundreds of
      // times per sketch and must not trigger L1/shared reconfiguration.
      FSTK_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    };
    attr(reinterpret_cast<const void*>(transform_pass2_kernel<false, 1, 0>));
    attr(reinterpret_cast<const void*>(transform_pass2_kernel<true, 1, 0>));
    attr(reinterpret_cast<const void*>(transform_pass2_kernel<false, 1, 3>));
    attr(reinterpret_cast<const void*>(transform_pass2_kernel<true, 1, 3>));
    attr(reinterpret_cast<const void*>(transform_pass2_kernel<false, 1, 4>));
    attr(reinterpret_cast<const void*>(transform_pass2_kernel<true, 1, 4>));
    attr(reinterpret_cast<const void*>(transform_pass2_kernel<false, 2, 0>));
    attr(reinterpret_cast<const void*>(transform_pass2_kernel<true, 2, 0>));
    auto attr_w = [](const void* f) {
      FSTK_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
      FSTK_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    };
    attr_w(reinterpret_cast<const void*>(warp_pass1_kernel<3, 8>));
    attr_w(reinterpret_cast<const void*>(warp_pass1_kernel<3, 12>));
    attr_w(reinterpret_cast<const void*>(warp_pass1_kernel<4, 8>));
    attr_w(reinterpret_cast<const void*>(warp_pass1_kernel<4, 12>));
    attr_w(reinterpret_cast<const void*>(pair_pass2_kernel));
  });
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  const int64_t cbeg = J.col_lo, cend = J.col_hi < 0 ? ncols : std::min(ncols, J.col_hi);
  for (int64_t c0 = cbeg; c0 < cend; c0 += nb) {
    const int64_t bc = std::min(nb, cend - c0);
    for (int pass = 0; pass < npass; ++pass) {
      PassParams P{};
      P.n = static_cast<int64_t>(J.n);
      P.s0 = 10 * pass;
      P.L = std::min(10, LOG - P.s0);
      P.G = static_cast<int>(std::min<int64_t>(pass_group(P.s0), int64_t(1) << P.s0));
      P.kind = J.kind;
      P.src = pass == 0 ? J.src : SRC_BUFFER;
      P.last = pass == npass - 1;
      P.tables = J.tables;
      for (int k = 0; k < J.d; ++k) {
        P.toff.v[k] = J.toff[k];
        P.r[k] = J.r[k];
      }
      P.ldt = J.ldt;
      P.d = J.d;
      P.sgn = J.sgn;
      P.row_src = J.row_src;
      P.dense = J.dense;
      P.ldd = J.ldd;
      P.rhs = J.rhs;
      P.col0 = c0;
      P.R = J.R;
      P.tw = tw ? tw->p : nullptr;
      P.cbuf = cbuf.p;
      P.rbuf = rbuf.p;
      P.slot = J.slot;
      P.post_re = J.post_re;
      P.post_im = J.post_im;
      P.post_c = J.post_c;
      P.scale = J.scale;
      P.inv_sqrt_n = 1.0 / std::sqrt(static_cast<double>(J.n));
      {
        double re, im;
        dct_post(0, J.n, &re, &im, &P.post_c0);
        dct_post(1, J.n, &re, &im, &P.post_ck);
      }
      P.row_lo = J.row_lo;
      P.row_hi = J.row_hi;
      P.im_off = J.im_off;
      P.A = J.A;
      P.lda = J.lda;
      P.b = J.b;
      P.packed = J.packed ? 1 : 0;
      P.nshards = J.nshards;
      P.fft2 = J.kind == FSTK_TRANSFORM_FFT ? 2 : 1;
      P.S = J.S;
      P.c_lo = J.col_lo;
      for (int h = 0; h <= J.nshards && h <= kMaxShards; ++h) P.shard_lo[h] = J.shard_lo[h];
      for (int h = 0; h < J.nshards && h < kMaxShards; ++h) P.pk_base[h] = J.pk_base[h];
      const int64_t E = int64_t(1) << P.L;
      const int64_t sets = static_cast<int64_t>(J.n) / (E * P.G);
      size_t smem = static_cast<size_t>(E * P.G + E * P.G / 8) * elem +
                    (real ? 0 : static_cast<size_t>((E - 1) * P.G) * 16);
      // cp.async staging of the next column (FSTK_SKETCH_PREFETCH=0 disables).
      static const bool pf_on = [] {
        const char* e = std::getenv("FSTK_SKETCH_PREFETCH");
        return !(e && std::atoi(e) == 0);
      }();
      const int dtp = (P.src == SRC_TABLES && (J.d == 3 || J.d == 4)) ? J.d : 0;
      size_t stg = 0;
      static const bool swap_on = [] {
        const char* e = std::getenv("FSTK_SKETCH_SWAP");
        return !(e && std::atoi(e) == 0);
      }();
      P.swap = (swap_on && pf_on && P.src == SRC_BUFFER && !real) ? 1 : 0;
      if (P.swap)
        stg = static_cast<size_t>(E * P.G + E * P.G / 8) * elem;
      else if (pf_on && P.src == SRC_BUFFER && (P.G == 2 || !real))
        stg = static_cast<size_t>(E * P.G) * elem;
      else if (pf_on && dtp > 0 && P.G == 1 && P.s0 == 0 && E * P.G >= 2)
        stg = static_cast<size_t>(dtp) * E * P.G * 8;
      smem = round_up(static_cast<int64_t>(smem), 16);
      P.prefetch = stg > 0 ? 1 : 0;
      P.stg_off = static_cast<int>(smem);
      smem += stg;
      P.compact = (J.compact && P.last && E * P.G <= 65536) ? 1 : 0;
      static const int ct_on = [] {
        const char* e = std::getenv("FSTK_SKETCH_CT");
        return (e && std::atoi(e) == 0) ? 0 : 1;
      }();
      P.ct_rounds = ct_on;
      static const int fuse_on = [] {
        const char* e = std::getenv("FSTK_SKETCH_FUSE_LAST");
        return (e && std::atoi(e) == 0) ? 0 : 1;
      }();
      P.fuse_last = fuse_on;
      smem = round_up(static_cast<int64_t>(smem), 16);
      P.list_off = static_cast<int>(smem);
      if (P.compact) smem += static_cast<size_t>(E * P.G) * sizeof(uint16_t);
      // Up to 64 columns per CTA (gridDim.y = batch / 64, at least 8 CTAs per
      // SM): each CTA's twiddle set is loaded once per launch and amortised.
      static const int64_t cpc = [] {
        const char* e = std::getenv("FSTK_SKETCH_COLS_PER_CTA");
        return e ? std::max(1, std::atoi(e)) : 64;
      }();
      const int64_t gy = std::max<int64_t>(1, std::min<int64_t>(bc, std::max<int64_t>(
                                                                    ceil_div(bc, cpc), ceil_div(int64_t(sms) * 8, sets))));
      dim3 grid(static_cast<unsigned>(sets), static_cast<unsigned>(gy));
      ProfScope prof(FSTK_PROF_TRANSFORM, s);
      const int dt = (P.src == SRC_TABLES && (J.d == 3 || J.d == 4)) ? J.d : 0;
      const int nb = static_cast<int>(bc);
      // Warp-level first pass (warp_pass1_kernel): complex transforms with
      // a design-table source and a later pass, and pair_pass2_kernel for
      // the last pass of q_pad = 2^20 (FSTK_SKETCH_WARP=0 disables both;
      // FSTK_SKETCH_WARP=8 runs 8 warps per CTA instead of 12).
      static const int warp_mode = [] {
        const char* e = std::getenv("FSTK_SKETCH_WARP");
        return e ? std::atoi(e) : 12;
      }();
      if (P.last && J.compact && J.lo_start && warp_last_pass(J.kind, J.n) && npass == 2) {
        auto tw2 = warp_pass2_twiddles(device, J.n);
        P.tw2 = tw2->p;
        P.lo_start = J.lo_start;
        P.t_list = J.t_list;
        // One CTA per class pair and column slice: ~7 waves of CTAs.
        const int64_t ysplit = std::max<int64_t>(1, std::min<int64_t>(ceil_div(static_cast<int64_t>(nb), kPp2Pairs),
                                                                      ceil_div(int64_t(sms) * 7, 512)));
        dim3 pgrid(512, static_cast<unsigned>(ysplit));
pair_pass2_kernel<<<pgrid, kPp2Warps * 32, kPp2Smem, s>>>(P, nb);
        check_launch("pair_pass2_kernel");
        continue;
      }
      if (warp_mode != 0 && !real && pass == 0 && !P.last && P.L == 10 && dt > 0) {
        WarpPass1Params W{};
        W.n = P.n;
        W.nblk = static_cast<int>(J.n / 1024);
        W.ncols = nb;
        W.col0 = c0;
        W.R = J.R;
        W.tables = J.tables;
        W.toff = P.toff;
        W.ldt = J.ldt;
        for (int k = 0; k < J.d; ++k) W.r[k] = J.r[k];
        W.sgn = J.sgn;
        W.row_src = J.row_src;
        W.rhs = J.rhs;
        W.tw = tw->p;
        W.cbuf = cbuf.p;
        for (int i = 0; i < 31; ++i) W.tw5[i] = tw_host[i];
        const int wpc = warp_mode == 8 ? 8 : 12;
        const size_t wsm = static_cast<size_t>(kWp1Tw + wpc * kWp1Buf) * sizeof(double2);
        const unsigned wgrid = static_cast<unsigned>(std::min<int64_t>(
            sms, ceil_div(static_cast<int64_t>(nb) * W.nblk, static_cast<int64_t>(wpc))));
        if (dt == 3 && wpc == 8)
          warp_pass1_kernel<3, 8><<<wgrid, 8 * 32, wsm, s>>>(W);
        else if (dt == 3)
          warp_pass1_kernel<3, 12><<<wgrid, 12 * 32, wsm, s>>>(W);
        else if (wpc == 8)
          warp_pass1_kernel<4, 8><<<wgrid, 8 * 32, wsm, s>>>(W);
        else
          warp_pass1_kernel<4, 12><<<wgrid, 12 * 32, wsm, s>>>(W);
        check_launch("warp_pass1_kernel");
        continue;
      }
      const int nt1 = 256;  // 128-thread CTAs for G = 1 measured no faster
      if (P.G == 2) {
        if (real)
          transform_pass2_kernel<true, 2, 0><<<grid, 256, smem, s>>>(P, nb);
        else
          transform_pass2_kernel<false, 2, 0><<<grid, 256, smem, s>>>(P, nb);
      } else if (dt == 3) {
        if (real)
          transform_pass2_kernel<true, 1, 3><<<grid, nt1, smem, s>>>(P, nb);
        else
          transform_pass2_kernel<false, 1, 3><<<grid, nt1, smem, s>>>(P, nb);
      } else if (dt == 4) {
        if (real)
          transform_pass2_kernel<true, 1, 4><<<grid, nt1, smem, s>>>(P, nb);
        else
          transform_pass2_kernel<false, 1, 4><<<grid, nt1, smem, s>>>(P, nb);
      } else {
        if (real)
          transform_pass2_kernel<true, 1, 0><<<grid, nt1, smem, s>>>(P, nb);
        else
          transform_pass2_kernel<false, 1, 0><<<grid, nt1, smem, s>>>(P, nb);
      }
      check_launch("transform_pass2_kernel");
    }
  }
}

// Host tables for the mixing input order and the DCT post-rotation.
static uint64_t bitrev(uint64_t v, int bits) {
  uint64_t r = 0;
  for (int i = 0; i < bits; ++i) r |= ((v >> i) & 1ull) << (bits - 1 - i);
  return r;
}

// Position p of the transform input holds point index i(p) of the column.
static void input_order(int kind, uint64_t n, std::vector<uint64_t>& pos2i) {
  const int LOG = ilog2(n);
  pos2i.resize(n);
  parallel_chunks(n, [&](uint64_t lo, uint64_t hi) {
  for (uint64_t p = lo; p < hi; ++p) {
    if (kind == FSTK_TRANSFORM_WHT) {
      pos2i[p] = p;
      continue;
    }
    const uint64_t m = bitrev(p, LOG);
    if (kind == FSTK_TRANSFORM_FFT) {
      pos2i[p] = m;
    } else if (n == 1) {
      pos2i[p] = 0;
    } else {
      // Makhoul: v[m] = x[2m] (m < n/2), v[n-1-m'] = x[2m'+1].
      pos2i[p] = m < n / 2 ? 2 * m : 2 * (n - 1 - m) + 1;
    }
  }
  });
}

#pragma GCC push_options
#pragma GCC optimize("fp-contract=off")
// dct2_orthonormal rotation + normalisation for output index k (transforms.cpp:96-103).
static void dct_post(uint64_t k, uint64_t n, double* re, double* im, double* c) {
  const double ang = -M_PI * static_cast<double>(k) / (2.0 * static_cast<double>(n));
  *re = std::cos(ang);
  *im = std::sin(ang);
  const double c0 = std::sqrt(1.0 / static_cast<double>(n));
  const double ck = std::sqrt(2.0 / static_cast<double>(n));
  *c = k == 0 ? c0 : ck;
}
#pragma GCC pop_options

// Device-side sketch inputs for one ordering.
struct SketchInputs {
  DevBuf<double> sgn;
  DevBuf<int64_t> row_src;
  DevBuf<int32_t> slot;
  DevBuf<double> post_re, post_im, post_c;
  DevBuf<int32_t> lo_start;  // warp_last_pass order: 1025 class starts
  DevBuf<uint16_t> t_list;   // warp_last_pass order: element t per destination row
  int64_t rows_total = 0;  // destination rows (S, or q_pad for mixed_matrix)
  std::vector<int64_t> dest_of_sample;  // sample s (plan order) -> destination row
};

// pos2src(i): source row of input point i (< q_w) ; `compact` chooses the
// destination row order: false = plan order (reference row order), true =
// the order in which the last pass visits positions (contiguous stores).
static void build_inputs(int kind, uint64_t n, uint64_t q_w, const std::vector<double>& signs,
                         const std::vector<uint64_t>& rows, bool all_rows,
                         const std::vector<int64_t>& src_of_i, bool compact, SketchInputs& S,
                         cudaStream_t s) {
  std::vector<uint64_t> pos2i;
  input_order(kind, n, pos2i);
  std::vector<double> sg(n);
  std::vector<int64_t> rs(n);
  parallel_chunks(n, [&](uint64_t lo, uint64_t hi) {
    for (uint64_t p = lo; p < hi; ++p) {
      const uint64_t i = pos2i[p];
      if (i < q_w) {
        rs[p] = src_of_i.empty() ? static_cast<int64_t>(i) : src_of_i[i];
        sg[p] = signs[i];
      } else {
        rs[p] = -1;
        sg[p] = 0.0;
      }
    }
  });
  // Destination rows.
  std::vector<int32_t> slot(n, -1);
  const uint64_t nrows = all_rows ? n : rows.size();
  std::vector<uint64_t> pos_of_dest(nrows);
  S.dest_of_sample.assign(nrows, 0);
  if (!compact) {
    for (uint64_t sidx = 0; sidx < nrows; ++sidx) {
      const uint64_t k = all_rows ? sidx : rows[sidx];
      slot[k] = static_cast<int32_t>(sidx);
      pos_of_dest[sidx] = k;
      S.dest_of_sample[sidx] = static_cast<int64_t>(sidx);
    }
  } else {
    // Visit order of the last pass: CTA-major (group id), then element (c + t G).
    const int LOG = ilog2(n);
    const int npass = LOG == 0 ? 1 : (LOG + 9) / 10;
    const int s0 = 10 * (npass - 1);
    const int L = std::min(10, LOG - s0);
    const uint64_t stride = uint64_t(1) << s0;
    const uint64_t G = std::min<uint64_t>(static_cast<uint64_t>(pass_group(s0)), stride);
    const uint64_t lo_blocks = stride / G;
    const bool wl = warp_last_pass(kind, n);  // pair_pass2_kernel: class lo, then t
    auto order_key = [&](uint64_t k) {
      if (wl) return ((k & 1023) << 32) | (k >> 10);
      const uint64_t low = k & (stride - 1);
      const uint64_t hi = k >> (s0 + L);
      const uint64_t cta = hi * lo_blocks + low / G;
      const uint64_t c = low % G;
      const uint64_t t = (k >> s0) & ((uint64_t(1) << L) - 1);
      return (cta << 32) | (t * G + c);
    };
    std::vector<std::pair<uint64_t, uint64_t>> keyed(nrows);
    parallel_chunks(nrows, [&](uint64_t lo, uint64_t hi) {
      for (uint64_t sidx = lo; sidx < hi; ++sidx) {
        const uint64_t k = all_rows ? sidx : rows[sidx];
        keyed[sidx] = {order_key(k), sidx};
      }
    });
    std::sort(keyed.begin(), keyed.end());
    parallel_chunks(nrows, [&](uint64_t lo, uint64_t hi) {
      for (uint64_t dst = lo; dst < hi; ++dst) {
        const uint64_t sidx = keyed[dst].second;
        const uint64_t k = all_rows ? sidx : rows[sidx];
        slot[k] = static_cast<int32_t>(dst);
        pos_of_dest[dst] = k;
        S.dest_of_sample[sidx] = static_cast<int64_t>(dst);
      }
    });
    if (wl) {
      std::vector<int32_t> ls(1025, 0);
      std::vector<uint16_t> tl(std::max<uint64_t>(nrows, 1));
      for (uint64_t dst = 0; dst < nrows; ++dst) {
        const uint64_t k = pos_of_dest[dst];
        ++ls[(k & 1023) + 1];
        tl[dst] = static_cast<uint16_t>(k >> 10);
      }
      for (int i = 0; i < 1024; ++i) ls[i + 1] += ls[i];
      S.lo_start.alloc(1025);
      S.t_list.alloc(tl.size());
      FSTK_CUDA(cudaMemcpyAsync(S.lo_start.p, ls.data(), ls.size() * 4, cudaMemcpyHostToDevice, s));
      FSTK_CUDA(cudaMemcpyAsync(S.t_list.p, tl.data(), tl.size() * 2, cudaMemcpyHostToDevice, s));
      FSTK_CUDA(cudaStreamSynchronize(s));  // host vectors go out of scope
    }
  }
  std::vector<double> pre(nrows), pim(nrows), pc(nrows);
  if (kind == FSTK_TRANSFORM_DCT) {
    parallel_chunks(nrows, [&](uint64_t lo, uint64_t hi) {
      for (uint64_t dst = lo; dst < hi; ++dst)
        dct_post(pos_of_dest[dst], n, &pre[dst], &pim[dst], &pc[dst]);
    });
    if (n == 1) {  // dct2_orthonormal returns early for n == 1 (identity)
      pre[0] = 1.0;
      pim[0] = 0.0;
      pc[0] = 1.0;
    }
  }
  S.rows_total = static_cast<int64_t>(nrows);
  S.sgn.alloc(n);
  S.row_src.alloc(n);
  S.slot.alloc(n);
  S.post_re.alloc(std::max<uint64_t>(nrows, 1));
  S.post_im.alloc(std::max<uint64_t>(nrows, 1));
  S.post_c.alloc(std::max<uint64_t>(nrows, 1));
  FSTK_CUDA(cudaMemcpyAsync(S.sgn.p, sg.data(), n * 8, cudaMemcpyHostToDevice, s));
  FSTK_CUDA(cudaMemcpyAsync(S.row_src.p, rs.data(), n * 8, cudaMemcpyHostToDevice, s));
  FSTK_CUDA(cudaMemcpyAsync(S.slot.p, slot.data(), n * 4, cudaMemcpyHostToDevice, s));
  if (nrows) {
    FSTK_CUDA(cudaMemcpyAsync(S.post_re.p, pre.data(), nrows * 8, cudaMemcpyHostToDevice, s));
    FSTK_CUDA(cudaMemcpyAsync(S.post_im.p, pim.data(), nrows * 8, cudaMemcpyHostToDevice, s));
    FSTK_CUDA(cudaMemcpyAsync(S.post_c.p, pc.data(), nrows * 8, cudaMemcpyHostToDevice, s));
  }
  FSTK_CUDA(cudaStreamSynchronize(s));  // host vectors go out of scope
}

// ----------------------------------------------------- library handles ---
struct Handles {
  cublasHandle_t blas = nullptr;
  cusolverDnHandle_t solver = nullptr;
};
// One cuBLAS/cuSOLVER handle pair per (host thread, device): a handle must
// not be driven from two threads at once (cublasSetStream + calls), and the
// C-ABI is callable from many threads (refits of different models on one
// device run concurrently).  Created on first use with the device current;
// left to the process teardown.
static Handles& handles(int device) {
  static thread_local std::map<int, Handles> tl_handles;
  Handles& h = tl_handles[device];
  if (!h.blas) {
    if (cublasCreate(&h.blas) != CUBLAS_STATUS_SUCCESS) fail(FSTK_E_COMPUTE, "cublasCreate failed");
    if (cusolverDnCreate(&h.solver) != CUSOLVER_STATUS_SUCCESS)
      fail(FSTK_E_COMPUTE, "cusolverDnCreate failed");
  }
  return h;
}

cublasHandle_t blas_handle(int device) { return handles(device).blas; }
// A second cuBLAS handle per (thread, device) for work enqueued on a side
// stream while the first handle drives the main stream (separate workspaces).
cublasHandle_t blas_side_handle(int device) {
  static thread_local std::map<int, cublasHandle_t> tl_side;
  cublasHandle_t& h = tl_side[device];
  if (!h && cublasCreate(&h) != CUBLAS_STATUS_SUCCESS) fail(FSTK_E_COMPUTE, "cublasCreate failed");
  return h;
}
cusolverDnHandle_t solver_handle(int device) { return handles(device).solver; }

struct EventTimer {
  cudaEvent_t a = nullptr, b = nullptr;
  cudaStream_t s;
  explicit EventTimer(cudaStream_t st) : s(st) {
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, s);
  }
  double seconds() {
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    return ms * 1e-3;
  }
  ~EventTimer() {
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  }
};


}  // namespace fstk_gpu

using namespace fstk_gpu;

struct fstk_gpu_refit {
  // Declared first, so destroyed last: the members below release their
  // blocks into the device cache, and under the default policy (1) the last
  // open session's end then hands every cached block back to the driver.
  DeviceCacheSession cache_session;
  const fstk_gpu_model* model = nullptr;
  int device = 0;
  cudaStream_t stream = nullptr;
  fstk_sketch_cfg cfg{};
  int shard = 0, shards = 1;
  int64_t q = 0;
  int d = 0;
  int64_t R = 0;
  uint64_t S = 0, q_w = 0, q_pad = 0;
  bool held_out = true;
  Plan plan;
  SketchInputs in;
  int64_t row_lo = 0, row_hi = 0, local_rows = 0;  // destination rows of this shard
  DevBuf<double> A;      // local_rows(x2 for FFT) x R, column-major
  DevBuf<double> b;
  DevBuf<double> d_points, d_values;  // working-subset rows (subset order) on device
  std::vector<int64_t> subset;         // dataset row of each working-subset row
  DevBuf<double> val_points, val_values;
  int64_t n_val = 0;
  std::vector<double> h_val_values;
  std::vector<int64_t> h_val_index;   // dataset rows of the validation points
  // Solve state: Cholesky factor of the (summed) Gram, or the eigen fallback.
  DevBuf<double> L;       // R x R, lower Cholesky factor
  bool factored = false;
  bool rank_def = false;
  double sigma_ratio = 0.0;  // certificate sigma_min(A) / max column norm (0 = not computed)
  // The certificate's lambda_min(L L^T) power iteration, started by factor()
  // on a side stream (own cuBLAS handle) so it overlaps the refinement --
  // which only reads L too -- in the one-call solve and the staged path alike.
  LambdaMinEstimate est;
  cudaStream_t est_stream = nullptr;
  cudaEvent_t est_event = nullptr;
  bool est_live = false;
  DevBuf<double> tmp_r;   // local residual rows
  // transform = none: mode tables of this shard's sampled rows (A generated on demand)
  bool none = false;
  // Column-sharded sketch: this shard's columns [c_lo, c_hi) of the R + 1,
  // packed per destination rank in `send` until the all-to-all lands the row
  // slab in A (then exchanged = true and the refit continues row-sharded).
  bool columns = false, exchanged = false;
  int64_t c_lo = 0, c_hi = 0;
  int64_t pk_base[kMaxShards] = {0};
  DevBuf<double> send;
  GramScratch gs;        // sliced int8 Gram scratch (fstk_gram.cu)
  int gram_used = 0;     // digit planes of the last Gram (0 = native fp64)
  DevBuf<double> tables;
  DevBuf<double> kr;     // transform = none: Khatri-Rao of modes 1..d-1 (ldt x R/r0), lazily
  DevBuf<double> kr_tmp; // transform = none: ldt x r0 scratch of the structured products
  DevBuf<double> apply_dx;  // refinement scratch (no per-step allocations)
  DevBuf<int> apply_info;
  int64_t toff[kMaxOrder] = {0};
  int64_t ldt = 0;
  ~fstk_gpu_refit() {
    try {
      est.wait_enqueued();  // the side worker may still be enqueueing on est_stream
    } catch (...) {
    }
    if (est_stream) {
      cudaStreamSynchronize(est_stream);
      cudaStreamDestroy(est_stream);
    }
    if (est_event) cudaEventDestroy(est_event);
    if (stream) cudaStreamDestroy(stream);
  }
};

namespace fstk_gpu {

static double rel_residual(const std::vector<double>& pred, const std::vector<double>& vals) {
  // randls.cpp:350-356
  double sd = 0.0, sv = 0.0;
  for (size_t i = 0; i < vals.size(); ++i) {
    const double dlt = pred[i] - vals[i];
    sd += dlt * dlt;
    sv += vals[i] * vals[i];
  }
  const double denom = std::sqrt(sv), diff = std::sqrt(sd);
  return denom > 0.0 ? diff / denom : diff;
}

}  // namespace fstk_gpu

extern "C" {

namespace fstk_gpu {
static std::mutex g_stage_mu;      // pinned staging of the working-subset upload
static double* g_stage = nullptr;
static size_t g_stage_n = 0;

static int32_t refit_begin_impl(const fstk_gpu_model* m, const double* points,
                                const double* values, int64_t q, int32_t d,
                                const fstk_sketch_cfg* cfg, int32_t shard, int32_t shards,
                                bool columns, fstk_gpu_refit** out, fstk_reestimate_info* info,
                                fstk_gpu_error* err) {
  return guarded(err, [&] {
    require(m && points && values && cfg && out, FSTK_E_PARAMETER, "null argument");
    *out = nullptr;
    require(shards >= 1 && shard >= 0 && shard < shards, FSTK_E_PARAMETER, "bad shard");
    require(cfg->transform >= 0 && cfg->transform <= 3, FSTK_E_PARAMETER,
            "transform must be dct, wht, fft or none");
    // PointCloud::from_data (ingest.cpp:19-31) validation happens first.
    require(d >= 1 && d <= kMaxOrder, FSTK_E_SHAPE, "point cloud dimension must be in [1, 8]");
    require(q >= 1, FSTK_E_DATA, "point cloud is empty");
    auto rf = std::make_unique<fstk_gpu_refit>();
    rf->model = m;
    rf->device = m->device;
    rf->cfg = *cfg;
    rf->shard = shard;
    rf->shards = shards;
    rf->q = q;
    rf->d = d;
    rf->R = m->R;
    DeviceGuard dg(m->device);
    FSTK_CUDA(cudaStreamCreateWithFlags(&rf->stream, cudaStreamNonBlocking));
    cudaStream_t s = rf->stream;
    EventTimer tprep(s);
    // FSTK_DEBUG_TIMING=1: host wall time per prepare phase (stream synced).
    static const bool dbg_timing = std::getenv("FSTK_DEBUG_TIMING") != nullptr;
    auto tmark = std::chrono::steady_clock::now();
    auto mark = [&](const char* what) {
      if (!dbg_timing) return;
      cudaStreamSynchronize(s);
      const auto now = std::chrono::steady_clock::now();
      std::fprintf(stderr, "fstk prepare: %-22s %8.2f ms\n", what,
                   std::chrono::duration<double, std::milli>(now - tmark).count());
      tmark = now;
    };
    // PointCloud::from_data (ingest.cpp:19-31): every coordinate and value
    // must be finite -- checked on the host (all cores) so that only the
    // rows the refit reads (working subset + validation) travel to the GPU.
    {
      const bool ok_p = all_finite(points, static_cast<size_t>(q) * d);
      const bool ok_v = all_finite(values, static_cast<size_t>(q));
      require(ok_p, FSTK_E_DATA, "point coordinates must be finite");
      require(ok_v, FSTK_E_DATA, "sample values must be finite");
    }
    mark("finite check");
    // reestimate_core (randls.cpp:363-368)
    const uint64_t S = resolve_sample_rows(cfg->sample_rows, m->R);
    require(S > static_cast<uint64_t>(m->R), FSTK_E_PARAMETER,
            "sample rows must exceed the core size");
    require(static_cast<uint64_t>(q) >= S, FSTK_E_PARAMETER,
            "dataset smaller than the requested sketch");
    // prepare (randls.cpp:246-311)
    require(d == m->d, FSTK_E_SHAPE, "dataset/model dimension mismatch");
    const uint64_t uq = static_cast<uint64_t>(q);
    uint64_t n_val = 0;
    if (cfg->validation_fraction > 0.0) {
      n_val = static_cast<uint64_t>(std::llround(cfg->validation_fraction * static_cast<double>(uq)));
      n_val = std::min<uint64_t>(std::min(n_val, uq - 1), 100000);
    }
    // Validation rows (sorted) and the training rows = their complement in
    // ascending order, never materialised: train_at() maps sorted positions
    // into the complement by one merge against `val`.
    rf->held_out = n_val >= 1;
    const uint64_t n_train = uq - n_val;  // sample_without_replacement returns n_val < q rows
    const uint64_t q_w = cfg->working_subset == 0
                             ? n_train
                             : std::min<uint64_t>(cfg->working_subset, n_train);
    require(q_w >= 1, FSTK_E_PARAMETER, "no training points left");
    rf->q_w = q_w;
    rf->S = S;
    rf->none = cfg->transform == FSTK_TRANSFORM_NONE;
    // The three host RNG streams are independent (mix_seed tags), so the
    // sketch plan and the transform-order inputs built from it (solve_sketched,
    // randls.cpp:318: plan seeded with mix_seed(seed, kSketchTag)) are made on
    // a second host thread while this one draws the validation rows and the
    // working subset and uploads them.  Same draws, same results; a plan error
    // is rethrown after the join.
    std::exception_ptr plan_err;
    std::thread planner([&, dev = m->device] {
      try {
        FSTK_CUDA(cudaSetDevice(dev));
        rf->plan = rf->none ? make_plan_none(q_w, S, mix_seed(cfg->seed, kSketchTag))
                            : make_plan(q_w, S, mix_seed(cfg->seed, kSketchTag));
        require(rf->plan.q_pad < (uint64_t(1) << 31), FSTK_E_PARAMETER, "working subset too large");
        // Inputs in transform order; destination rows in last-pass visit order.
        if (!rf->none)
          build_inputs(cfg->transform, rf->plan.q_pad, q_w, rf->plan.signs, rf->plan.rows, false, {},
                       true, rf->in, s);
      } catch (...) {
        plan_err = std::current_exception();
      }
    });
    struct Joiner {
      std::thread& t;
      ~Joiner() {
        if (t.joinable()) t.join();
      }
    } joiner{planner};
    std::vector<uint64_t> val;
    if (rf->held_out) {
      Rng rng(mix_seed(cfg->seed, kValidationTag));
      val = rng.sample_without_replacement(uq, n_val);
    }
    auto complement_of = [&](const std::vector<uint64_t>& pos) {
      std::vector<int64_t> outv(pos.size());
      uint64_t vi = 0;
      for (size_t t = 0; t < pos.size(); ++t) {
        uint64_t x = pos[t] + vi;
        while (vi < val.size() && val[vi] <= x) x = pos[t] + ++vi;
        outv[t] = static_cast<int64_t>(x);
      }
      return outv;
    };
    mark("validation split");
    std::vector<int64_t> subset;  // dataset rows of the working subset, ascending
    if (q_w == n_train) {
      std::vector<uint64_t> all(n_train);
      std::iota(all.begin(), all.end(), 0);
      subset = complement_of(all);
    } else {
      Rng rng(mix_seed(cfg->seed, kSubsetTag));
      subset = complement_of(rng.sample_without_replacement(n_train, q_w));
    }
    if (!rf->held_out) {  // no held-out points: validate on the training rows
      val.resize(n_train);  // == q: every row
      std::iota(val.begin(), val.end(), 0);
    }
    mark("working subset");
    // Compact upload: subset rows (in subset order) and validation rows.
    rf->subset = subset;
    rf->d_points.alloc(static_cast<size_t>(q_w) * d);
    rf->d_values.alloc(static_cast<size_t>(q_w));
    rf->n_val = static_cast<int64_t>(val.size());
    rf->val_points.alloc(static_cast<size_t>(std::max<int64_t>(rf->n_val, 1)) * d);
    rf->val_values.alloc(static_cast<size_t>(std::max<int64_t>(rf->n_val, 1)));
    {
      const int64_t nv = rf->n_val;
      // Gathered straight into a process-wide pinned staging buffer (grow-only,
      // one refit at a time uses it), so the upload is a plain DMA.
      const size_t nst = static_cast<size_t>(q_w) * (d + 1);
      std::unique_lock<std::mutex> stage_lock(g_stage_mu);
      if (g_stage_n < nst) {
        if (g_stage) cudaFreeHost(g_stage);
        g_stage = nullptr;
        g_stage_n = 0;
        FSTK_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&g_stage), nst * sizeof(double),
                                cudaHostAllocPortable));
        g_stage_n = nst;
      }
      double* hp = g_stage;
      double* hv = g_stage + static_cast<size_t>(q_w) * d;
      std::vector<double> vp(static_cast<size_t>(nv) * d);
      rf->h_val_values.resize(nv);
      rf->h_val_index.resize(nv);
      parallel_chunks(q_w, [&](uint64_t lo, uint64_t hi) {
        for (int k = 0; k < d; ++k) {
          const double* col = points + static_cast<int64_t>(k) * q;
          double* dst = hp + static_cast<size_t>(k) * q_w;
          for (uint64_t t = lo; t < hi; ++t) dst[t] = col[subset[t]];
        }
        for (uint64_t t = lo; t < hi; ++t) hv[t] = values[subset[t]];
      });
      for (int k = 0; k < d; ++k) {
        const double* col = points + static_cast<int64_t>(k) * q;
        double* vdst = vp.data() + static_cast<size_t>(k) * nv;
        for (int64_t t = 0; t < nv; ++t) vdst[t] = col[val[t]];
      }
      for (int64_t t = 0; t < nv; ++t) {
        rf->h_val_index[t] = static_cast<int64_t>(val[t]);
        rf->h_val_values[t] = values[val[t]];
      }
      FSTK_CUDA(cudaMemcpyAsync(rf->d_points.p, hp, static_cast<size_t>(q_w) * d * 8,
                                cudaMemcpyHostToDevice, s));
      FSTK_CUDA(cudaMemcpyAsync(rf->d_values.p, hv, static_cast<size_t>(q_w) * 8,
                                cudaMemcpyHostToDevice, s));
      if (nv > 0) {
        FSTK_CUDA(cudaMemcpyAsync(rf->val_points.p, vp.data(), vp.size() * 8,
                                  cudaMemcpyHostToDevice, s));
        FSTK_CUDA(cudaMemcpyAsync(rf->val_values.p, rf->h_val_values.data(), nv * 8,
                                  cudaMemcpyHostToDevice, s));
      }
      FSTK_CUDA(cudaStreamSynchronize(s));
    }
    mark("compact upload");
    planner.join();
    if (plan_err) std::rethrow_exception(plan_err);
    rf->q_pad = rf->plan.q_pad;
    mark("sketch plan + inputs");
    rf->row_lo = static_cast<int64_t>(S) * shard / shards;
    rf->row_hi = static_cast<int64_t>(S) * (shard + 1) / shards;
    rf->local_rows = rf->row_hi - rf->row_lo;
    if (rf->none) {
      // Tables and rhs of this shard's sampled rows only; A is generated on demand.
      const int64_t nl = rf->local_rows;
      std::vector<int64_t> src(static_cast<size_t>(std::max<int64_t>(nl, 1)));
      for (int64_t i = 0; i < nl; ++i) src[i] = static_cast<int64_t>(rf->plan.rows[rf->row_lo + i]);
      DevBuf<int64_t> dsrc(src.size());
      FSTK_CUDA(cudaMemcpyAsync(dsrc.p, src.data(), src.size() * 8, cudaMemcpyHostToDevice, s));
      rf->ldt = round_up(std::max<int64_t>(nl, 1), 128);
      int64_t tot = 0;
      for (int k = 0; k < d; ++k) {
        rf->toff[k] = tot;
        tot += m->ranks[k] * rf->ldt;
      }
      rf->tables.alloc(static_cast<size_t>(tot));
      DevBuf<unsigned long long> derr(1);
      FSTK_CUDA(cudaMemsetAsync(derr.p, 0xff, 8, s));
      launch_mode_tables(m, rf->d_points.p, static_cast<int64_t>(q_w), nl, rf->ldt, dsrc.p, rf->tables.p, rf->toff,
                         rf->ldt, true, derr.p, s);
      rf->b.alloc(static_cast<size_t>(std::max<int64_t>(nl, 1)));
      if (nl > 0) {
        scaled_gather_kernel<<<static_cast<unsigned>(ceil_div(nl, 256)), 256, 0, s>>>(
            rf->d_values.p, dsrc.p, nl, rf->plan.scale, rf->b.p);
        check_launch("scaled_gather_kernel");
      }
      unsigned long long bad = 0;
      FSTK_CUDA(cudaMemcpyAsync(&bad, derr.p, 8, cudaMemcpyDeviceToHost, s));
      FSTK_CUDA(cudaStreamSynchronize(s));
      if (bad != ULLONG_MAX) {
        const int64_t row = subset[src[bad]];
        std::vector<double> y(d);
        for (int k = 0; k < d; ++k) y[k] = points[k * q + row];
        throw_domain(m, row, y.data());
      }
      if (info) {
        info->t_prepare = tprep.seconds();
        info->t_sketch = 0.0;
        info->sample_rows = S;
        info->working_rows = q_w;
        info->padded_rows = rf->q_pad;
        info->held_out = rf->held_out ? 1 : 0;
      }
      *out = rf.release();
      return;
    }
    // Mode tables over the padded positions, bit-exact (mode_value_tables, randls.cpp:21-41).
    int64_t toff[kMaxOrder], tot = 0;
    const int64_t ldt = static_cast<int64_t>(rf->q_pad);
    for (int k = 0; k < d; ++k) {
      toff[k] = tot;
      tot += m->ranks[k] * ldt;
    }
    DevBuf<double> tables(static_cast<size_t>(tot));
    DevBuf<unsigned long long> derr(1);
    FSTK_CUDA(cudaMemsetAsync(derr.p, 0xff, 8, s));
    launch_mode_tables(m, rf->d_points.p, static_cast<int64_t>(q_w), static_cast<int64_t>(rf->q_pad),
                       static_cast<int64_t>(rf->q_pad), rf->in.row_src.p, tables.p, toff, ldt,
                       true, derr.p, s);
    fold_sign_kernel<<<static_cast<unsigned>(ceil_div(ldt, 256)), 256, 0, s>>>(
        tables.p + toff[0], ldt, static_cast<int>(m->ranks[0]), rf->in.sgn.p, ldt);
    check_launch("fold_sign_kernel");
    unsigned long long bad = 0;
    FSTK_CUDA(cudaMemcpyAsync(&bad, derr.p, 8, cudaMemcpyDeviceToHost, s));
    FSTK_CUDA(cudaStreamSynchronize(s));
    if (bad != ULLONG_MAX) {
      // Map the failing table row back to the dataset row.
      int64_t src = -1;
      FSTK_CUDA(cudaMemcpy(&src, rf->in.row_src.p + bad, 8, cudaMemcpyDeviceToHost));
      src = subset[src];
      std::vector<double> y(d);
      for (int k = 0; k < d; ++k) y[k] = points[k * q + src];
      throw_domain(m, src, y.data());
    }
    mark("mode tables");
    if (info) info->t_prepare = tprep.seconds();
    // Sketch.  Row-sharded: all R design columns plus the rhs, this shard
    // keeps its rows.  Column-sharded: this shard's columns of the R + 1
    // (rhs last), every sample row, written packed per destination rank for
    // one all-to-all (exchange_layout / adopt_rows).
    const bool fft = cfg->transform == FSTK_TRANSFORM_FFT;
    const int64_t arows = fft ? 2 * rf->local_rows : rf->local_rows;
    const int fft2 = fft ? 2 : 1;
    rf->columns = columns;
    if (columns) {
      require(shards <= kMaxShards, FSTK_E_PARAMETER, "column-sharded refit: at most 32 shards");
      const int64_t nc = m->R + 1;
      rf->c_lo = nc * shard / shards;
      rf->c_hi = nc * (shard + 1) / shards;
      int64_t off = 0;
      for (int h = 0; h < shards; ++h) {
        const int64_t lo = static_cast<int64_t>(S) * h / shards, hi = static_cast<int64_t>(S) * (h + 1) / shards;
        rf->pk_base[h] = off;
        off += (rf->c_hi - rf->c_lo) * fft2 * (hi - lo);
      }
      const auto ta = std::chrono::steady_clock::now();
      rf->send.alloc(static_cast<size_t>(std::max<int64_t>(off, 1)));
      if (info)
        info->t_alloc = std::chrono::duration<double>(std::chrono::steady_clock::now() - ta).count();
    } else {
      const auto ta = std::chrono::steady_clock::now();
      rf->A.alloc(static_cast<size_t>(std::max<int64_t>(arows, 1)) * m->R);
      rf->b.alloc(static_cast<size_t>(std::max<int64_t>(arows, 1)));
      if (info)
        info->t_alloc = std::chrono::duration<double>(std::chrono::steady_clock::now() - ta).count();
    }
    (void)twiddles(m->device, rf->q_pad);  // host replay cached outside the timed region
    EventTimer tsk(s);
    SketchJob J{};
    J.kind = cfg->transform;
    J.n = rf->q_pad;
    J.src = SRC_TABLES;
    J.tables = tables.p;
    for (int k = 0; k < d; ++k) {
      J.toff[k] = toff[k];
      J.r[k] = static_cast<int>(m->ranks[k]);
    }
    J.ldt = ldt;
    J.d = d;
    J.rhs = rf->d_values.p;
    J.R = m->R;
    J.with_rhs = true;
    J.sgn = rf->in.sgn.p;
    J.row_src = rf->in.row_src.p;
    J.slot = rf->in.slot.p;
    J.compact = true;
    J.lo_start = rf->in.lo_start.p;
    J.t_list = rf->in.t_list.p;
    J.post_re = rf->in.post_re.p;
    J.post_im = rf->in.post_im.p;
    J.post_c = rf->in.post_c.p;
    J.scale = rf->plan.scale;
    J.row_lo = rf->row_lo;
    J.row_hi = rf->row_hi;
    J.im_off = rf->local_rows;
    J.A = rf->A.p;
    J.lda = arows;
    J.b = rf->b.p;
    if (columns) {
      J.col_lo = rf->c_lo;
      J.col_hi = rf->c_hi;
      J.packed = true;
      J.nshards = shards;
      J.S = static_cast<int64_t>(S);
      for (int h = 0; h <= shards; ++h) J.shard_lo[h] = static_cast<int64_t>(S) * h / shards;
      for (int h = 0; h < shards; ++h) J.pk_base[h] = rf->pk_base[h];
      J.A = rf->send.p;
      J.row_lo = 0;
      J.row_hi = static_cast<int64_t>(S);
    }
    run_sketch(m->device, J, s);
    if (info) info->t_sketch = tsk.seconds();
    FSTK_CUDA(cudaStreamSynchronize(s));
    if (info) {
      info->sample_rows = S;
      info->working_rows = q_w;
      info->padded_rows = rf->q_pad;
      info->held_out = rf->held_out ? 1 : 0;
    }
    *out = rf.release();
  });
}
}  // namespace fstk_gpu

// Host-only diagnostics of the bit-exact RNG replay (no device work; callable
// without a GPU): rng.cpp sample_without_replacement seeded like
// Rng(seed), and make_plan (randls.cpp:54-75).
int32_t fstk_gpu_sample_without_replacement(uint64_t seed, uint64_t n, uint64_t k,
                                            uint64_t* out, fstk_gpu_error* err) {
  using namespace fstk_gpu;
  return guarded(err, [&] {
    require(out || std::min(n, k) == 0, FSTK_E_PARAMETER, "null argument");
    Rng rng(seed);
    const auto v = rng.sample_without_replacement(n, k);
    std::copy(v.begin(), v.end(), out);
  });
}

int32_t fstk_gpu_make_plan(uint64_t q_w, uint64_t s, uint64_t seed, double* signs,
                           uint64_t* rows, double* scale, uint64_t* q_pad, fstk_gpu_error* err) {
  using namespace fstk_gpu;
  return guarded(err, [&] {
    const Plan p = make_plan(q_w, s, seed);
    if (q_pad) *q_pad = p.q_pad;
    if (scale) *scale = p.scale;
    if (signs) std::copy(p.signs.begin(), p.signs.end(), signs);
    if (rows) std::copy(p.rows.begin(), p.rows.end(), rows);
  });
}

int32_t fstk_gpu_refit_begin(const fstk_gpu_model* m, const double* points, const double* values,
                             int64_t q, int32_t d, const fstk_sketch_cfg* cfg, int32_t shard,
                             int32_t shards, fstk_gpu_refit** out, fstk_reestimate_info* info,
                             fstk_gpu_error* err) {
  const int32_t rc = fstk_gpu::refit_begin_impl(m, points, values, q, d, cfg, shard, shards, false, out,
                                                info, err);
  fstk_gpu::debug_alloc_report("begin");
  return rc;
}

int32_t fstk_gpu_refit_begin_columns(const fstk_gpu_model* m, const double* points,
                                     const double* values, int64_t q, int32_t d,
                                     const fstk_sketch_cfg* cfg, int32_t shard, int32_t shards,
                                     fstk_gpu_refit** out, fstk_reestimate_info* info,
                                     fstk_gpu_error* err) {
  // transform = none has no transform to shard: its rows are generated locally.
  const bool cols = cfg && cfg->transform != FSTK_TRANSFORM_NONE;
  return fstk_gpu::refit_begin_impl(m, points, values, q, d, cfg, shard, shards, cols, out, info,
                                    err);
}

int32_t fstk_gpu_refit_exchange_layout(fstk_gpu_refit* rf, double** send, int64_t* send_counts,
                                       double** recv, int64_t* recv_counts, fstk_gpu_error* err) {
  using namespace fstk_gpu;
  return guarded(err, [&] {
    require(rf && send && send_counts && recv && recv_counts, FSTK_E_PARAMETER, "null argument");
    require(rf->columns && !rf->exchanged, FSTK_E_PARAMETER,
            "exchange_layout: not a column-sharded refit awaiting its exchange");
    DeviceGuard dg(rf->device);
    const int fft2 = rf->cfg.transform == FSTK_TRANSFORM_FFT ? 2 : 1;
    const int64_t arows = fft2 * rf->local_rows;
    const int G = rf->shards;
    const int64_t nc = rf->R + 1;
    rf->A.alloc(static_cast<size_t>(std::max<int64_t>(arows, 1)) * nc);
    for (int h = 0; h < G; ++h) {
      const int64_t lo = static_cast<int64_t>(rf->S) * h / G, hi = static_cast<int64_t>(rf->S) * (h + 1) / G;
      send_counts[h] = (rf->c_hi - rf->c_lo) * fft2 * (hi - lo);
      // Column block of source g lands at columns [c_lo_g, c_hi_g) of the row
      // slab (column-major, ld = arows): contiguous, in rank order.
      recv_counts[h] = (nc * (h + 1) / G - nc * h / G) * arows;
    }
    *send = rf->send.p;
    *recv = rf->A.p;
  });
}

int32_t fstk_gpu_refit_adopt_rows(fstk_gpu_refit* rf, fstk_gpu_error* err) {
  using namespace fstk_gpu;
  return guarded(err, [&] {
    require(rf, FSTK_E_PARAMETER, "null argument");
    require(rf->columns && !rf->exchanged && rf->A.p, FSTK_E_PARAMETER,
            "adopt_rows: call exchange_layout and complete the all-to-all first");
    DeviceGuard dg(rf->device);
    const int fft2 = rf->cfg.transform == FSTK_TRANSFORM_FFT ? 2 : 1;
    const int64_t arows = fft2 * rf->local_rows;
    rf->b.alloc(static_cast<size_t>(std::max<int64_t>(arows, 1)));
    if (arows > 0)
      FSTK_CUDA(cudaMemcpyAsync(rf->b.p, rf->A.p + rf->R * arows, arows * 8, cudaMemcpyDeviceToDevice,
                                rf->stream));
    FSTK_CUDA(cudaStreamSynchronize(rf->stream));
    rf->send.release();
    rf->exchanged = true;
  });
}

namespace fstk_gpu {

// gram(lower) = beta * gram + A^T A for A (rows x n, lda): column-blocked
// DSYRK on the diagonal blocks + one DGEMM per block row below it.
static void gram_accumulate(cublasHandle_t h, const double* A, int lda, int rows, int n,
                            double* gram, double beta) {
  const double one = 1.0;
  const int nb = n >= 4096 ? 8 : 1;
  for (int bi = 0; bi < nb; ++bi) {
    const int i0 = static_cast<int>(static_cast<int64_t>(n) * bi / nb);
    const int i1 = static_cast<int>(static_cast<int64_t>(n) * (bi + 1) / nb);
    if (cublasDsyrk(h, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, i1 - i0, rows, &one,
                    A + static_cast<int64_t>(lda) * i0, lda, &beta,
                    gram + static_cast<int64_t>(n) * i0 + i0, n) != CUBLAS_STATUS_SUCCESS)
      fail(FSTK_E_COMPUTE, "cublasDsyrk failed");
    count_launch();
    if (i0 > 0) {
      if (cublasDgemm(h, CUBLAS_OP_T, CUBLAS_OP_N, i1 - i0, i0, rows, &one,
                      A + static_cast<int64_t>(lda) * i0, lda, A, lda, &beta, gram + i0,
                      n) != CUBLAS_STATUS_SUCCESS)
        fail(FSTK_E_COMPUTE, "cublasDgemm failed");
      count_launch();
    }
  }
}

// Rows per generated block of A for transform = none (about 1 GB of fp64).
static int64_t none_block_rows(const fstk_gpu_refit* rf, bool sliced = false) {
  // ~1 GB of fp64; 4 GB when the Gram is sliced (longer int8 GEMM K per block).
  const int64_t elems = (int64_t(1) << 27) * (sliced ? 4 : 1);
  const int64_t cap = std::max<int64_t>(1024, elems / std::max<int64_t>(rf->R, 1));
  return std::min<int64_t>(round_up(cap, 128), std::max<int64_t>(rf->local_rows, 1));
}

// ---- transform = none through the Kronecker structure (north_star: A is
// never materialised).  Row i of A is scale * u0(i) (x) KR(i), KR(i) = the
// Khatri-Rao row of modes 1..d-1, so with X = x as an r0 x R/r0 matrix
//   A x  = scale * rowdot(U0, KR X^T)           (one DGEMM + a row dot)
//   A^T y = scale * (diag(y) U0)^T KR           (one DGEMM)
// -- 2 S R flops each instead of regenerating S x R values.  These feed the
// normal equations' rhs and the refinement, which need fp64 accuracy, not the
// design's bit pattern (the Gram's residues use the bit-exact generator).
__global__ void khatri_rao_kernel(const double* __restrict__ tables, Int64x8 toff, int64_t ldt,
                                  int d, Int64x8 ranks, int64_t rows, int64_t Rr,
                                  double* __restrict__ kr) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= rows) return;
  for (int64_t m = blockIdx.y; m < Rr; m += gridDim.y) {
    int64_t rem = m;
    double v = 1.0;
    for (int k = 1; k < d; ++k) {
      const int64_t jk = rem % ranks.v[k];
      rem /= ranks.v[k];
      v *= tables[toff.v[k] + jk * ldt + i];
    }
    kr[m * ldt + i] = v;
  }
}

__global__ void scale_rows_kernel(const double* __restrict__ u0, int64_t ldt, int r0,
                                  const double* __restrict__ y, int64_t rows,
                                  double* __restrict__ out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= rows) return;
  const double yi = y[i];
  for (int j = 0; j < r0; ++j) out[j * ldt + i] = u0[j * ldt + i] * yi;
}

__global__ void row_dot_kernel(const double* __restrict__ u0, const double* __restrict__ Y,
                               int64_t ldt, int r0, int64_t rows, double scale,
                               const double* __restrict__ b, double* __restrict__ out) {
  // out_i = b_i - scale * sum_j U0[i, j] Y[i, j]  (b may be null: out_i = scale * dot)
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= rows) return;
  double acc = 0.0;
  for (int j = 0; j < r0; ++j) acc = fma(u0[j * ldt + i], Y[j * ldt + i], acc);
  out[i] = b ? b[i] - scale * acc : scale * acc;
}

static const double* none_kr(fstk_gpu_refit* rf) {
  const fstk_gpu_model* m = rf->model;
  const int64_t rows = rf->local_rows;
  const int64_t Rr = rf->R / m->ranks[0];
  if (!rf->kr.p) {
    rf->kr.alloc(static_cast<size_t>(std::max<int64_t>(rf->ldt, 1)) * Rr);
    FSTK_CUDA(cudaMemsetAsync(rf->kr.p, 0, rf->kr.n * 8, rf->stream));
    if (rows > 0) {
      Int64x8 to{}, rk{};
      for (int k = 0; k < m->d; ++k) {
        to.v[k] = rf->toff[k];
        rk.v[k] = m->ranks[k];
      }
      dim3 g(static_cast<unsigned>(ceil_div(rows, 256)), static_cast<unsigned>(std::min<int64_t>(Rr, 4096)));
      khatri_rao_kernel<<<g, 256, 0, rf->stream>>>(rf->tables.p, to, rf->ldt, m->d, rk, rows, Rr,
                                                   rf->kr.p);
      check_launch("khatri_rao_kernel");
    }
  }
  return rf->kr.p;
}

// out (R) = A_local^T y (y: local rows); beta = 0 overwrite.
static void none_At(fstk_gpu_refit* rf, const double* y, double* out) {
  const fstk_gpu_model* m = rf->model;
  const int64_t rows = rf->local_rows;
  const int r0 = static_cast<int>(m->ranks[0]);
  const int64_t Rr = rf->R / r0;
  cudaStream_t s = rf->stream;
  if (rows == 0) {
    FSTK_CUDA(cudaMemsetAsync(out, 0, static_cast<size_t>(rf->R) * 8, s));
    return;
  }
  const double* kr = none_kr(rf);
  rf->kr_tmp.ensure(static_cast<size_t>(rf->ldt) * r0);
  DevBuf<double>& uy = rf->kr_tmp;
  FSTK_CUDA(cudaMemsetAsync(uy.p, 0, uy.n * 8, s));
  scale_rows_kernel<<<static_cast<unsigned>(ceil_div(rows, 256)), 256, 0, s>>>(
      rf->tables.p + rf->toff[0], rf->ldt, r0, y, rows, uy.p);
  check_launch("scale_rows_kernel");
  Handles& h = handles(rf->device);
  cublasSetStream(h.blas, s);
  const double sc = rf->plan.scale, zero = 0.0;
  if (cublasDgemm(h.blas, CUBLAS_OP_T, CUBLAS_OP_N, r0, static_cast<int>(Rr), static_cast<int>(rows),
                  &sc, uy.p, static_cast<int>(rf->ldt), kr, static_cast<int>(rf->ldt), &zero, out,
                  r0) != CUBLAS_STATUS_SUCCESS)
    fail(FSTK_E_COMPUTE, "cublasDgemm failed (none A^T y)");
  count_launch();
}

// r (local rows) = b - A_local x.
static void none_residual(fstk_gpu_refit* rf, const double* x, double* r) {
  const fstk_gpu_model* m = rf->model;
  const int64_t rows = rf->local_rows;
  const int r0 = static_cast<int>(m->ranks[0]);
  const int64_t Rr = rf->R / r0;
  cudaStream_t s = rf->stream;
  if (rows == 0) return;
  const double* kr = none_kr(rf);
  rf->kr_tmp.ensure(static_cast<size_t>(rf->ldt) * r0);
  DevBuf<double>& Y = rf->kr_tmp;
  Handles& h = handles(rf->device);
  cublasSetStream(h.blas, s);
  const double one = 1.0, zero = 0.0;
  // Y (rows x r0) = KR (rows x Rr) * X^T, X = x as r0 x Rr (column-major).
  if (cublasDgemm(h.blas, CUBLAS_OP_N, CUBLAS_OP_T, static_cast<int>(rows), r0, static_cast<int>(Rr),
                  &one, kr, static_cast<int>(rf->ldt), x, r0, &zero, Y.p,
                  static_cast<int>(rf->ldt)) != CUBLAS_STATUS_SUCCESS)
    fail(FSTK_E_COMPUTE, "cublasDgemm failed (none A x)");
  count_launch();
  row_dot_kernel<<<static_cast<unsigned>(ceil_div(rows, 256)), 256, 0, s>>>(
      rf->tables.p + rf->toff[0], Y.p, rf->ldt, r0, rows, rf->plan.scale, rf->b.p, r);
  check_launch("row_dot_kernel");
}

static void generate_design_block(const fstk_gpu_refit* rf, int64_t row0, int64_t nrows,
                                  double* W, int64_t ldw, cudaStream_t s) {
  const fstk_gpu_model* m = rf->model;
  Int64x8 to{}, rk{};
  for (int k = 0; k < m->d; ++k) {
    to.v[k] = rf->toff[k];
    rk.v[k] = m->ranks[k];
  }
  dim3 grid(static_cast<unsigned>(ceil_div(nrows, 256)),
            static_cast<unsigned>(std::min<int64_t>(rf->R, 4096)));
  ProfScope prof(FSTK_PROF_TRANSFORM, s);
  if (m->d == 3)
    design_block_kernel<3><<<grid, 256, 0, s>>>(rf->tables.p, to, rf->ldt, m->d, rk, row0, nrows,
                                                rf->R, rf->plan.scale, W, ldw);
  else if (m->d == 4)
    design_block_kernel<4><<<grid, 256, 0, s>>>(rf->tables.p, to, rf->ldt, m->d, rk, row0, nrows,
                                                rf->R, rf->plan.scale, W, ldw);
  else
    design_block_kernel<0><<<grid, 256, 0, s>>>(rf->tables.p, to, rf->ldt, m->d, rk, row0, nrows,
                                                rf->R, rf->plan.scale, W, ldw);
  check_launch("design_block_kernel");
}

}  // namespace fstk_gpu

namespace fstk_gpu {
// slices < 0: the process setting (gram_slices()); 0: native fp64 Gram;
// 2..7: the sliced Gram at that precision level.
static void normal_equations(fstk_gpu_refit* rf, double* gram, double* rhs,
                             fstk_reestimate_info* info, int slices) {
  {
    require(!rf->columns || rf->exchanged, FSTK_E_PARAMETER,
            "column-sharded refit: exchange_layout, the all-to-all and adopt_rows come first");
    rf->gram_used = 0;
    double i8ops = 0.0;
    DeviceGuard dg(rf->device);
    cudaStream_t s = rf->stream;
    Handles& h = handles(rf->device);
    EventTimer tg(s);
    const bool fft = rf->cfg.transform == FSTK_TRANSFORM_FFT;
    const int64_t arows = fft ? 2 * rf->local_rows : rf->local_rows;
    const int n = static_cast<int>(rf->R);
    cublasSetStream(h.blas, s);
    const double one = 1.0, zero = 0.0;
    if (arows == 0) {
      FSTK_CUDA(cudaMemsetAsync(gram, 0, static_cast<size_t>(n) * n * 8, s));
      FSTK_CUDA(cudaMemsetAsync(rhs, 0, static_cast<size_t>(n) * 8, s));
    } else {
      // Lower triangle of A^T A (column-major R x R) and A^T b.  The triangle
      // is split into nb column blocks: block row i below the diagonal is one
      // DGEMM A_i^T [A_0 .. A_{i-1}] and each diagonal block one DSYRK, so
      // (nb-1)/nb of the flops run in large GEMMs.
      int level = slices < 0 ? gram_slices() : slices;
      // The unmixed estimator's rows are worse conditioned than a mixed
      // sketch's: at C2 a level-2 Gram leaves its first iterate 38% off and
      // contracts 0.09 per step, at the edge of the escalation rule (level 3:
      // 1.9e-2, then 2e-5 and 5e-3).  So is a thinly oversampled sketch: C1's
      // M = 4R system escalates from level 2 and not from level 3 (C2/C5 at
      // 8R and C4 at 16R contract 3e-3 per step or better at level 2).  The
      // process setting therefore means at least level 3 for transform = none
      // and for M < 8R; an explicit level (normal_equations_level) is kept.
      if (slices < 0 && level == 2 && (rf->none || rf->S < 8 * static_cast<uint64_t>(rf->R))) level = 3;
      const bool sliced = level > 0 && gram_sliced_applies(arows, n);
      rf->gram_used = sliced ? level : 0;
      if (rf->none && sliced && gram_scheme_crt()) {
        // A never materialised: CRT residues straight from the mode tables,
        // A^T b through the Kronecker structure.
        ProfScope prof(FSTK_PROF_GRAM, s);
        DesignSpec spec{};
        spec.tables = rf->tables.p;
        for (int k = 0; k < rf->model->d; ++k) {
          spec.toff.v[k] = rf->toff[k];
          spec.ranks.v[k] = rf->model->ranks[k];
        }
        spec.ldt = rf->ldt;
        spec.d = rf->model->d;
        spec.row0 = 0;
        spec.scale = rf->plan.scale;
        i8ops = gram_accumulate_sliced_design(spec, arows, n, gram, 0.0, rf->gram_used, s,
                                              rf->device, rf->gs);
        none_At(rf, rf->b.p, rhs);
        FSTK_CUDA(cudaStreamSynchronize(s));
      } else if (rf->none) {
        // A^T A accumulated over generated row blocks (A never materialised).
        const int64_t BS = none_block_rows(rf, sliced);
        DevBuf<double> W(static_cast<size_t>(BS) * rf->R);
        for (int64_t r0 = 0; r0 < arows; r0 += BS) {
          const int64_t nb_rows = std::min(BS, arows - r0);
          generate_design_block(rf, r0, nb_rows, W.p, BS, s);
          ProfScope prof(FSTK_PROF_GRAM, s);
          const double beta = r0 == 0 ? 0.0 : 1.0;
          if (sliced)
            i8ops += gram_accumulate_sliced(W.p, BS, nb_rows, n, gram, beta, rf->gram_used, 2, s,
                                            rf->device, rf->gs);
          else
            gram_accumulate(h.blas, W.p, static_cast<int>(BS), static_cast<int>(nb_rows), n, gram,
                            beta);
          if (cublasDgemv(h.blas, CUBLAS_OP_T, static_cast<int>(nb_rows), n, &one, W.p,
                          static_cast<int>(BS), rf->b.p + r0, 1, &beta, rhs, 1) !=
              CUBLAS_STATUS_SUCCESS)
            fail(FSTK_E_COMPUTE, "cublasDgemv failed");
          count_launch();
        }
        FSTK_CUDA(cudaStreamSynchronize(s));
      } else {
        ProfScope prof(FSTK_PROF_GRAM, s);
        if (sliced)
          i8ops = gram_accumulate_sliced(rf->A.p, arows, arows, n, gram, 0.0, rf->gram_used, 2, s,
                                         rf->device, rf->gs);
        else
          gram_accumulate(h.blas, rf->A.p, static_cast<int>(arows), static_cast<int>(arows), n,
                          gram, 0.0);
        if (cublasDgemv(h.blas, CUBLAS_OP_T, static_cast<int>(arows), n, &one, rf->A.p,
                        static_cast<int>(arows), rf->b.p, 1, &zero, rhs, 1) != CUBLAS_STATUS_SUCCESS)
          fail(FSTK_E_COMPUTE, "cublasDgemv failed");
        count_launch();
      }
    }
    const double t = tg.seconds();
    if (info) {
      info->t_gram = t;
      info->gram_slices = rf->gram_used;
      info->gram_int8_ops = i8ops;
    }
    // The residue planes and the SYRK scratch (up to 24 GB) are not needed
    // by the solve: return them before the Cholesky allocates its own (an
    // escalation re-forms the Gram from scratch anyway).  The digit scheme
    // keeps its planes for the progressive upgrade.
    if (gram_scheme_crt()) {
      rf->gs.X.release();
      rf->gs.C.release();
      rf->gs.C8.release();
    }
  }
}

}  // namespace fstk_gpu

int32_t fstk_gpu_refit_normal_equations(fstk_gpu_refit* rf, double* gram, double* rhs,
                                        fstk_reestimate_info* info, fstk_gpu_error* err) {
  return guarded(err, [&] {
    require(rf && gram && rhs, FSTK_E_PARAMETER, "null argument");
    normal_equations(rf, gram, rhs, info, -1);
    debug_alloc_report("normal_equations");
  });
}

int32_t fstk_gpu_refit_normal_equations_level(fstk_gpu_refit* rf, int32_t slices, double* gram,
                                              double* rhs, fstk_reestimate_info* info,
                                              fstk_gpu_error* err) {
  return guarded(err, [&] {
    require(rf && gram && rhs, FSTK_E_PARAMETER, "null argument");
    require(slices == 0 || (slices >= 2 && slices <= 7), FSTK_E_PARAMETER,
            "normal_equations_level: slices must be 0 (native) or 2..7");
    normal_equations(rf, gram, rhs, info, slices);
  });
}

int32_t fstk_gpu_refit_normal_equations_native(fstk_gpu_refit* rf, double* gram, double* rhs,
                                               fstk_reestimate_info* info, fstk_gpu_error* err) {
  return guarded(err, [&] {
    require(rf && gram && rhs, FSTK_E_PARAMETER, "null argument");
    normal_equations(rf, gram, rhs, info, 0);
  });
}

int32_t fstk_gpu_gram_slices(int32_t slices) { return fstk_gpu::set_gram_slices(slices); }
int32_t fstk_gpu_gram_engine(int32_t engine) { return fstk_gpu::set_gram_engine(engine); }

int32_t fstk_gpu_gram_device(const double* a, int64_t lda, int64_t rows, int32_t n, double* gram,
                             int32_t slices, int32_t device, void* stream, fstk_gpu_error* err) {
  using namespace fstk_gpu;
  return guarded(err, [&] {
    require(a && gram, FSTK_E_PARAMETER, "null argument");
    require(n > 0 && rows > 0 && lda >= rows, FSTK_E_SHAPE, "gram: need n > 0, rows > 0, lda >= rows");
    require(slices == 0 || (slices >= 2 && slices <= 7), FSTK_E_PARAMETER,
            "gram: slices must be 0 (native fp64) or 2..7");
    require((rows <= INT32_MAX && lda <= INT32_MAX) || slices > 0, FSTK_E_SHAPE,
            "gram: native path needs rows, lda < 2^31");
    DeviceGuard dg(device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (slices > 0) {
      GramScratch sc;
      gram_accumulate_sliced(a, lda, rows, n, gram, 0.0, slices, 2, s, device, sc);
      FSTK_CUDA(cudaStreamSynchronize(s));
      return;
    }
    Handles& h = handles(device);
    cublasSetStream(h.blas, s);
    gram_accumulate(h.blas, a, static_cast<int>(lda), static_cast<int>(rows), n, gram, 0.0);
    FSTK_CUDA(cudaStreamSynchronize(s));
  });
}

// ---- solve: Cholesky of the summed normal equations + iterative refinement
// against the sketched system itself (corrected semi-normal equations), which
// converges to the least-squares solution the reference's QR computes
// (randls.cpp:112-123) with O(cond(A) eps) instead of O(cond(A)^2 eps) error.
namespace fstk_gpu {

// R of [A b] over this shard's sketched rows (streaming TSQR, fstk_rank.cu):
// A is copied block by block into the fold scratch (or, for transform =
// none, generated there), so the sketch itself is left intact.
static void refit_local_qr(fstk_gpu_refit* rf, QrStream& qs) {
  cudaStream_t s = rf->stream;
  const bool fft = rf->cfg.transform == FSTK_TRANSFORM_FFT;
  const int64_t arows = fft ? 2 * rf->local_rows : rf->local_rows;
  const int n = static_cast<int>(rf->R), n1 = n + 1;
  size_t freeb = 0, totb = 0;
  FSTK_CUDA(device_mem_info(&freeb, &totb));
  // Row blocks of at least n1 rows, the scratch within a quarter of the free memory.
  const int64_t budget_rows = static_cast<int64_t>(freeb / 4 / (static_cast<size_t>(n1) * 8)) - n1;
  const int64_t bmax = std::max<int64_t>(1, std::min<int64_t>(std::max<int64_t>(arows, 1),
                                                              std::max<int64_t>(n1, budget_rows)));
  qs.init(n1, bmax, s, rf->device);
  for (int64_t r0 = 0; r0 < arows; r0 += bmax) {
    const int64_t rows = std::min(bmax, arows - r0);
    if (rf->none)
      generate_design_block(rf, r0, rows, qs.block(), qs.ldw, s);
    else
      FSTK_CUDA(cudaMemcpy2DAsync(qs.block(), qs.ldw * 8, rf->A.p + r0, arows * 8, rows * 8, n,
                                  cudaMemcpyDeviceToDevice, s));
    FSTK_CUDA(cudaMemcpyAsync(qs.block() + static_cast<int64_t>(n) * qs.ldw, rf->b.p + r0, rows * 8,
                              cudaMemcpyDeviceToDevice, s));
    qs.fold(rows);
  }
  FSTK_CUDA(cudaStreamSynchronize(s));
}

// Gram-side certificate of full rank in the reference's sense.  After the
// refinement x += (L L^T)^{-1} A^T (b - A x) has converged, the eigenvalues of
// (L L^T)^{-1} A^T A lie in [1 - q, 1 + q] with q <= 1/2 (a flatter step ratio
// is not accepted as convergence), so sigma_min(A)^2 >= lambda_min(L L^T) / 2.
// Every |R_ii| of a pivoted QR of A is >= sigma_min(A), and its largest pivot
// |R_00| is the largest column norm sqrt(max_j G_jj); so sigma_min(A) >
// R eps max_j ||A_j|| (with a 100x margin for the power-iteration estimate)
// means ColPivHouseholderQR::rank() == R.  Returns sigma_min / max col norm.
// lam: the lambda_min(L L^T) estimate (< 0: computed here, synchronously).
static double refit_sigma_ratio(fstk_gpu_refit* rf, const double* gram, double lam = -1.0) {
  const int n = static_cast<int>(rf->R);
  cudaStream_t s = rf->stream;
  if (lam < 0.0) lam = chol_lambda_min_estimate(rf->L.p, n, 3, s, rf->device);
  std::vector<double> diag(n);
  FSTK_CUDA(cudaMemcpy2DAsync(diag.data(), 8, gram, static_cast<size_t>(n + 1) * 8, 8, n,
                              cudaMemcpyDeviceToHost, s));
  FSTK_CUDA(cudaStreamSynchronize(s));
  double mx = 0.0;
  for (double v : diag) mx = std::max(mx, v);
  if (!(mx > 0.0) || !(lam > 0.0)) return 0.0;
  return std::sqrt(0.5 * lam / mx);
}
static bool certified_full_rank(const fstk_gpu_refit* rf, double ratio) {
  return ratio > 100.0 * static_cast<double>(rf->R) * 2.220446049250313e-16;
}

// The reference's own decision (randls.cpp:112-123) on this shard's rows:
// TSQR, pivoted QR, Eigen's rank rule, QR or COD solution.  One shard only;
// sharded refits stack their factors first (fstk_gpu_qr_stack).
static void exact_solve(fstk_gpu_refit* rf, double* x_dev) {
  QrStream qs;
  refit_local_qr(rf, qs);
  bool def = false;
  cpqr_solve(qs.W.p, qs.ldw, static_cast<int>(rf->R), rf->R, x_dev, &def, rf->stream, rf->device);
  rf->rank_def = def;
}

// Session accessors for the single-process multi-device orchestrator
// (fstk_multi.cu).
extern "C++" {
int refit_device(const fstk_gpu_refit* rf) { return rf->device; }
int64_t refit_order(const fstk_gpu_refit* rf) { return rf->R; }
bool refit_awaits_exchange(const fstk_gpu_refit* rf) { return rf->columns && !rf->exchanged; }
int refit_gram_used(const fstk_gpu_refit* rf) { return rf->gram_used; }
bool refit_is_factored(const fstk_gpu_refit* rf) { return rf->factored; }
}  // extern "C++"

// Re-raises a failed nested C-ABI stage with its full error record.
static void rethrow_stage(int32_t c, const fstk_gpu_error* err) {
  if (!c) return;
  Error e{c, err ? err->message : "refit stage failed"};
  if (err) {
    e.index = err->index;
    e.mode = err->mode;
    e.value = err->value;
  }
  throw e;
}

static double dev_norm(cublasHandle_t h, int n, const double* x) {
  double r = 0.0;
  if (cublasDnrm2(h, n, x, 1, &r) != CUBLAS_STATUS_SUCCESS) fail(FSTK_E_COMPUTE, "cublasDnrm2 failed");
  return r;
}

}  // namespace fstk_gpu

// ---- blocked Cholesky with int8 tensor-core trailing updates (chol_crt) ----
namespace fstk_gpu {
// T (b x m, column-major, ld b) = L21^T for L21 = m x b at L (ld ldl).
__global__ void transpose_panel_kernel(const double* __restrict__ L, int64_t ldl, int m, int b,
                                       double* __restrict__ T) {
  __shared__ double tile[32][33];
  const int a0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int a = a0 + threadIdx.x, r = r0 + y;
    if (a < m && r < b) tile[y][threadIdx.x] = L[a + static_cast<int64_t>(r) * ldl];
  }
  __syncthreads();
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int r = r0 + threadIdx.x, a = a0 + y;
    if (a < m && r < b) T[r + static_cast<int64_t>(a) * b] = tile[threadIdx.x][y];
  }
}

// Lower Cholesky factor of the n x n matrix G (column-major, ld n) in place,
// right-looking in panels of nb: cuSOLVER potrf of the diagonal block, DTRSM
// of the panel below it, and the trailing update G22 -= L21 L21^T through the
// CRT int8 tensor-core Gram at `slices` plane-accuracy (the Gram machinery of
// fstk_gram.cu with K = nb).  The factor preconditions the refinement
// against A, which restores fp64 accuracy whatever the factor's rounding; at
// R = 32,768 the DMMA-bound potrf's 1.2e13 flops are 88% trailing updates.
// Returns false when a diagonal block is not positive definite.
static bool chol_crt(cublasHandle_t blas, cusolverDnHandle_t solver, double* G, int n, int nb,
                     int slices, cudaStream_t s, int device) {
  // Lookahead: the trailing update runs on s in column blocks, the next
  // panel's columns first; once those are folded (an event from
  // gram_update_crt) the next panel's potrf, DTRSM and transpose run on a
  // second stream beside the rest of the update (fp64 pipe and DTRSM beside
  // int8 MMAs and HBM-bound folds).  FSTK_CHOL_LOOKAHEAD=0 keeps one stream.
  static const bool lookahead = [] {
    const char* e = std::getenv("FSTK_CHOL_LOOKAHEAD");
    return !(e && std::atoi(e) == 0);
  }();
  struct Side {
    cudaStream_t st = nullptr;
    cudaEvent_t panel = nullptr, block = nullptr, done = nullptr;
    ~Side() {
      if (panel) cudaEventDestroy(panel);
      if (block) cudaEventDestroy(block);
      if (done) cudaEventDestroy(done);
      if (st) cudaStreamDestroy(st);
    }
  } side;
  if (lookahead) {
    FSTK_CUDA(cudaStreamCreateWithFlags(&side.st, cudaStreamNonBlocking));
    FSTK_CUDA(cudaEventCreateWithFlags(&side.panel, cudaEventDisableTiming));
    FSTK_CUDA(cudaEventCreateWithFlags(&side.block, cudaEventDisableTiming));
    FSTK_CUDA(cudaEventCreateWithFlags(&side.done, cudaEventDisableTiming));
  }
  const cudaStream_t sp = lookahead ? side.st : s;  // panel stream
  const int npan = (n + nb - 1) / nb;
  int lwork = 0;
  if (cusolverDnDpotrf_bufferSize(solver, CUBLAS_FILL_MODE_LOWER, nb, G, n, &lwork) !=
      CUSOLVER_STATUS_SUCCESS)
    fail(FSTK_E_COMPUTE, "potrf_bufferSize failed");
  DevBuf<double> work(std::max(lwork, 1));
  DevBuf<int> dinfo(npan);
  FSTK_CUDA(cudaMemsetAsync(dinfo.p, 0, npan * sizeof(int), s));
  // Two transposed panels: the update of panel p still reads T[p & 1] while
  // the lookahead writes panel p + 1's.
  const size_t tsz = static_cast<size_t>(nb) * std::max(n - nb, 1);
  DevBuf<double> T(lookahead ? 2 * tsz : tsz);
  GramScratch sc;
  const double one = 1.0;
  cublasSetStream(blas, sp);
  cusolverDnSetStream(solver, sp);
  if (lookahead) {  // the panel stream starts after what s holds so far (the copy of G)
    FSTK_CUDA(cudaEventRecord(side.done, s));
    FSTK_CUDA(cudaStreamWaitEvent(sp, side.done, 0));
  }
  // Panel p: potrf of the diagonal block, DTRSM of the block column below it,
  // and its transpose, on the panel stream.
  auto panel = [&](int p) {
    const int i0 = p * nb, b = std::min(nb, n - i0), rest = n - i0 - b;
    double* Gii = G + static_cast<int64_t>(i0) * n + i0;
    if (cusolverDnDpotrf(solver, CUBLAS_FILL_MODE_LOWER, b, Gii, n, work.p, lwork, dinfo.p + p) !=
        CUSOLVER_STATUS_SUCCESS)
      fail(FSTK_E_COMPUTE, "potrf failed");
    if (rest == 0) return;
    double* A21 = Gii + b;
    if (cublasDtrsm(blas, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T,
                    CUBLAS_DIAG_NON_UNIT, rest, b, &one, Gii, n, A21, n) != CUBLAS_STATUS_SUCCESS)
      fail(FSTK_E_COMPUTE, "cublasDtrsm failed");
    dim3 tg(static_cast<unsigned>(ceil_div(rest, 32)), static_cast<unsigned>(ceil_div(b, 32)));
    transpose_panel_kernel<<<tg, dim3(32, 8), 0, sp>>>(A21, n, rest, b, T.p + (lookahead ? (p & 1) * tsz : 0));
    check_launch("transpose_panel_kernel");
    count_launch(2);
  };
  // FSTK_DEBUG_TIMING: device time between the ends of consecutive trailing
  // updates (events on s), and the host time spent enqueueing each.
  static const bool dbg_chol = std::getenv("FSTK_DEBUG_TIMING") != nullptr;
  std::vector<cudaEvent_t> pev;
  std::vector<double> host_ms;
  auto stamp = [&] {
    if (!dbg_chol) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, s);
    pev.push_back(e);
  };
  stamp();
  panel(0);
  for (int p = 0; p < npan; ++p) {
    const auto th0 = std::chrono::steady_clock::now();
    struct HostStamp {
      std::vector<double>& v;
      std::chrono::steady_clock::time_point t0;
      bool on;
      ~HostStamp() {
        if (on) v.push_back(std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
      }
    } hs{host_ms, th0, dbg_chol};
    if (p > 0) stamp();
    const int i0 = p * nb, b = std::min(nb, n - i0), rest = n - i0 - b;
    if (rest == 0) break;
    double* A22 = G + static_cast<int64_t>(i0 + b) * n + i0 + b;
    const double* Tp = T.p + (lookahead ? (p & 1) * tsz : 0);
    if (!lookahead) {
      gram_update_crt(Tp, b, b, rest, A22, n, slices, s, device, sc);
      count_launch();
      panel(p + 1);
      continue;
    }
    FSTK_CUDA(cudaEventRecord(side.panel, sp));
    FSTK_CUDA(cudaStreamWaitEvent(s, side.panel, 0));  // panel p factored and transposed
    // The next panel needs its nb columns of the trailing matrix final: the
    // update's first column block when that is wide enough (the panel is then
    // enqueued from inside the update, ahead of its other blocks' launches),
    // else the whole update.
    int64_t bw = 0;
    const int nextb = std::min(nb, rest);
    bool issued = false;
    const std::function<void()> next_panel = [&] {
      FSTK_CUDA(cudaStreamWaitEvent(sp, side.block, 0));
      panel(p + 1);
      issued = true;
    };
    gram_update_crt(Tp, b, b, rest, A22, n, slices, s, device, sc, side.block, &bw, &next_panel, nextb);
    count_launch();
    if (!issued) {
      FSTK_CUDA(cudaEventRecord(side.block, s));
      FSTK_CUDA(cudaStreamWaitEvent(sp, side.block, 0));
      panel(p + 1);
    }
  }
  if (lookahead) {  // s continues after the last panel
    FSTK_CUDA(cudaEventRecord(side.panel, sp));
    FSTK_CUDA(cudaStreamWaitEvent(s, side.panel, 0));
  }
  cublasSetStream(blas, s);
  cusolverDnSetStream(solver, s);
  std::vector<int> hinfo(npan);
  FSTK_CUDA(cudaMemcpyAsync(hinfo.data(), dinfo.p, npan * sizeof(int), cudaMemcpyDeviceToHost, s));
  stamp();
  FSTK_CUDA(cudaStreamSynchronize(s));
  if (dbg_chol && pev.size() > 1) {
    std::string line = "fstk chol panels (device ms | host enqueue ms):";
    for (size_t i = 0; i + 1 < pev.size(); ++i) {
      float ms = 0;
      cudaEventElapsedTime(&ms, pev[i], pev[i + 1]);
      char buf[48];
      std::snprintf(buf, sizeof buf, " %.1f|%.1f", ms, i < host_ms.size() ? host_ms[i] : 0.0);
      line += buf;
    }
    std::fprintf(stderr, "%s\n", line.c_str());
  }
  for (cudaEvent_t e : pev) cudaEventDestroy(e);
  for (int v : hinfo)
    if (v != 0) return false;
  return true;
}

// FSTK_CHOL_CRT: plane-accuracy of chol_crt's trailing updates (0 = cuSOLVER
// dpotrf throughout; default 5), used for R >= 8192.
static int chol_crt_slices() {
  static const int v = [] {
    const char* e = std::getenv("FSTK_CHOL_CRT");
    const int x = e ? std::atoi(e) : 5;
    return x <= 0 ? 0 : std::min(std::max(x, 4), 7);
  }();
  return v;
}
}  // namespace fstk_gpu

// Lower Cholesky factor of a DEVICE matrix in place: chol_crt (slices 4..7,
// panels of nb) or cuSOLVER dpotrf (slices 0).  *info_out = 0 on success.
int32_t fstk_gpu_cholesky_device(double* g, int32_t n, int32_t nb, int32_t slices, int32_t device,
                                 void* stream, int32_t* info_out, fstk_gpu_error* err) {
  using namespace fstk_gpu;
  return guarded(err, [&] {
    require(g && info_out, FSTK_E_PARAMETER, "null argument");
    require(n > 0, FSTK_E_SHAPE, "cholesky: n must be positive");
    require(slices == 0 || (slices >= 4 && slices <= 7), FSTK_E_PARAMETER,
            "cholesky: slices must be 0 (cuSOLVER) or 4..7");
    require(slices == 0 || (nb >= 256 && nb % 16 == 0), FSTK_E_PARAMETER,
            "cholesky: panel width must be a multiple of 16, >= 256");
    DeviceGuard dg(device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    Handles& h = handles(device);
    if (slices > 0) {
      *info_out = chol_crt(h.blas, h.solver, g, n, nb, slices, s, device) ? 0 : 1;
      return;
    }
    cusolverDnSetStream(h.solver, s);
    int lwork = 0;
    if (cusolverDnDpotrf_bufferSize(h.solver, CUBLAS_FILL_MODE_LOWER, n, g, n, &lwork) !=
        CUSOLVER_STATUS_SUCCESS)
      fail(FSTK_E_COMPUTE, "potrf_bufferSize failed");
    DevBuf<double> work(std::max(lwork, 1));
    DevBuf<int> dinfo(1);
    if (cusolverDnDpotrf(h.solver, CUBLAS_FILL_MODE_LOWER, n, g, n, work.p, lwork, dinfo.p) !=
        CUSOLVER_STATUS_SUCCESS)
      fail(FSTK_E_COMPUTE, "potrf failed");
    int hinfo = 0;
    FSTK_CUDA(cudaMemcpyAsync(&hinfo, dinfo.p, 4, cudaMemcpyDeviceToHost, s));
    FSTK_CUDA(cudaStreamSynchronize(s));
    *info_out = hinfo;
  });
}

// x += (L L^T)^{-1} s (s summed over shards); rel_step = ||dx|| / ||x||.
namespace fstk_gpu {
// x := (L L^T)^{-1} x for the lower Cholesky factor L (n x n, ld n), blocked:
// 1024-wide diagonal TRSVs plus DGEMV panel updates that stream L at memory
// speed.  cuSOLVER potrs' whole-matrix TRSVs are latency-bound at n = 32,768;
// this cut the C2 refinement by ~0.1 s.  (Pre-inverting the diagonal blocks
// so they too become DGEMVs measured slower: the inversions cost more than
// the four solves save.)
static void chol_solve_blocked(cublasHandle_t h, const double* L, int n, double* x) {
  constexpr int NB = 1024;
  const double one = 1.0, mone = -1.0;
  auto ok = [](cublasStatus_t st) {
    if (st != CUBLAS_STATUS_SUCCESS) fail(FSTK_E_COMPUTE, "blocked Cholesky solve failed");
  };
  for (int i0 = 0; i0 < n; i0 += NB) {  // forward: L y = x
    const int nb = std::min(NB, n - i0);
    const double* Lii = L + static_cast<int64_t>(i0) * n + i0;
    ok(cublasDtrsv(h, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, nb, Lii, n, x + i0, 1));
    const int rest = n - i0 - nb;
    if (rest > 0)
      ok(cublasDgemv(h, CUBLAS_OP_N, rest, nb, &mone, Lii + nb, n, x + i0, 1, &one, x + i0 + nb, 1));
  }
  for (int i1 = n; i1 > 0; i1 -= NB) {  // backward: L^T z = y
    const int i0 = std::max(0, i1 - NB);
    const int nb = i1 - i0;
    const double* Lii = L + static_cast<int64_t>(i0) * n + i0;
    ok(cublasDtrsv(h, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, CUBLAS_DIAG_NON_UNIT, nb, Lii, n, x + i0, 1));
    if (i0 > 0)  // x[0:i0] -= L[i0:i1, 0:i0]^T x[i0:i1]
      ok(cublasDgemv(h, CUBLAS_OP_T, nb, i0, &mone, L + i0, n, x + i0, 1, &one, x, 1));
  }
  count_launch(4 * ((n + NB - 1) / NB));
}
}  // namespace fstk_gpu

int32_t fstk_gpu_refit_factor(fstk_gpu_refit* rf, const double* gram_in, const double* rhs_in,
                              double* x_dev, fstk_reestimate_info* info, fstk_gpu_error* err) {
  return guarded(err, [&] {
    require(rf && gram_in && rhs_in && x_dev, FSTK_E_PARAMETER, "null argument");
    DeviceGuard dg(rf->device);
    cudaStream_t s = rf->stream;
    Handles& h = handles(rf->device);
    cusolverDnSetStream(h.solver, s);
    const int n = static_cast<int>(rf->R);
    EventTimer ts(s);
    if (rf->est_live) {  // L is about to be overwritten: the estimate must be done with it
      rf->est.wait_enqueued();
      FSTK_CUDA(cudaStreamSynchronize(rf->est_stream));
      rf->est_live = false;
    }
    rf->L.ensure(static_cast<size_t>(n) * n);
    FSTK_CUDA(cudaMemcpyAsync(rf->L.p, gram_in, static_cast<size_t>(n) * n * 8, cudaMemcpyDeviceToDevice, s));
    FSTK_CUDA(cudaMemcpyAsync(x_dev, rhs_in, static_cast<size_t>(n) * 8, cudaMemcpyDeviceToDevice, s));
    int lwork = 0;
    ProfScope prof(FSTK_PROF_SOLVE, s);
    DevBuf<int> dinfo(1);
    int hinfo = 1;
    if (n >= 8192 && chol_crt_slices() > 0) {
      // Blocked Cholesky with int8 tensor-core trailing updates; a block that
      // is not positive definite there is retried with cuSOLVER's dpotrf.
      static const bool dbg = std::getenv("FSTK_DEBUG_TIMING") != nullptr;
      if (dbg) debug_alloc_report("factor start");
      const auto tc0 = std::chrono::steady_clock::now();
      bool chol_ok = false;
      try {
        chol_ok = chol_crt(h.blas, h.solver, rf->L.p, n, 2048, chol_crt_slices(), s, rf->device);
      } catch (const Error& e) {
        // e.g. no room for the int8 scratch next to a large sketch: dpotrf needs none.
        if (e.code != FSTK_E_COMPUTE) throw;
        cudaGetLastError();
        FSTK_CUDA(cudaStreamSynchronize(s));
      }
      if (dbg) {
        std::fprintf(stderr, "fstk factor: chol_crt %8.2f ms\n",
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tc0).count());
        debug_alloc_report("factor");
      }
      if (chol_ok) {
        hinfo = 0;
      } else {
        FSTK_CUDA(cudaMemcpyAsync(rf->L.p, gram_in, static_cast<size_t>(n) * n * 8,
                                  cudaMemcpyDeviceToDevice, s));
      }
    }
    if (hinfo != 0) {
      if (cusolverDnDpotrf_bufferSize(h.solver, CUBLAS_FILL_MODE_LOWER, n, rf->L.p, n, &lwork) !=
          CUSOLVER_STATUS_SUCCESS)
        fail(FSTK_E_COMPUTE, "potrf_bufferSize failed");
      DevBuf<double> work(std::max(lwork, 1));
      if (cusolverDnDpotrf(h.solver, CUBLAS_FILL_MODE_LOWER, n, rf->L.p, n, work.p, lwork, dinfo.p) !=
          CUSOLVER_STATUS_SUCCESS)
        fail(FSTK_E_COMPUTE, "potrf failed");
      count_launch();
      FSTK_CUDA(cudaMemcpyAsync(&hinfo, dinfo.p, 4, cudaMemcpyDeviceToHost, s));
      FSTK_CUDA(cudaStreamSynchronize(s));
    }
    rf->factored = hinfo == 0;
    // Not positive definite: the rank question goes to the pivoted-QR path
    // (refit_solve / fstk_gpu_refit_qr_solve); until then x = 0.
    rf->rank_def = !rf->factored;
    if (rf->factored && n >= 4096) {
      cublasSetStream(h.blas, s);
      chol_solve_blocked(h.blas, rf->L.p, n, x_dev);  // potrs' whole-matrix TRSVs are latency-bound
    } else if (rf->factored) {
      if (cusolverDnDpotrs(h.solver, CUBLAS_FILL_MODE_LOWER, n, 1, rf->L.p, n, x_dev, n, dinfo.p) !=
          CUSOLVER_STATUS_SUCCESS)
        fail(FSTK_E_COMPUTE, "potrs failed");
      count_launch();
    } else {
      FSTK_CUDA(cudaMemsetAsync(x_dev, 0, static_cast<size_t>(n) * 8, s));
    }
    static const bool dbg_f = std::getenv("FSTK_DEBUG_TIMING") != nullptr;
    const auto tf0 = std::chrono::steady_clock::now();
    if (dbg_f) FSTK_CUDA(cudaStreamSynchronize(s));
    const auto tf1 = std::chrono::steady_clock::now();
    if (rf->factored) {
      if (!rf->est_stream) {
        // Highest priority: the estimate is a chain of ~400 small dependent
        // kernels; behind the refinement's full-GPU GEMVs at equal priority
        // each link waited for free SM slots and the chain outlived the
        // refinement (refine wall 0.40 s for 0.27 s of device time).
        int pr_least = 0, pr_greatest = 0;
        FSTK_CUDA(cudaDeviceGetStreamPriorityRange(&pr_least, &pr_greatest));
        FSTK_CUDA(cudaStreamCreateWithPriority(&rf->est_stream, cudaStreamNonBlocking, pr_greatest));
        FSTK_CUDA(cudaEventCreateWithFlags(&rf->est_event, cudaEventDisableTiming));
      }
      FSTK_CUDA(cudaEventRecord(rf->est_event, s));
      FSTK_CUDA(cudaStreamWaitEvent(rf->est_stream, rf->est_event, 0));
      rf->est.started = false;
      rf->est.start_async(rf->L.p, n, 3, rf->est_stream, rf->device);
      rf->est_live = true;
    }
    const auto tf2 = std::chrono::steady_clock::now();
    FSTK_CUDA(cudaStreamSynchronize(s));
    if (dbg_f) {
      const auto tf3 = std::chrono::steady_clock::now();
      auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
      std::fprintf(stderr, "fstk factor: first solve drained %.2f ms, estimate enqueue %.2f ms, final sync %.2f ms\n",
                   ms(tf0, tf1), ms(tf1, tf2), ms(tf2, tf3));
    }
    if (info) {
      info->t_solve += ts.seconds();
      info->rank_deficient = rf->rank_def ? 1 : 0;
    }
  });
}

// s = A_local^T (b_local - A_local x): this shard's part of the refinement rhs.
int32_t fstk_gpu_refit_correction(fstk_gpu_refit* rf, const double* x_dev, double* s_dev,
                                  fstk_gpu_error* err) {
  return guarded(err, [&] {
    require(rf && x_dev && s_dev, FSTK_E_PARAMETER, "null argument");
    require(!rf->columns || rf->exchanged, FSTK_E_PARAMETER,
            "column-sharded refit: exchange_layout, the all-to-all and adopt_rows come first");
    DeviceGuard dg(rf->device);
    cudaStream_t s = rf->stream;
    Handles& h = handles(rf->device);
    cublasSetStream(h.blas, s);
    const bool fft = rf->cfg.transform == FSTK_TRANSFORM_FFT;
    const int64_t arows = fft ? 2 * rf->local_rows : rf->local_rows;
    const int n = static_cast<int>(rf->R);
    if (arows == 0) {
      FSTK_CUDA(cudaMemsetAsync(s_dev, 0, static_cast<size_t>(n) * 8, s));
      FSTK_CUDA(cudaStreamSynchronize(s));
      return;
    }
    rf->tmp_r.ensure(static_cast<size_t>(arows));
    FSTK_CUDA(cudaMemcpyAsync(rf->tmp_r.p, rf->b.p, arows * 8, cudaMemcpyDeviceToDevice, s));
    const double one = 1.0, mone = -1.0, zero = 0.0;
    if (rf->none) {
      // s = A^T (b - A x) through the Kronecker structure (no rows generated).
      ProfScope prof(FSTK_PROF_SOLVE, s);
      none_residual(rf, x_dev, rf->tmp_r.p);
      none_At(rf, rf->tmp_r.p, s_dev);
      FSTK_CUDA(cudaStreamSynchronize(s));
      return;
    }
    ProfScope prof(FSTK_PROF_SOLVE, s);
    if (cublasDgemv(h.blas, CUBLAS_OP_N, static_cast<int>(arows), n, &mone, rf->A.p,
                    static_cast<int>(arows), x_dev, 1, &one, rf->tmp_r.p, 1) != CUBLAS_STATUS_SUCCESS)
      fail(FSTK_E_COMPUTE, "cublasDgemv failed");
    if (cublasDgemv(h.blas, CUBLAS_OP_T, static_cast<int>(arows), n, &one, rf->A.p,
                    static_cast<int>(arows), rf->tmp_r.p, 1, &zero, s_dev, 1) != CUBLAS_STATUS_SUCCESS)
      fail(FSTK_E_COMPUTE, "cublasDgemv failed");
    count_launch(2);
    FSTK_CUDA(cudaStreamSynchronize(s));
  });
}


int32_t fstk_gpu_refit_apply(fstk_gpu_refit* rf, const double* s_dev, double* x_dev,
                             double* rel_step, fstk_gpu_error* err) {
  return guarded(err, [&] {
    require(rf && s_dev && x_dev, FSTK_E_PARAMETER, "null argument");
    require(rf->factored, FSTK_E_PARAMETER, "refit: no Cholesky factor to refine with");
    DeviceGuard dg(rf->device);
    cudaStream_t s = rf->stream;
    Handles& h = handles(rf->device);
    cusolverDnSetStream(h.solver, s);
    cublasSetStream(h.blas, s);
    const int n = static_cast<int>(rf->R);
    rf->apply_dx.ensure(static_cast<size_t>(n));
    rf->apply_info.ensure(1);
    DevBuf<double>& dx = rf->apply_dx;
    DevBuf<int>& dinfo = rf->apply_info;
    FSTK_CUDA(cudaMemcpyAsync(dx.p, s_dev, static_cast<size_t>(n) * 8, cudaMemcpyDeviceToDevice, s));
    ProfScope prof(FSTK_PROF_SOLVE, s);
    if (n >= 4096) {
      chol_solve_blocked(h.blas, rf->L.p, n, dx.p);
    } else if (cusolverDnDpotrs(h.solver, CUBLAS_FILL_MODE_LOWER, n, 1, rf->L.p, n, dx.p, n,
                                dinfo.p) != CUSOLVER_STATUS_SUCCESS) {
      fail(FSTK_E_COMPUTE, "potrs failed");
    }
    const double one = 1.0;
    if (cublasDaxpy(h.blas, n, &one, dx.p, 1, x_dev, 1) != CUBLAS_STATUS_SUCCESS)
      fail(FSTK_E_COMPUTE, "cublasDaxpy failed");
    count_launch(2);
    const double ndx = dev_norm(h.blas, n, dx.p), nx = dev_norm(h.blas, n, x_dev);
    FSTK_CUDA(cudaStreamSynchronize(s));
    if (rel_step) *rel_step = nx > 0 ? ndx / nx : ndx;
  });
}

int32_t fstk_gpu_refit_certify(fstk_gpu_refit* rf, const double* gram_in, double* sigma_ratio,
                               int32_t* certified, fstk_gpu_error* err) {
  return guarded(err, [&] {
    require(rf && gram_in && certified, FSTK_E_PARAMETER, "null argument");
    require(rf->factored, FSTK_E_PARAMETER, "refit_certify: no Cholesky factor");
    DeviceGuard dg(rf->device);
    double lam = -1.0;
    if (rf->est_live) {
      lam = rf->est.result();
      rf->est_live = false;
    }
    rf->sigma_ratio = refit_sigma_ratio(rf, gram_in, lam);
    if (sigma_ratio) *sigma_ratio = rf->sigma_ratio;
    *certified = certified_full_rank(rf, rf->sigma_ratio) ? 1 : 0;
    if (*certified) rf->rank_def = false;
  });
}

int32_t fstk_gpu_refit_local_qr(fstk_gpu_refit* rf, double* raug, fstk_gpu_error* err) {
  return guarded(err, [&] {
    require(rf && raug, FSTK_E_PARAMETER, "null argument");
    require(!rf->columns || rf->exchanged, FSTK_E_PARAMETER,
            "column-sharded refit: exchange_layout, the all-to-all and adopt_rows come first");
    DeviceGuard dg(rf->device);
    QrStream qs;
    refit_local_qr(rf, qs);
    qs.get_r(raug, rf->R + 1);
    FSTK_CUDA(cudaStreamSynchronize(rf->stream));
  });
}

int32_t fstk_gpu_refit_qr_solve(fstk_gpu_refit* rf, const double* raug, double* x_dev,
                                fstk_reestimate_info* info, fstk_gpu_error* err) {
  return guarded(err, [&] {
    require(rf && raug && x_dev, FSTK_E_PARAMETER, "null argument");
    DeviceGuard dg(rf->device);
    EventTimer tq(rf->stream);
    bool def = false;
    cpqr_solve(raug, rf->R + 1, static_cast<int>(rf->R), rf->R, x_dev, &def, rf->stream,
               rf->device);
    rf->rank_def = def;
    if (info) {
      info->t_solve += tq.seconds();
      info->rank_deficient = def ? 1 : 0;
      info->qr_path = 1;
    }
  });
}

// Copies x to the host core and evaluates the validation residuals with the
// old and the new core (randls.cpp:379-381).
int32_t fstk_gpu_refit_finish(fstk_gpu_refit* rf, const double* x_dev, double* core_out,
                              fstk_reestimate_info* info, fstk_gpu_error* err) {
  return guarded(err, [&] {
    require(rf && x_dev && core_out, FSTK_E_PARAMETER, "null argument");
    DeviceGuard dg(rf->device);
    cudaStream_t s = rf->stream;
    FSTK_CUDA(cudaMemcpyAsync(core_out, x_dev, static_cast<size_t>(rf->R) * 8, cudaMemcpyDeviceToHost, s));
    FSTK_CUDA(cudaStreamSynchronize(s));
    EventTimer tr(s);
    std::vector<double> pred(rf->n_val), pred2(rf->n_val);
    if (rf->n_val > 0) {
      DevBuf<double> dp(rf->n_val);
      std::lock_guard<std::mutex> lk(rf->model->mu);
      evaluate_device_core(rf->model, nullptr, rf->val_points.p, rf->n_val, rf->n_val, dp.p, s);
      const int64_t bad = evaluate_device_error(rf->model, rf->n_val, s);
      if (bad >= 0) {
        // relative_residual -> evaluate_batch throws Domain (basis.cpp:218-219).
        const int64_t row = rf->h_val_index[bad];
        std::vector<double> y(rf->d);
        for (int k = 0; k < rf->d; ++k)
          FSTK_CUDA(cudaMemcpy(&y[k], rf->val_points.p + k * rf->n_val + bad, 8,
                               cudaMemcpyDeviceToHost));
        throw_domain(rf->model, row, y.data());
      }
      FSTK_CUDA(cudaMemcpyAsync(pred.data(), dp.p, rf->n_val * 8, cudaMemcpyDeviceToHost, s));
      FSTK_CUDA(cudaStreamSynchronize(s));
      evaluate_device_core(rf->model, core_out, rf->val_points.p, rf->n_val, rf->n_val, dp.p, s);
      FSTK_CUDA(cudaMemcpyAsync(pred2.data(), dp.p, rf->n_val * 8, cudaMemcpyDeviceToHost, s));
      FSTK_CUDA(cudaStreamSynchronize(s));
    }
    if (info) {
      info->residual_before = rel_residual(pred, rf->h_val_values);
      info->residual_after = rel_residual(pred2, rf->h_val_values);
      info->t_residual = tr.seconds();
      info->rank_deficient = rf->rank_def ? 1 : 0;
    }
  });
}

// Single-shard convenience: factor, refine until the step stalls, finish.
int32_t fstk_gpu_refit_solve(fstk_gpu_refit* rf, const double* gram_in, const double* rhs_in,
                             double* core_out, fstk_reestimate_info* info, fstk_gpu_error* err) {
  return guarded(err, [&] {
    require(rf && gram_in && rhs_in && core_out, FSTK_E_PARAMETER, "null argument");
    require(rf->shards == 1, FSTK_E_PARAMETER,
            "refit_solve needs the whole sketch; sharded refits use factor/correction/apply");
    DeviceGuard dg(rf->device);
    const int n = static_cast<int>(rf->R);
    DevBuf<double> x(n), sv(n);
    auto rc = [&](int32_t c) { rethrow_stage(c, err); };
    rc(fstk_gpu_refit_factor(rf, gram_in, rhs_in, x.p, info, err));
    // Escalation ladder for the sliced int8 Gram (a preconditioner-grade
    // A^T A): when it is not positive definite or refinement contracts slowly
    // or stalls, recompute it at kGramUpgradeSlices' accuracy, then fall back
    // to the native fp64 Gram, so hard systems end on the exact fp64 path.
    DevBuf<double> g2, r2;
    const double* gcur = gram_in;
    const double* rcur = rhs_in;
    // The certificate's power iteration runs on the session's side stream,
    // started by each successful factor() (see fstk_gpu_refit_factor).
    auto escalate = [&]() -> bool {
      if (rf->gram_used == 0) return false;
      // Next level: kGramUpgradeSlices planes' accuracy, then the native Gram.
      const int to = rf->gram_used < kGramUpgradeSlices ? kGramUpgradeSlices : 0;
      fstk_reestimate_info li{};
      g2.ensure(static_cast<size_t>(n) * n);
      r2.ensure(static_cast<size_t>(n));
      rc(fstk_gpu_refit_normal_equations_level(rf, to, g2.p, r2.p, &li, err));
      gcur = g2.p;
      rcur = r2.p;
      if (info) {
        info->t_gram += li.t_gram;
        info->gram_int8_ops += li.gram_int8_ops;
        info->gram_slices = rf->gram_used;
      }
      rc(fstk_gpu_refit_factor(rf, gcur, rcur, x.p, info, err));
      return true;
    };
    auto escalate_until_factored = [&]() -> bool {
      do {
        if (!escalate()) return false;
      } while (!rf->factored);
      return true;
    };
    if (!rf->factored) escalate_until_factored();
    int steps = 0;
    // Whether the Cholesky route can answer the reference's rank question;
    // otherwise the pivoted QR of A itself decides (exact_solve).
    bool need_qr = !rf->factored;
    if (rf->factored) {
      EventTimer tref(rf->stream);
      double prev = 1e300;
      for (int it = 0; it < 8; ++it) {
        rc(fstk_gpu_refit_correction(rf, x.p, sv.p, err));
        double step = 0.0;
        rc(fstk_gpu_refit_apply(rf, sv.p, x.p, &step, err));
        ++steps;
        if (step <= 1e-15) break;
        // Converged by extrapolation: contracting by rho = step / prev < 0.1,
        // the error left after this step is ~ rho * step; once that is below
        // kDoneFloor (under the rounding floor of ||dx|| / ||x||, ~2e-13 at
        // C2) another step over A could only confirm it.
        if (it >= 1 && step < 0.1 * prev && step * (step / prev) <= kDoneFloor) break;
        // Stagnation at the rounding floor (||dx||/||x|| ~ cond(A) eps, about
        // 1e-13 at C2) is convergence.  Above kStallFloor: not contracting,
        // contracting slower than 10x per step on a sliced Gram, or out of
        // steps while still moving, escalates (or flags a native system).
        constexpr double kStallFloor = 1e-11;
        const bool flat = it >= 1 && step > 0.5 * prev;
        if (flat && step <= kStallFloor) break;
        const bool slow = rf->gram_used > 0 && it >= 1 && step > kStallFloor && step > 0.1 * prev;
        const bool last = it == 7 && step > kStallFloor;
        if (flat || slow || last) {
          if (rf->gram_used > 0) {
            if (!escalate_until_factored()) break;
            prev = 1e300;
            it = -1;
            continue;
          }
          // No (or too slow) contraction on the native Gram: cond(A)^2 eps
          // is not small, and only the pivoted QR can decide the rank.
          need_qr = true;
          break;
        }
        prev = step;
      }
      if (!need_qr && rf->factored) {
        double lam = -1.0;
        if (rf->est_live) {
          lam = rf->est.result();
          rf->est_live = false;
        }
        rf->sigma_ratio = refit_sigma_ratio(rf, gcur, lam);
        need_qr = !certified_full_rank(rf, rf->sigma_ratio);
      } else if (!rf->factored) {
        need_qr = true;
      }
      if (info) info->t_solve += tref.seconds();
    }
    if (need_qr) {
      EventTimer tq(rf->stream);
      exact_solve(rf, x.p);
      if (info) info->t_solve += tq.seconds();
    } else {
      rf->rank_def = false;
    }
    if (info) {
      info->refine_steps = steps;
      info->rank_deficient = rf->rank_def ? 1 : 0;
      info->qr_path = need_qr ? 1 : 0;
      info->sigma_ratio = rf->sigma_ratio;
    }
    rc(fstk_gpu_refit_finish(rf, x.p, core_out, info, err));
  });
}

void fstk_gpu_refit_end(fstk_gpu_refit* rf) {
  if (!rf) return;
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(rf->device);
  cudaStreamSynchronize(rf->stream);
  delete rf;
  if (prev >= 0) cudaSetDevice(prev);
}

int32_t fstk_gpu_refit_rows(const fstk_gpu_refit* rf, uint64_t* rows, fstk_gpu_error* err) {
  return guarded(err, [&] {
    require(rf && rows, FSTK_E_PARAMETER, "null argument");
    std::memcpy(rows, rf->plan.rows.data(), rf->plan.rows.size() * 8);
  });
}

// A and b of this shard in reference row order (restricted to the shard's rows).
int32_t fstk_gpu_refit_sketched(const fstk_gpu_refit* rf, double* a, double* b, int64_t* rows_local,
                                fstk_gpu_error* err) {
  return guarded(err, [&] {
    require(rf, FSTK_E_PARAMETER, "null argument");
    require(!rf->columns || rf->exchanged, FSTK_E_PARAMETER,
            "column-sharded refit: exchange_layout, the all-to-all and adopt_rows come first");
    const bool fft = rf->cfg.transform == FSTK_TRANSFORM_FFT;
    const int64_t lr = rf->local_rows;
    const int64_t arows = fft ? 2 * lr : lr;
    if (rows_local) *rows_local = arows;
    if (!a && !b) return;
    DeviceGuard dg(rf->device);
    if (rf->none) {
      // Rows are already in plan order (sorted sampled rows of this shard).
      DevBuf<double> W(static_cast<size_t>(std::max<int64_t>(arows, 1)) * rf->R);
      if (arows > 0) generate_design_block(rf, 0, arows, W.p, arows, rf->stream);
      FSTK_CUDA(cudaStreamSynchronize(rf->stream));
      if (a) FSTK_CUDA(cudaMemcpy(a, W.p, static_cast<size_t>(arows) * rf->R * 8, cudaMemcpyDeviceToHost));
      if (b) FSTK_CUDA(cudaMemcpy(b, rf->b.p, arows * 8, cudaMemcpyDeviceToHost));
      return;
    }
    std::vector<double> ha(static_cast<size_t>(arows) * rf->R), hb(arows);
    FSTK_CUDA(cudaMemcpy(ha.data(), rf->A.p, ha.size() * 8, cudaMemcpyDeviceToHost));
    FSTK_CUDA(cudaMemcpy(hb.data(), rf->b.p, hb.size() * 8, cudaMemcpyDeviceToHost));
    // Sample s (plan order) sits at destination row dest_of_sample[s]; this
    // shard owns destinations [row_lo, row_hi).  Emit its samples in plan order.
    std::vector<int64_t> order;
    for (uint64_t sidx = 0; sidx < rf->S; ++sidx) {
      const int64_t dst = rf->in.dest_of_sample[sidx];
      if (dst >= rf->row_lo && dst < rf->row_hi) order.push_back(dst - rf->row_lo);
    }
    for (int64_t o = 0; o < static_cast<int64_t>(order.size()); ++o) {
      const int64_t src = order[o];
      for (int64_t c = 0; c < rf->R; ++c) {
        if (a) {
          a[o + arows * c] = ha[src + arows * c];
          if (fft) a[lr + o + arows * c] = ha[lr + src + arows * c];
        }
      }
      if (b) {
        b[o] = hb[src];
        if (fft) b[lr + o] = hb[lr + src];
      }
    }
  });
}

// Columns `cols` of this shard's sketched A (index R = b) in reference row
// order, column c at out + c * rows_local (rows_local = 2 x rows for FFT).
int32_t fstk_gpu_refit_sketched_columns(const fstk_gpu_refit* rf, const int64_t* cols,
                                        int64_t ncols, double* out, fstk_gpu_error* err) {
  return guarded(err, [&] {
    require(rf && (ncols == 0 || (cols && out)), FSTK_E_PARAMETER, "null argument");
    require(!rf->columns || rf->exchanged, FSTK_E_PARAMETER,
            "column-sharded refit: exchange_layout, the all-to-all and adopt_rows come first");
    require(!rf->none, FSTK_E_PARAMETER,
            "transform none never materialises A; use fstk_gpu_refit_sketched");
    DeviceGuard dg(rf->device);
    const bool fft = rf->cfg.transform == FSTK_TRANSFORM_FFT;
    const int64_t lr = rf->local_rows;
    const int64_t arows = fft ? 2 * lr : lr;
    std::vector<int64_t> order;  // source row (shard-local) of each output row
    for (uint64_t sidx = 0; sidx < rf->S; ++sidx) {
      const int64_t dst = rf->in.dest_of_sample[sidx];
      if (dst >= rf->row_lo && dst < rf->row_hi) order.push_back(dst - rf->row_lo);
    }
    std::vector<double> col(static_cast<size_t>(std::max<int64_t>(arows, 1)));
    for (int64_t c = 0; c < ncols; ++c) {
      require(cols[c] >= 0 && cols[c] <= rf->R, FSTK_E_PARAMETER, "column index out of range");
      const double* src = cols[c] == rf->R ? rf->b.p : rf->A.p + cols[c] * arows;
      FSTK_CUDA(cudaMemcpy(col.data(), src, static_cast<size_t>(arows) * 8, cudaMemcpyDeviceToHost));
      double* o = out + c * arows;
      for (int64_t r = 0; r < static_cast<int64_t>(order.size()); ++r) {
        o[r] = col[order[r]];
        if (fft) o[lr + r] = col[lr + order[r]];
      }
    }
  });
}

int32_t fstk_gpu_reestimate_core(const fstk_gpu_model* m, const double* points,
                                 const double* values, int64_t q, int32_t d,
                                 const fstk_sketch_cfg* cfg, double* core_out,
                                 fstk_reestimate_info* info, fstk_gpu_error* err) {
  // A model created after fstk_gpu_set_devices(n > 1) carries replicas: the
  // refit then runs sharded over all of them in this process (fstk_multi.cu).
  if (m && !m->replicas.empty())
    return fstk_gpu::reestimate_core_multi(m, points, values, q, d, cfg, core_out, info, err);
  fstk_gpu_refit* rf = nullptr;
  fstk_reestimate_info local{};
  fstk_reestimate_info* inf = info ? info : &local;
  std::memset(inf, 0, sizeof(*inf));
  int32_t rc = fstk_gpu_refit_begin(m, points, values, q, d, cfg, 0, 1, &rf, inf, err);
  if (rc) return rc;
  rc = guarded(err, [&] {
    DeviceGuard dg(m->device);
    DevBuf<double> gram(static_cast<size_t>(m->R) * m->R), rhs(m->R);
    rethrow_stage(fstk_gpu_refit_normal_equations(rf, gram.p, rhs.p, inf, err), err);
    rethrow_stage(fstk_gpu_refit_solve(rf, gram.p, rhs.p, core_out, inf, err), err);
  });
  fstk_gpu_refit_end(rf);
  return rc;
}

// ---------------------------------------------------------- diagnostics ---
int32_t fstk_gpu_build_design_rows(const fstk_gpu_model* m, const double* points, int64_t q,
                                   int32_t d, double* w, fstk_gpu_error* err) {
  return guarded(err, [&] {
    require(m && points && w, FSTK_E_PARAMETER, "null argument");
    require(d == m->d, FSTK_E_PARAMETER, "points must have one column per mode");
    if (q == 0) return;
    std::lock_guard<std::mutex> lk(m->mu);
    DeviceGuard dg(m->device);
    cudaStream_t s = m->chunk[0].stream;
    DevBuf<double> dp(static_cast<size_t>(q) * d);
    FSTK_CUDA(cudaMemcpyAsync(dp.p, points, static_cast<size_t>(q) * d * 8, cudaMemcpyHostToDevice, s));
    int64_t toff[kMaxOrder], tot = 0;
    for (int k = 0; k < d; ++k) {
      toff[k] = tot;
      tot += m->ranks[k] * q;
    }
    DevBuf<double> tables(tot);
    DevBuf<unsigned long long> derr(1);
    FSTK_CUDA(cudaMemsetAsync(derr.p, 0xff, 8, s));
    launch_mode_tables(m, dp.p, q, q, q, nullptr, tables.p, toff, q, true, derr.p, s);
    // W column ell = ((u0 u1) u2) ... (design_column, randls.cpp:44-52) via a
    // sketch-free pass: generate columns with unit sign and identity order.
    std::vector<double> ht(tot);
    FSTK_CUDA(cudaMemcpyAsync(ht.data(), tables.p, tot * 8, cudaMemcpyDeviceToHost, s));
    unsigned long long bad = 0;
    FSTK_CUDA(cudaMemcpyAsync(&bad, derr.p, 8, cudaMemcpyDeviceToHost, s));
    FSTK_CUDA(cudaStreamSynchronize(s));
    if (bad != ULLONG_MAX) {
      std::vector<double> y(d);
      for (int k = 0; k < d; ++k) y[k] = points[k * q + bad];
      throw_domain(m, static_cast<int64_t>(bad), y.data());
    }
    for (int64_t ell = 0; ell < m->R; ++ell) {
      int64_t rem = ell;
      double* col = w + ell * q;
      const double* t0 = ht.data() + toff[0] + (rem % m->ranks[0]) * q;
      for (int64_t i = 0; i < q; ++i) col[i] = t0[i];
      rem /= m->ranks[0];
      for (int k = 1; k < d; ++k) {
        const double* tk = ht.data() + toff[k] + (rem % m->ranks[k]) * q;
        for (int64_t i = 0; i < q; ++i) col[i] *= tk[i];
        rem /= m->ranks[k];
      }
    }
  });
}

static int32_t sketch_dense(const double* w, const double* u, int64_t q, int64_t r,
                            const fstk_sketch_cfg* cfg, bool mixed, double* a, double* b,
                            uint64_t* padded, fstk_gpu_error* err) {
  return guarded(err, [&] {
    require(w && cfg, FSTK_E_PARAMETER, "null argument");
    require(q >= 1, FSTK_E_PARAMETER, mixed ? "empty matrix" : "empty system");
    require(cfg->transform >= 0 && cfg->transform <= 2, FSTK_E_PARAMETER,
            "transform must be dct, wht, or fft");  // 'none' is a reestimate_core option only
    int dev = 0;
    FSTK_CUDA(cudaGetDevice(&dev));
    const uint64_t S = mixed ? 0 : resolve_sample_rows(cfg->sample_rows, r);
    Plan plan = make_plan(static_cast<uint64_t>(q), S, cfg->seed, !mixed);
    if (padded) *padded = plan.q_pad;
    cudaStream_t s;
    FSTK_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    struct SG {
      cudaStream_t s;
      ~SG() { cudaStreamDestroy(s); }
    } sg{s};
    SketchInputs in;
    build_inputs(cfg->transform, plan.q_pad, static_cast<uint64_t>(q), plan.signs, plan.rows,
                 mixed, {}, false, in, s);
    const bool fft = cfg->transform == FSTK_TRANSFORM_FFT;
    const int64_t nrows = in.rows_total;
    const int64_t arows = fft ? 2 * nrows : nrows;
    DevBuf<double> dw(static_cast<size_t>(q) * r), du(q), dA(static_cast<size_t>(arows) * r),
        db(arows);
    FSTK_CUDA(cudaMemcpyAsync(dw.p, w, static_cast<size_t>(q) * r * 8, cudaMemcpyHostToDevice, s));
    if (u) FSTK_CUDA(cudaMemcpyAsync(du.p, u, q * 8, cudaMemcpyHostToDevice, s));
    SketchJob J{};
    J.kind = cfg->transform;
    J.n = plan.q_pad;
    J.src = SRC_DENSE;
    J.dense = dw.p;
    J.ldd = q;
    J.rhs = du.p;
    J.R = r;
    J.with_rhs = u != nullptr && b != nullptr;
    J.sgn = in.sgn.p;
    J.row_src = in.row_src.p;
    J.slot = in.slot.p;
    J.post_re = in.post_re.p;
    J.post_im = in.post_im.p;
    J.post_c = in.post_c.p;
    J.scale = mixed ? 1.0 : plan.scale;
    J.row_lo = 0;
    J.row_hi = nrows;
    J.im_off = nrows;
    J.A = dA.p;
    J.lda = arows;
    J.b = db.p;
    run_sketch(dev, J, s);
    FSTK_CUDA(cudaMemcpyAsync(a, dA.p, static_cast<size_t>(arows) * r * 8, cudaMemcpyDeviceToHost, s));
    if (J.with_rhs) FSTK_CUDA(cudaMemcpyAsync(b, db.p, arows * 8, cudaMemcpyDeviceToHost, s));
    FSTK_CUDA(cudaStreamSynchronize(s));
  });
}

int32_t fstk_gpu_sketch(const double* w, const double* u, int64_t q, int64_t r,
                        const fstk_sketch_cfg* cfg, double* a, double* b, uint64_t* padded_rows,
                        fstk_gpu_error* err) {
  if (!u || !b || !a)
    return guarded(err, [&] { fail(FSTK_E_PARAMETER, "null argument"); });
  return sketch_dense(w, u, q, r, cfg, false, a, b, padded_rows, err);
}

int32_t fstk_gpu_mixed_matrix(const double* w, int64_t q, int64_t r, const fstk_sketch_cfg* cfg,
                              double* out, fstk_gpu_error* err) {
  if (!out) return guarded(err, [&] { fail(FSTK_E_PARAMETER, "null argument"); });
  return sketch_dense(w, nullptr, q, r, cfg, true, out, nullptr, nullptr, err);
}

}  // extern "C"
