// fstk B200 library — model upload and point evaluation (sm_100a).
//
// Replaces, on the GPU, the reference evaluation path
//   evaluate_batch (proj/src/model.cpp:208-227)
//     -> mode_values (model.cpp:71-94) -> eval_basis/to_reference/legendre_values
//        (proj/src/basis.cpp:49-61, 215-234)
//     -> contract_core (model.cpp:176-191)
// with two kernels:
//   K1a mode_tables_kernel: per point and mode, domain map + Legendre
//       recurrence (bit-exact: same rounding sequence, Markstein-corrected
//       division) + sparse coefficient dot -> u_k tables in HBM/L2;
//   K1b contract_kernel: the core contraction as fp64 tensor-core (DMMA
//       m8n8k4) tiles T = U_0 * G_(0) with a fused per-point bilinear
//       epilogue y += (sum_j1 T u_1) * prod_{k>=2} u_k, the core streamed
//       through a TMA bulk-copy / mbarrier ring (warp-specialised producer).
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <condition_variable>
#include <thread>
#include <vector>

#include "fstk_internal.h"

namespace fstk_gpu {

std::atomic<uint64_t> g_launches{0};

// Legendre constants: for n = 1..63, (2n+1), n, n+1, RN(1/(n+1)); and
// norm[n] = sqrt(2n+1) exactly as basis.cpp:54,59 computes it.
struct LegConst {
  double a[kMaxDegree + 1];    // 2n+1
  double b[kMaxDegree + 1];    // n
  double c[kMaxDegree + 1];    // n+1
  double rc[kMaxDegree + 1];   // RN(1/(n+1))
  double norm[kMaxDegree + 2]; // sqrt(2n+1); norm[1] = sqrt(3)
};
__constant__ LegConst c_leg;

static void upload_leg_constants(int device) {
  LegConst h;
  for (int n = 0; n <= kMaxDegree; ++n) {
    h.a[n] = static_cast<double>(2 * n + 1);
    h.b[n] = static_cast<double>(n);
    h.c[n] = static_cast<double>(n + 1);
    h.rc[n] = 1.0 / static_cast<double>(n + 1);
  }
  for (int n = 0; n <= kMaxDegree + 1; ++n) h.norm[n] = std::sqrt(2.0 * n + 1.0);
  h.norm[1] = std::sqrt(3.0);
  FSTK_CUDA(cudaMemcpyToSymbol(c_leg, &h, sizeof(h)));
}

int device_sm_count(int device) {
  int n = 0;
  FSTK_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device));
  return n;
}

// ---------------------------------------------------------- K1a modes ---
// Thread per output row; Legendre values of the current mode staged in
// shared memory (column per thread) so the sparse dot can gather them.
template <bool EXACT>
__global__ void __launch_bounds__(128) mode_tables_kernel(
    ModesDev M, int mode_begin, int mode_end, const double* __restrict__ pts, int64_t ldp,
    int64_t n, int64_t n_out, const int64_t* __restrict__ row_src, double* __restrict__ tables,
    Int64x8 toff, int64_t ldt, unsigned long long* err_row) {
  extern __shared__ double Ls[];  // (pmax+1) x blockDim
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int tid = threadIdx.x;
  const int nt = blockDim.x;
  int64_t src = i;
  bool valid = i < n;
  if (row_src && i < n_out) {
    src = i < n ? row_src[i] : -1;
    valid = src >= 0;
  }
  for (int k = mode_begin; k < mode_end; ++k) {
    const ModeDev& md = M.m[k];
    double* tk = tables + toff.v[k];
    if (i >= n_out) continue;
    if (!valid) {
      for (int j = 0; j < md.r; ++j) tk[j * ldt + i] = 0.0;
      continue;
    }
    const double x = pts[k * ldp + src];
    // to_reference (basis.cpp:215-222): Domain error beyond the slack, clamp within.
    double t;
    if (!(x >= md.lo - md.slack && x <= md.hi + md.slack)) {
      atomicMin(err_row, static_cast<unsigned long long>(i));
      t = 0.0;
    } else {
      const double cl = fmin(md.hi, fmax(md.lo, x));
      t = xadd(-1.0, __ddiv_rn(xmul(2.0, xsub(cl, md.lo)), md.span));
    }
    // legendre_values (basis.cpp:49-61), same rounding sequence.
    const int p = md.pmax;
    Ls[tid] = 1.0;
    if (p >= 1) Ls[nt + tid] = xmul(c_leg.norm[1], t);
    double pm1 = 1.0, pm0 = t;
    for (int q = 1; q < p; ++q) {
      const double num = xsub(xmul(xmul(c_leg.a[q], t), pm0), xmul(c_leg.b[q], pm1));
      const double pn1 = xdiv_small(num, c_leg.c[q], c_leg.rc[q]);
      pm1 = pm0;
      pm0 = pn1;
      Ls[(q + 1) * nt + tid] = xmul(c_leg.norm[q + 1], pn1);
    }
    // Sparse dot in ascending index order (model.cpp:86-88).
    for (int j = 0; j < md.r; ++j) {
      double v = 0.0;
      const int e = md.rowptr[j + 1];
      for (int s = md.rowptr[j]; s < e; ++s) {
        const double c = md.coef[s];
        const double l = Ls[md.idx[s] * nt + tid];
        v = EXACT ? xadd(v, xmul(c, l)) : fma(c, l, v);
      }
      tk[j * ldt + i] = v;
    }
  }
}

// Dense-coefficient variant (the hot one): thread per (row, JC functions).
// The mode's coefficient block C[i][j] (zero where a function has no index i)
// sits in shared memory and is read with uniform (broadcast) loads; the
// Legendre value L_i is produced by the recurrence in registers and applied
// to JC independent accumulators, in ascending i.  Adding the zero entries
// leaves every partial sum unchanged, so with EXACT (separate multiply/add)
// this reproduces the reference's sparse dot (model.cpp:86-88) bit for bit
// whenever the indices are strictly increasing (format.md:67).
// PPT points per thread (rows i and i + 128): one broadcast coefficient load
// then feeds 2*PPT independent FMAs, which keeps the shared-memory (MIO) queue
// off the critical path.
template <bool EXACT, int JC>
struct DensePPT {
  static constexpr int value = JC <= 32 ? 2 : 1;
};

template <bool EXACT, int JC, int PPT>
__global__ void __launch_bounds__(128) mode_dense_kernel(
    ModeDev md, const double* __restrict__ xs, int64_t n, int64_t n_out,
    const int64_t* __restrict__ row_src, double* __restrict__ tk, int64_t ldt,
    unsigned long long* err_row) {
  extern __shared__ __align__(16) double Cs[];  // (pmax+1) x JC
  const int j0 = blockIdx.y * JC;
  const int p = md.pmax;
  for (int e = threadIdx.x; e < (p + 1) * JC; e += blockDim.x)
    Cs[e] = md.dense[(e / JC) * md.ldc + j0 + (e % JC)];
  __syncthreads();
  const int64_t base = static_cast<int64_t>(blockIdx.x) * (128 * PPT) + threadIdx.x;
  const int jn = min(JC, md.r - j0);
  double t[PPT];
  bool live[PPT];
#pragma unroll
  for (int u = 0; u < PPT; ++u) {
    const int64_t i = base + u * 128;
    live[u] = i < n_out;
    t[u] = 0.0;
    if (!live[u]) continue;
    int64_t src = i;
    bool valid = i < n;
    if (row_src) {
      src = i < n ? row_src[i] : -1;
      valid = src >= 0;
    }
    if (!valid) {
#pragma unroll
      for (int j = 0; j < JC; ++j)
        if (j < jn) tk[(j0 + j) * ldt + i] = 0.0;
      live[u] = false;
      continue;
    }
    const double x = xs[src];
    if (!(x >= md.lo - md.slack && x <= md.hi + md.slack)) {
      atomicMin(err_row, static_cast<unsigned long long>(i));
    } else {
      const double cl = fmin(md.hi, fmax(md.lo, x));
      t[u] = xadd(-1.0, __ddiv_rn(xmul(2.0, xsub(cl, md.lo)), md.span));
    }
  }
  if (PPT == 1 ? !live[0] : !(live[0] || live[PPT - 1])) return;
  double acc[PPT][JC];
#pragma unroll
  for (int u = 0; u < PPT; ++u)
#pragma unroll
    for (int j = 0; j < JC; ++j) acc[u][j] = 0.0;
  auto apply = [&](const double* row, const double (&L)[PPT]) {
    const double2* r2 = reinterpret_cast<const double2*>(row);
#pragma unroll
    for (int j = 0; j < JC / 2; ++j) {
      const double2 c = r2[j];
#pragma unroll
      for (int u = 0; u < PPT; ++u) {
        if (EXACT) {
          acc[u][2 * j] = xadd(acc[u][2 * j], xmul(c.x, L[u]));
          acc[u][2 * j + 1] = xadd(acc[u][2 * j + 1], xmul(c.y, L[u]));
        } else {
          acc[u][2 * j] = fma(c.x, L[u], acc[u][2 * j]);
          acc[u][2 * j + 1] = fma(c.y, L[u], acc[u][2 * j + 1]);
        }
      }
    }
  };
  // legendre_values (basis.cpp:49-61), same rounding sequence.
  double L[PPT], pm1[PPT], pm0[PPT];
#pragma unroll
  for (int u = 0; u < PPT; ++u) L[u] = 1.0;
  apply(Cs, L);
  if (p >= 1) {
#pragma unroll
    for (int u = 0; u < PPT; ++u) L[u] = xmul(c_leg.norm[1], t[u]);
    apply(Cs + JC, L);
  }
#pragma unroll
  for (int u = 0; u < PPT; ++u) {
    pm1[u] = 1.0;
    pm0[u] = t[u];
  }
  for (int q = 1; q < p; ++q) {
    const double a = c_leg.a[q], b = c_leg.b[q], c = c_leg.c[q], rc = c_leg.rc[q];
    const double nq = c_leg.norm[q + 1];
#pragma unroll
    for (int u = 0; u < PPT; ++u) {
      const double num = xsub(xmul(xmul(a, t[u]), pm0[u]), xmul(b, pm1[u]));
      const double pn1 = xdiv_small(num, c, rc);
      pm1[u] = pm0[u];
      pm0[u] = pn1;
      L[u] = xmul(nq, pn1);
    }
    apply(Cs + (q + 1) * JC, L);
  }
#pragma unroll
  for (int u = 0; u < PPT; ++u) {
    if (!live[u]) continue;
    const int64_t i = base + u * 128;
#pragma unroll
    for (int j = 0; j < JC; ++j)
      if (j < jn) tk[(j0 + j) * ldt + i] = acc[u][j];
  }
}

// ------------------------------------------------------- K1b contract ---
// Tile of TP points per CTA; consumer warps = (TP/32 point groups) x 2 column
// halves; one producer warp streams the u tables (per tile) and the core
// tiles (ring of nstage) with TMA bulk copies completing on mbarriers.
struct ContractParams {
  const double* tables;
  Int64x8 toff;
  int64_t ldt;
  int64_t n;
  int64_t ntiles;
  int d;
  int r[kMaxOrder];
  int Kp, N1p, NC, Mout, N1;  // N1 = rows of u1 staged (NC * N1p)
  int nstage;
  const double* bpack;
  double* out;
};

__host__ __device__ constexpr int u0_ld(int tp) { return tp + 4; }  // conflict-free A fragments
__host__ __device__ constexpr int u1_ld(int tp) { return tp + 2; }  // conflict-free epilogue

struct SmemLayout {
  uint32_t bars, u0, u1, uk, bst, ybuf, total;
};

__host__ __device__ inline SmemLayout smem_layout(const ContractParams& P, int tp) {
  SmemLayout L{};
  uint32_t o = 0;
  L.bars = o;
  o += ((2 * P.nstage + 2) * 8 + 127) / 128 * 128;
  L.u0 = o;
  o += static_cast<uint32_t>(P.Kp) * u0_ld(tp) * 8;
  L.u1 = o;
  o += static_cast<uint32_t>(P.N1) * u1_ld(tp) * 8;
  L.uk = o;
  for (int k = 2; k < P.d; ++k) o += static_cast<uint32_t>(P.r[k]) * tp * 8;
  o = (o + 127) / 128 * 128;
  L.bst = o;
  o += static_cast<uint32_t>(P.nstage) * P.Kp * P.N1p * 8;
  L.ybuf = o;
  o += 2 * tp * 8;
  L.total = o;
  return L;
}

template <int NCW>
__device__ __forceinline__ void consumer_bar() {
  asm volatile("bar.sync 1, %0;" ::"n"(NCW * 32) : "memory");
}

// Outer factor prod_{k>=2} u_k[j_k(m)] for one row; D = compile-time order
// (0 = generic runtime order, d >= 5).
template <int D>
__device__ __forceinline__ double outer_factor(const ContractParams& P, const double* uk_base,
                                               const int* jk, int row, int tp) {
  if constexpr (D == 2) {
    return 1.0;
  } else if constexpr (D == 3) {
    return uk_base[jk[0] * tp + row];
  } else if constexpr (D > 3) {
    double o = uk_base[jk[0] * tp + row];
    const double* base = uk_base + P.r[2] * tp;
#pragma unroll
    for (int k = 3; k < D; ++k) {
      o = o * base[jk[k - 2] * tp + row];
      base += P.r[k] * tp;
    }
    return o;
  } else {
    double o = 1.0;
    const double* base = uk_base;
    for (int k = 2; k < P.d; ++k) {
      o = o * base[jk[k - 2] * tp + row];
      base += P.r[k] * tp;
    }
    return o;
  }
}

template <int NSW, int D, int TP, int NH>
__global__ void __launch_bounds__((TP / 32 * NH + 1) * 32) contract_kernel(const ContractParams P) {
  constexpr int NPG = TP / 32;        // 32-point groups
  constexpr int NCW = NPG * NH;       // consumer warps (NH column groups per point group)
  constexpr int U0_LD = u0_ld(TP), U1_LD = u1_ld(TP);
  extern __shared__ __align__(1024) unsigned char smem[];
  const SmemLayout L = smem_layout(P, TP);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bars);
  uint64_t* empty = full + P.nstage;
  uint64_t* ufull = empty + P.nstage;
  uint64_t* uempty = ufull + 1;
  double* u0s = reinterpret_cast<double*>(smem + L.u0);
  double* u1s = reinterpret_cast<double*>(smem + L.u1);
  double* uks = reinterpret_cast<double*>(smem + L.uk);
  double* bst = reinterpret_cast<double*>(smem + L.bst);
  double* ybuf = reinterpret_cast<double*>(smem + L.ybuf);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int NT = P.NC * P.Mout;
  const int stage_elems = P.Kp * P.N1p;
  const uint32_t stage_bytes = static_cast<uint32_t>(stage_elems) * 8u;

  if (threadIdx.x == 0) {
    for (int s = 0; s < P.nstage; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    mbar_init(ufull, 1);
    mbar_init(uempty, NCW);
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == NCW) {
    // ===== producer warp: u tables per tile + core tiles ring (TMA bulk) =====
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      uint32_t ubytes = static_cast<uint32_t>(P.Kp + P.N1) * TP * 8u;
      for (int k = 2; k < P.d; ++k) ubytes += static_cast<uint32_t>(P.r[k]) * TP * 8u;
      for (int64_t tile = blockIdx.x; tile < P.ntiles; tile += gridDim.x, ++it) {
        if (it > 0) mbar_wait(uempty, (it - 1) & 1);
        mbar_arrive_expect_tx(ufull, ubytes);
        const int64_t row0 = tile * TP;
        const double* t0 = P.tables + P.toff.v[0] + row0;
        for (int j = 0; j < P.Kp; ++j) bulk_g2s(u0s + j * U0_LD, t0 + j * P.ldt, TP * 8, ufull);
        const double* t1 = P.tables + P.toff.v[1] + row0;
        for (int j = 0; j < P.N1; ++j) bulk_g2s(u1s + j * U1_LD, t1 + j * P.ldt, TP * 8, ufull);
        double* dst = uks;
        for (int k = 2; k < P.d; ++k) {
          const double* tk = P.tables + P.toff.v[k] + row0;
          for (int j = 0; j < P.r[k]; ++j) bulk_g2s(dst + j * TP, tk + j * P.ldt, TP * 8, ufull);
          dst += P.r[k] * TP;
        }
        for (int tt = 0; tt < NT; ++tt) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full[stage], stage_bytes);
          bulk_g2s(bst + static_cast<size_t>(stage) * stage_elems,
                   P.bpack + static_cast<size_t>(tt) * stage_elems, stage_bytes, &full[stage]);
          if (++stage == P.nstage) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
    return;
  }

  // ===== consumer warps =====
  const int pg = warp % NPG;  // 32-point group
  const int nh = warp / NPG;  // column group
  const int g = lane >> 2, t = lane & 3;
  constexpr int NS = NH * NSW;
  int stage = 0;
  uint32_t phase = 0;
  int it = 0;
  const int ksteps = P.Kp / 4;
  for (int64_t tile = blockIdx.x; tile < P.ntiles; tile += gridDim.x, ++it) {
    mbar_wait(ufull, it & 1);
    double y[4] = {0.0, 0.0, 0.0, 0.0};
    int c = 0;                              // j1 chunk
    constexpr int NJK = D == 0 ? kMaxOrder - 2 : (D > 2 ? D - 2 : 1);
    int jk[NJK] = {0};  // digits j_2, j_3, ... of m
    for (int tt = 0; tt < NT; ++tt) {
      mbar_wait(&full[stage], phase);
      const double* B = bst + static_cast<size_t>(stage) * stage_elems;
      double acc[4][NSW][2];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < NSW; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
      const double* ua = u0s + t * U0_LD + pg * 32 + g;
      const double* bb = B + (nh * NSW) * 32 + lane;
#pragma unroll 4
      for (int ks = 0; ks < ksteps; ++ks) {
        double av[4], bv[NSW];
#pragma unroll
        for (int a = 0; a < 4; ++a) av[a] = ua[(4 * ks) * U0_LD + a * 8];
#pragma unroll
        for (int b = 0; b < NSW; ++b) bv[b] = bb[(ks * NS + b) * 32];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < NSW; ++b) dmma_8x8x4(acc[a][b][0], acc[a][b][1], av[a], bv[b]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == P.nstage) {
        stage = 0;
        phase ^= 1;
      }
      // Epilogue: W = sum_j1 T u1; y += W * prod_{k>=2} u_k (no integer division:
      // the digits of m advance like an odometer).
      const double* u1c = u1s + (c * P.N1p + nh * NSW * 8 + 2 * t) * U1_LD;
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const int row = pg * 32 + a * 8 + g;
        const double o = outer_factor<D>(P, uks, jk, row, TP);
        double w = 0.0;
#pragma unroll
        for (int b = 0; b < NSW; ++b) {
          w = fma(acc[a][b][0], u1c[(b * 8) * U1_LD + row], w);
          w = fma(acc[a][b][1], u1c[(b * 8 + 1) * U1_LD + row], w);
        }
        y[a] = fma(w, o, y[a]);
      }
      if (++c == P.NC) {
        c = 0;
        if constexpr (D != 2) {
          const int dd = (D == 0) ? P.d : D;
          for (int k = 2; k < dd; ++k) {
            if (++jk[k - 2] < P.r[k]) break;
            jk[k - 2] = 0;
          }
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(uempty);
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      y[a] += __shfl_xor_sync(0xffffffffu, y[a], 1);
      y[a] += __shfl_xor_sync(0xffffffffu, y[a], 2);
      if (t == 0) ybuf[nh * TP + pg * 32 + a * 8 + g] = y[a];
    }
    consumer_bar<NCW>();
    if (nh == 0) {
      const int row = pg * 32 + lane;
      const int64_t gi = tile * TP + row;
      if (gi < P.n) P.out[gi] = NH == 2 ? ybuf[row] + ybuf[TP + row] : ybuf[row];
    }
    consumer_bar<NCW>();
  }
}

// ------------------------------------------------- K1b' Khatri-Rao form ---
// For d = 3, 4: T[p, n] = sum_{j0,j1} (u0[p,j0] u1[p,j1]) G[j0, j1, n] with
// n = (j2, j3): K = r0 * r1 (A generated per j1 as the u0 fragment times the
// point's u1 value — one DMUL per fragment), N = r2 (r3), and a single
// epilogue per tile y_p = sum_n T[p, n] prod_{k>=2} u_k[p, j_k(n)].  The
// accumulators live across the whole K loop (no per-n epilogue bubbles).
// B tiles (one per j1, Kp x Np, fragment-ordered) stream through the same
// TMA bulk-copy / mbarrier ring; u tables arrive per tile as before.
struct KRParams {
  const double* tables;
  Int64x8 toff;
  int64_t ldt;
  int64_t n;
  int64_t ntiles;
  int d;
  int r[kMaxOrder];
  int Kp, Nn, Np, nstage;
  const double* bpack;  // [j1][Kp/4][Np/8][32]
  double* out;
};

struct KRSmem {
  uint32_t bars, u0, u1, uk, bst, ybuf, total;
};

__host__ __device__ inline KRSmem kr_smem(const KRParams& P, int tp, int nh) {
  KRSmem L{};
  uint32_t o = 0;
  L.bars = o;
  o += ((2 * P.nstage + 2) * 8 + 127) / 128 * 128;
  L.u0 = o;
  o += static_cast<uint32_t>(P.Kp) * u0_ld(tp) * 8;
  L.u1 = o;
  o += static_cast<uint32_t>(P.r[1]) * tp * 8;
  L.uk = o;
  for (int k = 2; k < P.d; ++k) o += static_cast<uint32_t>(P.r[k]) * tp * 8;
  o = (o + 127) / 128 * 128;
  L.bst = o;
  o += static_cast<uint32_t>(P.nstage) * P.Kp * P.Np * 8;
  L.ybuf = o;
  o += static_cast<uint32_t>(nh) * tp * 8;
  L.total = o;
  return L;
}

template <int NSW, int D, int NH>
__global__ void __launch_bounds__((64 / 32 * NH + 1) * 32) contract_kr_kernel(const KRParams P) {
  constexpr int TP = 64;
  constexpr int NPG = TP / 32;
  constexpr int NCW = NPG * NH;
  constexpr int NS = NH * NSW;
  constexpr int U0_LD = u0_ld(TP);
  extern __shared__ __align__(1024) unsigned char smem[];
  const KRSmem L = kr_smem(P, TP, NH);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bars);
  uint64_t* empty = full + P.nstage;
  uint64_t* ufull = empty + P.nstage;
  uint64_t* uempty = ufull + 1;
  double* u0s = reinterpret_cast<double*>(smem + L.u0);
  double* u1s = reinterpret_cast<double*>(smem + L.u1);
  double* uks = reinterpret_cast<double*>(smem + L.uk);
  double* bst = reinterpret_cast<double*>(smem + L.bst);
  double* ybuf = reinterpret_cast<double*>(smem + L.ybuf);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int r1 = P.r[1];
  const int stage_elems = P.Kp * P.Np;
  const uint32_t stage_bytes = static_cast<uint32_t>(stage_elems) * 8u;

  if (threadIdx.x == 0) {
    for (int s = 0; s < P.nstage; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    mbar_init(ufull, 1);
    mbar_init(uempty, NCW);
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == NCW) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      uint32_t ubytes = static_cast<uint32_t>(P.Kp + r1) * TP * 8u;
      for (int k = 2; k < P.d; ++k) ubytes += static_cast<uint32_t>(P.r[k]) * TP * 8u;
      for (int64_t tile = blockIdx.x; tile < P.ntiles; tile += gridDim.x, ++it) {
        if (it > 0) mbar_wait(uempty, (it - 1) & 1);
        mbar_arrive_expect_tx(ufull, ubytes);
        const int64_t row0 = tile * TP;
        const double* t0 = P.tables + P.toff.v[0] + row0;
        for (int j = 0; j < P.Kp; ++j) bulk_g2s(u0s + j * U0_LD, t0 + j * P.ldt, TP * 8, ufull);
        const double* t1 = P.tables + P.toff.v[1] + row0;
        for (int j = 0; j < r1; ++j) bulk_g2s(u1s + j * TP, t1 + j * P.ldt, TP * 8, ufull);
        double* dst = uks;
        for (int k = 2; k < P.d; ++k) {
          const double* tk = P.tables + P.toff.v[k] + row0;
          for (int j = 0; j < P.r[k]; ++j) bulk_g2s(dst + j * TP, tk + j * P.ldt, TP * 8, ufull);
          dst += P.r[k] * TP;
        }
        for (int j1 = 0; j1 < r1; ++j1) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full[stage], stage_bytes);
          bulk_g2s(bst + static_cast<size_t>(stage) * stage_elems,
                   P.bpack + static_cast<size_t>(j1) * stage_elems, stage_bytes, &full[stage]);
          if (++stage == P.nstage) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
    return;
  }

  const int pg = warp % NPG;
  const int nh = warp / NPG;
  const int g = lane >> 2, t = lane & 3;
  // Outer-factor offsets of this thread's 2*NSW columns (fixed across tiles).
  int off2[NSW][2], off3[NSW][2];
  bool nval[NSW][2];
#pragma unroll
  for (int b = 0; b < NSW; ++b)
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int nn = (nh * NSW + b) * 8 + 2 * t + i;
      nval[b][i] = nn < P.Nn;
      const int nc = nval[b][i] ? nn : 0;
      if constexpr (D == 3) {
        off2[b][i] = nc * TP;
        off3[b][i] = 0;
      } else {
        off2[b][i] = (nc % P.r[2]) * TP;
        off3[b][i] = (P.r[2] + nc / P.r[2]) * TP;
      }
    }
  int stage = 0;
  uint32_t phase = 0;
  int it = 0;
  const int ksteps = P.Kp / 4;
  for (int64_t tile = blockIdx.x; tile < P.ntiles; tile += gridDim.x, ++it) {
    mbar_wait(ufull, it & 1);
    double acc[4][NSW][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < NSW; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    const double* ua = u0s + t * U0_LD + pg * 32 + g;
    const double* u1p = u1s + pg * 32 + g;
    for (int j1 = 0; j1 < r1; ++j1) {
      double u1v[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) u1v[a] = u1p[j1 * TP + a * 8];
      mbar_wait(&full[stage], phase);
      const double* bb = bst + static_cast<size_t>(stage) * stage_elems + (nh * NSW) * 32 + lane;
#pragma unroll 4
      for (int ks = 0; ks < ksteps; ++ks) {
        double av[4], bv[NSW];
#pragma unroll
        for (int a = 0; a < 4; ++a) av[a] = ua[(4 * ks) * U0_LD + a * 8] * u1v[a];
#pragma unroll
        for (int b = 0; b < NSW; ++b) bv[b] = bb[(ks * NS + b) * 32];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < NSW; ++b) dmma_8x8x4(acc[a][b][0], acc[a][b][1], av[a], bv[b]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == P.nstage) {
        stage = 0;
        phase ^= 1;
      }
    }
    // Epilogue: y_p = sum_n T[p, n] prod_{k>=2} u_k[p, j_k(n)].
    double y[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int row = pg * 32 + a * 8 + g;
      double s = 0.0;
#pragma unroll
      for (int b = 0; b < NSW; ++b)
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          if (!nval[b][i]) continue;
          double o = uks[off2[b][i] + row];
          if constexpr (D == 4) o = o * uks[off3[b][i] + row];
          s = fma(acc[a][b][i], o, s);
        }
      y[a] = s;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(uempty);
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      y[a] += __shfl_xor_sync(0xffffffffu, y[a], 1);
      y[a] += __shfl_xor_sync(0xffffffffu, y[a], 2);
      if (t == 0) ybuf[nh * TP + pg * 32 + a * 8 + g] = y[a];
    }
    consumer_bar<NCW>();
    if (nh == 0) {
      const int row = pg * 32 + lane;
      const int64_t gi = tile * TP + row;
      if (gi < P.n) {
        double v = ybuf[row];
#pragma unroll
        for (int h = 1; h < NH; ++h) v += ybuf[h * TP + row];
        P.out[gi] = v;
      }
    }
    consumer_bar<NCW>();
  }
}

// Generic contraction (any d <= 8, any ranks): thread per point, core read
// through L1/L2 with incremental multi-index; used when the DMMA layout does
// not apply (d == 1, or shared-memory budget exceeded).
__global__ void contract_generic_kernel(const double* __restrict__ tables, Int64x8 toff,
                                        int64_t ldt, int64_t n, int d, Int64x8 ranks,
                                        const double* __restrict__ core, int64_t R,
                                        double* __restrict__ out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int j[kMaxOrder] = {0};
  double y = 0.0;
  for (int64_t lin = 0; lin < R; ++lin) {
    double w = core[lin];
    for (int k = 0; k < d; ++k) w *= tables[toff.v[k] + j[k] * ldt + i];
    y += w;
    for (int k = 0; k < d; ++k) {
      if (++j[k] < ranks.v[k]) break;
      j[k] = 0;
    }
  }
  out[i] = y;
}

// ------------------------------------------------------------- launches ---
static void mode_kernel_attrs(int device) {
  static std::once_flag once[64];
  std::call_once(once[device & 63], [&] {
    const int bytes = (kMaxDegree + 1) * 128 * static_cast<int>(sizeof(double));
    FSTK_CUDA(cudaFuncSetAttribute(mode_tables_kernel<true>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    FSTK_CUDA(cudaFuncSetAttribute(mode_tables_kernel<false>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  });
}

static size_t mode_smem(const fstk_gpu_model* m, int k0, int k1, int threads) {
  mode_kernel_attrs(m->device);
  int pm = 0;
  for (int k = k0; k < k1; ++k) pm = std::max(pm, m->modes[k].pmax);
  return static_cast<size_t>(pm + 1) * threads * sizeof(double);
}

// Coefficients as a by-value kernel parameter (CUDA >= 12.1: up to 32 KB):
// with the degree loop unrolled for a compile-time pmax, every coefficient is
// a constant-bank operand of its FMA -- no shared-memory loads (the MIO stall
// of mode_dense_kernel), no shared memory at all, ~50 registers per thread,
// so these CTAs co-reside with the contraction of the other stream.  The
// arithmetic is mode_dense_kernel's, step for step (bit-identical results).
template <int NQ, int JC>
struct CoefParam {
  double c[NQ][JC];
};

template <bool EXACT, int JC, int P>
__global__ void __launch_bounds__(128) mode_param_kernel(
    const ModeDev md, const CoefParam<P + 1, JC> cp, int j0, const double* __restrict__ xs,
    int64_t n, int64_t n_out, const int64_t* __restrict__ row_src, double* __restrict__ tk,
    int64_t ldt, unsigned long long* err_row) {
  constexpr int PPT = 2;  // rows i and i + 128: each constant operand feeds two FMAs
  const int64_t base = static_cast<int64_t>(blockIdx.x) * (128 * PPT) + threadIdx.x;
  const int jn = min(JC, md.r - j0);
  double t[PPT];
  bool live[PPT];
#pragma unroll
  for (int u = 0; u < PPT; ++u) {
    const int64_t i = base + u * 128;
    live[u] = i < n_out;
    t[u] = 0.0;
    if (!live[u]) continue;
    int64_t src = i;
    bool valid = i < n;
    if (row_src) {
      src = i < n ? row_src[i] : -1;
      valid = src >= 0;
    }
    if (!valid) {
#pragma unroll
      for (int j = 0; j < JC; ++j)
        if (j < jn) tk[(j0 + j) * ldt + i] = 0.0;
      live[u] = false;
      continue;
    }
    const double x = xs[src];
    if (!(x >= md.lo - md.slack && x <= md.hi + md.slack)) {
      atomicMin(err_row, static_cast<unsigned long long>(i));
    } else {
      const double cl = fmin(md.hi, fmax(md.lo, x));
      t[u] = xadd(-1.0, __ddiv_rn(xmul(2.0, xsub(cl, md.lo)), md.span));
    }
  }
  if (!(live[0] || live[1])) return;
  double acc[PPT][JC];
#pragma unroll
  for (int u = 0; u < PPT; ++u)
#pragma unroll
    for (int j = 0; j < JC; ++j) acc[u][j] = 0.0;
  auto apply = [&](const double (&row)[JC], const double (&L)[PPT]) {
#pragma unroll
    for (int j = 0; j < JC; ++j)
#pragma unroll
      for (int u = 0; u < PPT; ++u)
        acc[u][j] = EXACT ? xadd(acc[u][j], xmul(row[j], L[u])) : fma(row[j], L[u], acc[u][j]);
  };
  // legendre_values (basis.cpp:49-61), same rounding sequence.
  double L[PPT], pm1[PPT], pm0[PPT];
#pragma unroll
  for (int u = 0; u < PPT; ++u) L[u] = 1.0;
  apply(cp.c[0], L);
  if (P >= 1) {
#pragma unroll
    for (int u = 0; u < PPT; ++u) L[u] = xmul(c_leg.norm[1], t[u]);
    apply(cp.c[1], L);
  }
#pragma unroll
  for (int u = 0; u < PPT; ++u) {
    pm1[u] = 1.0;
    pm0[u] = t[u];
  }
#pragma unroll
  for (int q = 1; q < P; ++q) {
#pragma unroll
    for (int u = 0; u < PPT; ++u) {
      const double num = xsub(xmul(xmul(c_leg.a[q], t[u]), pm0[u]), xmul(c_leg.b[q], pm1[u]));
      const double pn1 = xdiv_small(num, c_leg.c[q], c_leg.rc[q]);
      pm1[u] = pm0[u];
      pm0[u] = pn1;
      L[u] = xmul(c_leg.norm[q + 1], pn1);
    }
    apply(cp.c[q + 1], L);
  }
#pragma unroll
  for (int u = 0; u < PPT; ++u) {
    if (!live[u]) continue;
    const int64_t i = base + u * 128;
#pragma unroll
    for (int j = 0; j < JC; ++j)
      if (j < jn) tk[(j0 + j) * ldt + i] = acc[u][j];
  }
}

template <bool EXACT, int JC, int P>
static void launch_param_t(const ModeDev& md, const double* xs, int64_t n, int64_t n_out,
                           const int64_t* row_src, double* tk, int64_t ldt,
                           unsigned long long* err_row, cudaStream_t s) {
  for (int c = 0; c < md.nchunk; ++c) {
    CoefParam<P + 1, JC> cp;
    for (int q = 0; q <= P; ++q)
      for (int j = 0; j < JC; ++j) cp.c[q][j] = md.h_dense[static_cast<size_t>(q) * md.ldc + c * JC + j];
    mode_param_kernel<EXACT, JC, P><<<static_cast<unsigned>(ceil_div(n_out, 256)), 128, 0, s>>>(
        md, cp, c * JC, xs, n, n_out, row_src, tk, ldt, err_row);
    check_launch("mode_param_kernel");
  }
}

// The parameter kernel for the (pmax, jc) pairs it is instantiated for
// (measured: C2 +3%, C1 +7%, C4 +2% over mode_dense_kernel).
template <bool EXACT>
static bool launch_param(const ModeDev& md, const double* xs, int64_t n, int64_t n_out,
                         const int64_t* row_src, double* tk, int64_t ldt,
                         unsigned long long* err_row, cudaStream_t s) {
  static const bool on = [] {
    const char* e = std::getenv("FSTK_MODE_PARAM");
    return !(e && std::atoi(e) == 0);
  }();
  if (!on || !md.h_dense) return false;
#define FSTK_PJ(P, J)                                                                 \
  if (md.pmax == P && md.jc == J) {                                                    \
    launch_param_t<EXACT, J, P>(md, xs, n, n_out, row_src, tk, ldt, err_row, s);       \
    return true;                                                                       \
  }
#define FSTK_P(P) FSTK_PJ(P, 8) FSTK_PJ(P, 16) FSTK_PJ(P, 32)
  // pmax 64 measured slower (C3: its 16.6 KB block streams poorly through the
  // constant cache when no co-residency is possible): shared-memory kernel.
  FSTK_P(16) FSTK_P(20) FSTK_P(32) FSTK_P(48)
#undef FSTK_P
#undef FSTK_PJ
  return false;
}

template <bool EXACT, int JC>
static void launch_dense_t(const ModeDev& md, const double* xs, int64_t n, int64_t n_out,
                           const int64_t* row_src, double* tk, int64_t ldt,
                           unsigned long long* err_row, cudaStream_t s, int device) {
  static std::once_flag once[64];
  constexpr int smax = (kMaxDegree + 1) * JC * static_cast<int>(sizeof(double));
  std::call_once(once[device & 63], [&] {
    FSTK_CUDA(cudaFuncSetAttribute(mode_dense_kernel<EXACT, JC, 1>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, smax));
    FSTK_CUDA(cudaFuncSetAttribute(mode_dense_kernel<EXACT, JC, DensePPT<EXACT, JC>::value>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, smax));
  });
  // FSTK_MODE_PPT=1: one point per thread (fewer registers, so mode CTAs can
  // co-reside with the contraction of the other stream).
  static const bool one = [] {
    const char* e = std::getenv("FSTK_MODE_PPT");
    return e && std::atoi(e) == 1;
  }();
  const size_t sm = static_cast<size_t>(md.pmax + 1) * JC * sizeof(double);
  constexpr int ppt = DensePPT<EXACT, JC>::value;
  const int rows_per_cta = 128 * (one ? 1 : ppt);
  dim3 grid(static_cast<unsigned>(ceil_div(n_out, rows_per_cta)), static_cast<unsigned>(md.nchunk));
  if (one || ppt == 1)
    mode_dense_kernel<EXACT, JC, 1><<<grid, 128, sm, s>>>(md, xs, n, n_out, row_src, tk, ldt, err_row);
  else
    mode_dense_kernel<EXACT, JC, ppt><<<grid, 128, sm, s>>>(md, xs, n, n_out, row_src, tk, ldt, err_row);
  check_launch("mode_dense_kernel");
}

template <bool EXACT>
static void launch_dense(const ModeDev& md, const double* xs, int64_t n, int64_t n_out,
                         const int64_t* row_src, double* tk, int64_t ldt,
                         unsigned long long* err_row, cudaStream_t s, int device) {
  switch (md.jc) {
#define FSTK_JC(J) \
  case J: launch_dense_t<EXACT, J>(md, xs, n, n_out, row_src, tk, ldt, err_row, s, device); break;
    FSTK_JC(8) FSTK_JC(16) FSTK_JC(24) FSTK_JC(32) FSTK_JC(40) FSTK_JC(48) FSTK_JC(56) FSTK_JC(64)
#undef FSTK_JC
    default: fail(FSTK_E_COMPUTE, "internal: bad dense chunk width");
  }
}

// One mode's table: wavelet-capable general kernel, dense Legendre kernel, or
// the sparse Legendre kernel (indices not strictly increasing).
static void launch_mode_k(const fstk_gpu_model* m, int k, const double* xs, int64_t n,
                          int64_t n_out, const int64_t* row_src, double* tk, int64_t ldt,
                          bool exact, unsigned long long* err_row, cudaStream_t s) {
  if (m->modes[k].general) {
    launch_mode_general(m->gen[k], xs, n, n_out, row_src, tk, ldt, exact, err_row, s, m->device);
    return;
  }
  const ModeDev& md = m->modes_dev.m[k];
  if (m->modes[k].sorted) {
    if (exact) {
      if (!launch_param<true>(md, xs, n, n_out, row_src, tk, ldt, err_row, s))
        launch_dense<true>(md, xs, n, n_out, row_src, tk, ldt, err_row, s, m->device);
    } else if (!launch_param<false>(md, xs, n, n_out, row_src, tk, ldt, err_row, s)) {
      launch_dense<false>(md, xs, n, n_out, row_src, tk, ldt, err_row, s, m->device);
    }
    return;
  }
  const int threads = 128;
  Int64x8 to{};
  to.v[k] = 0;
  const size_t sm = mode_smem(m, k, k + 1, threads);
  const unsigned blocks = static_cast<unsigned>(ceil_div(n_out, threads));
  // pts[k * ldp + src] with ldp = 0 addresses xs[src].
  if (exact)
    mode_tables_kernel<true><<<blocks, threads, sm, s>>>(m->modes_dev, k, k + 1, xs, 0, n, n_out,
                                                         row_src, tk, to, ldt, err_row);
  else
    mode_tables_kernel<false><<<blocks, threads, sm, s>>>(m->modes_dev, k, k + 1, xs, 0, n, n_out,
                                                          row_src, tk, to, ldt, err_row);
  check_launch("mode_tables_kernel");
}

void launch_mode_tables(const fstk_gpu_model* m, const double* pts, int64_t ldp, int64_t n,
                        int64_t n_out, const int64_t* row_src, double* tables,
                        const int64_t* toff, int64_t ldt, bool exact,
                        unsigned long long* err_row, cudaStream_t s) {
  if (n_out <= 0) return;
  ProfScope prof(FSTK_PROF_MODE_TABLES, s);
  for (int k = 0; k < m->d; ++k)
    launch_mode_k(m, k, pts + k * ldp, n, n_out, row_src, tables + toff[k], ldt, exact, err_row, s);
}

void launch_mode_table_one(const fstk_gpu_model* m, int mode, const double* x, int64_t n,
                           double* out, int64_t ldt, bool exact, unsigned long long* err_row,
                           cudaStream_t s) {
  if (n <= 0) return;
  launch_mode_k(m, mode, x, n, n, nullptr, out, ldt, exact, err_row, s);
}

void eval_table_offsets(const fstk_gpu_model* m, int64_t ldt, int64_t* toff, int64_t* total) {
  int64_t o = 0;
  for (int k = 0; k < m->d; ++k) {
    toff[k] = o;
    o += static_cast<int64_t>(m->rp[k]) * ldt;
  }
  *total = o;
}

static ContractParams make_params(const fstk_gpu_model* m, const double* tables,
                                  const int64_t* toff, int64_t ldt, int64_t n, double* out) {
  ContractParams P{};
  P.tables = tables;
  for (int k = 0; k < m->d; ++k) P.toff.v[k] = toff[k];
  P.ldt = ldt;
  P.n = n;
  P.ntiles = ceil_div(n, m->lay.tp);
  P.d = m->d;
  for (int k = 0; k < m->d; ++k) P.r[k] = static_cast<int>(m->ranks[k]);
  P.Kp = m->lay.Kp;
  P.N1p = m->lay.N1p;
  P.NC = m->lay.NC;
  P.Mout = m->lay.Mout;
  P.N1 = m->lay.NC * m->lay.N1p;
  P.nstage = m->lay.nstage;
  P.bpack = m->d_bpack.p;
  P.out = out;
  return P;
}

template <int NSW, int D, int TPL, int NH>
static void launch_contract_t(const fstk_gpu_model* m, const ContractParams& P, cudaStream_t s) {
  static std::once_flag once[64];
  const size_t smem = m->lay.smem;
  std::call_once(once[m->device & 63], [&] {
    int optin = 0;
    FSTK_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, m->device));
    FSTK_CUDA(cudaFuncSetAttribute(contract_kernel<NSW, D, TPL, NH>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
  });
  const int64_t grid = std::min<int64_t>(P.ntiles, static_cast<int64_t>(m->num_sms) * m->lay.ctas_per_sm);
  contract_kernel<NSW, D, TPL, NH><<<static_cast<unsigned>(grid), (TPL / 32 * NH + 1) * 32, smem, s>>>(P);
  check_launch("contract_kernel");
}

template <int NSW, int D, int NH>
static void launch_contract_tp(const fstk_gpu_model* m, const ContractParams& P, cudaStream_t s) {
  if (m->lay.tp == 64)
    launch_contract_t<NSW, D, 64, NH>(m, P, s);
  else
    launch_contract_t<NSW, D, 128, NH>(m, P, s);
}

template <int NSW, int NH>
static void launch_contract_d(const fstk_gpu_model* m, const ContractParams& P, cudaStream_t s) {
  switch (m->d) {
    case 2: launch_contract_tp<NSW, 2, NH>(m, P, s); break;
    case 3: launch_contract_tp<NSW, 3, NH>(m, P, s); break;
    case 4: launch_contract_tp<NSW, 4, NH>(m, P, s); break;
    default: launch_contract_tp<NSW, 0, NH>(m, P, s); break;
  }
}

template <int NSW, int D, int NH>
static void launch_kr_t(const fstk_gpu_model* m, const KRParams& P, cudaStream_t s) {
  static std::once_flag once[64];
  std::call_once(once[m->device & 63], [&] {
    int optin = 0;
    FSTK_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, m->device));
    FSTK_CUDA(cudaFuncSetAttribute(contract_kr_kernel<NSW, D, NH>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
  });
  const int64_t grid = std::min<int64_t>(P.ntiles, static_cast<int64_t>(m->num_sms) * m->lay.ctas_per_sm);
  contract_kr_kernel<NSW, D, NH><<<static_cast<unsigned>(grid), (2 * NH + 1) * 32, m->lay.smem, s>>>(P);
  check_launch("contract_kr_kernel");
}

template <int D, int NH>
static void launch_kr_n(const fstk_gpu_model* m, const KRParams& P, cudaStream_t s) {
  switch (m->lay.nsw) {
    case 2: launch_kr_t<2, D, NH>(m, P, s); break;
    case 3: launch_kr_t<3, D, NH>(m, P, s); break;
    case 4: launch_kr_t<4, D, NH>(m, P, s); break;
    default: fail(FSTK_E_COMPUTE, "internal: bad KR layout");
  }
}

template <int D>
static void launch_kr_h(const fstk_gpu_model* m, const KRParams& P, cudaStream_t s) {
  switch (m->lay.nh) {
    case 1: launch_kr_n<D, 1>(m, P, s); break;
    case 2: launch_kr_n<D, 2>(m, P, s); break;
    case 4: launch_kr_n<D, 4>(m, P, s); break;
    default: fail(FSTK_E_COMPUTE, "internal: bad KR layout");
  }
}

static void launch_kr(const fstk_gpu_model* m, const KRParams& P, cudaStream_t s) {
  if (m->d == 3)
    launch_kr_h<3>(m, P, s);
  else
    launch_kr_h<4>(m, P, s);
}

void launch_contract(const fstk_gpu_model* m, const double* tables, const int64_t* toff,
                     int64_t ldt, int64_t n, double* out, cudaStream_t s,
                     const double* bpack_override, const double* core_override) {
  if (n <= 0) return;
  ProfScope prof(FSTK_PROF_CONTRACT, s);
  if (!m->lay.fast) {
    Int64x8 to{}, rk{};
    for (int k = 0; k < m->d; ++k) {
      to.v[k] = toff[k];
      rk.v[k] = m->ranks[k];
    }
    contract_generic_kernel<<<static_cast<unsigned>(ceil_div(n, 128)), 128, 0, s>>>(
        tables, to, ldt, n, m->d, rk, core_override ? core_override : m->d_core.p, m->R, out);
    check_launch("contract_generic_kernel");
    return;
  }
  if (m->lay.kr) {
    KRParams P{};
    P.tables = tables;
    for (int k = 0; k < m->d; ++k) {
      P.toff.v[k] = toff[k];
      P.r[k] = static_cast<int>(m->ranks[k]);
    }
    P.ldt = ldt;
    P.n = n;
    P.ntiles = ceil_div(n, 64);
    P.d = m->d;
    P.Kp = m->lay.Kp;
    P.Nn = m->lay.Mout;
    P.Np = m->lay.kr_np;
    P.nstage = m->lay.nstage;
    P.bpack = bpack_override ? bpack_override : m->d_bpack.p;
    P.out = out;
    launch_kr(m, P, s);
    return;
  }
  ContractParams P = make_params(m, tables, toff, ldt, n, out);
  if (bpack_override) P.bpack = bpack_override;
  if (m->lay.nh == 1) {
    switch (m->lay.nsw) {  // NSW = N1p / 8
      case 2: launch_contract_d<2, 1>(m, P, s); break;
      case 4: launch_contract_d<4, 1>(m, P, s); break;
      case 6: launch_contract_d<6, 1>(m, P, s); break;
      default: fail(FSTK_E_COMPUTE, "internal: bad contraction layout");
    }
    return;
  }
  switch (m->lay.nsw) {  // NSW = N1p / 16
    case 1: launch_contract_d<1, 2>(m, P, s); break;
    case 2: launch_contract_d<2, 2>(m, P, s); break;
    case 3: launch_contract_d<3, 2>(m, P, s); break;
    case 4: launch_contract_d<4, 2>(m, P, s); break;
    default: fail(FSTK_E_COMPUTE, "internal: bad contraction layout");
  }
}

// ------------------------------------------------------------ model setup ---
// Chooses the tile (TP = 64 or 128 points) and ring depth that maximise
// resident consumer warps per SM (so one CTA's u-table prologue overlaps the
// other CTAs' DMMA work), preferring deeper rings at equal residency.
// Khatri-Rao form (d = 3, 4): K = r0 r1, N = prod_{k>=2} r_k <= 128 split over
// NH warps of NSW 8-column subtiles; TP = 64 points; ring depth and residency
// as for the classic layout.
static bool plan_kr(fstk_gpu_model* m) {
  ContractLayout& L = m->lay;
  if (!(m->d == 3 || m->d == 4)) return false;
  // Measured on B200 (round 1): the KR form wins for d = 4 (C4 +4%) and loses
  // for d = 3 (C1 -12%, C2 -4%, C3 -3%: the per-fragment DMUL sits on the
  // A-operand path); FSTK_CONTRACT_KR=0/1 overrides.
  bool want = m->d == 4;
  if (const char* e = std::getenv("FSTK_CONTRACT_KR")) want = std::atoi(e) != 0;
  if (!want) return false;
  int Nn = 1;
  for (int k = 2; k < m->d; ++k) Nn *= static_cast<int>(m->ranks[k]);
  int best_np = 1 << 30, bnh = 0, bnsw = 0;
  for (int nh : {2, 1, 4})
    for (int nsw : {2, 3, 4}) {
      const int np = nh * nsw * 8;
      if (np >= Nn && np < best_np) {
        best_np = np;
        bnh = nh;
        bnsw = nsw;
      }
    }
  if (const char* e = std::getenv("FSTK_KR_NH")) {
    const int nh = std::atoi(e);
    for (int nsw : {2, 3, 4})
      if ((nh == 1 || nh == 2 || nh == 4) && nh * nsw * 8 >= Nn) {
        bnh = nh;
        bnsw = nsw;
        best_np = nh * nsw * 8;
        break;
      }
  }
  if (!bnh) return false;
  L.Kp = static_cast<int>(round_up(m->ranks[0], 4));
  L.Mout = Nn;
  L.kr_np = best_np;
  L.nh = bnh;
  L.nsw = bnsw;
  int optin = 0, per_sm = 0;
  FSTK_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, m->device));
  FSTK_CUDA(cudaDeviceGetAttribute(&per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, m->device));
  double best = -1;
  for (int ns = 2; ns <= 6; ++ns) {
    KRParams P{};
    P.d = m->d;
    for (int k = 0; k < m->d; ++k) P.r[k] = static_cast<int>(m->ranks[k]);
    P.Kp = L.Kp;
    P.Np = L.kr_np;
    P.nstage = ns;
    const KRSmem S = kr_smem(P, 64, L.nh);
    if (S.total > static_cast<uint32_t>(optin)) continue;
    const int ctas = std::min<int>(per_sm / static_cast<int>(S.total + 1024), 4);
    if (ctas < 1) continue;
    const int warps = ctas * 2 * L.nh;
    const double score =
        std::min(warps, 16) * 100.0 + std::min(ctas, 3) * 50.0 + std::min(ns, 4) * 10.0;
    if (score > best) {
      best = score;
      L.nstage = ns;
      L.smem = S.total;
      L.ctas_per_sm = ctas;
    }
  }
  if (best < 0) return false;
  L.kr = true;
  L.fast = true;
  L.tp = 64;
  m->rp[0] = L.Kp;
  m->rp[1] = static_cast<int>(m->ranks[1]);
  return true;
}

static void plan_layout(fstk_gpu_model* m) {
  ContractLayout& L = m->lay;
  L = ContractLayout{};
  for (int k = 0; k < m->d; ++k) m->rp[k] = static_cast<int>(m->ranks[k]);
  if (m->d < 2) return;
  if (plan_kr(m)) return;
  L = ContractLayout{};
  const int r0 = static_cast<int>(m->ranks[0]), r1 = static_cast<int>(m->ranks[1]);
  L.Kp = static_cast<int>(round_up(r0, 4));
  const int r1p = static_cast<int>(round_up(r1, 16));
  L.N1p = std::min(r1p, 64);
  L.NC = static_cast<int>(ceil_div(r1, L.N1p));
  L.Mout = 1;
  for (int k = 2; k < m->d; ++k) L.Mout *= static_cast<int>(m->ranks[k]);
  // Column groups per 32-point group: 1 (a warp owns all N1p/8 subtiles:
  // more independent DMMAs, half the A-fragment loads) or 2.
  // Measured on B200 (round 1): one group wins at N1p = 16 (C1 +7%, C4 +4%),
  // two groups win at N1p >= 32 (register pressure of 4-6 subtiles per warp).
  L.nh = L.N1p <= 16 ? 1 : 2;
  if (const char* e = std::getenv("FSTK_CONTRACT_NH")) L.nh = std::atoi(e) == 1 ? 1 : 2;
  if (L.nh == 1 && L.N1p > 48) L.nh = 2;
  L.nsw = L.N1p / (8 * L.nh);
  L.btile_elems = static_cast<int64_t>(L.Kp) * L.N1p;
  int optin = 0, per_sm = 0;
  FSTK_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, m->device));
  FSTK_CUDA(cudaDeviceGetAttribute(&per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, m->device));
  double best = -1;
  const int force_ns = std::getenv("FSTK_CONTRACT_NSTAGE") ? std::atoi(std::getenv("FSTK_CONTRACT_NSTAGE")) : 0;
  const int force_ctas = std::getenv("FSTK_CONTRACT_CTAS") ? std::atoi(std::getenv("FSTK_CONTRACT_CTAS")) : 0;
  for (int tp : {64, 128}) {
    for (int ns = 2; ns <= 6; ++ns) {
      if (force_ns && ns != force_ns) continue;
      ContractParams P{};
      P.d = m->d;
      for (int k = 0; k < m->d; ++k) P.r[k] = static_cast<int>(m->ranks[k]);
      P.Kp = L.Kp;
      P.N1p = L.N1p;
      P.NC = L.NC;
      P.N1 = L.NC * L.N1p;
      P.nstage = ns;
      const SmemLayout S = smem_layout(P, tp);
      if (S.total > static_cast<uint32_t>(optin)) continue;
      int ctas = std::min<int>(per_sm / static_cast<int>(S.total + 1024), 4);
      if (force_ctas) ctas = std::min(ctas, force_ctas);
      if (ctas < 1) continue;
      const int warps = ctas * (tp / 32 * L.nh);
      const double score =
          std::min(warps, 16) * 100.0 + std::min(ctas, 3) * 50.0 + std::min(ns, 4) * 10.0 + tp / 64.0;
      if (score > best) {
        best = score;
        L.tp = tp;
        L.nstage = ns;
        L.smem = S.total;
        L.ctas_per_sm = ctas;
        L.fast = true;
      }
    }
  }
  if (L.fast) {
    m->rp[0] = L.Kp;
    m->rp[1] = L.NC * L.N1p;
  }
  if (std::getenv("FSTK_DEBUG_LAYOUT"))
    std::fprintf(stderr, "fstk layout: tp=%d nstage=%d ctas/sm=%d nh=%d nsw=%d smem=%zu kr=%d\n",
                 L.tp, L.nstage, L.ctas_per_sm, L.nh, L.nsw, L.smem, L.kr ? 1 : 0);
}

static void pack_core_into(const fstk_gpu_model* m, const double* core, DevBuf<double>& out) {
  const ContractLayout& L = m->lay;
  if (!L.fast) return;
  const int r0 = static_cast<int>(m->ranks[0]), r1 = static_cast<int>(m->ranks[1]);
  if (L.kr) {
    // [j1][ks][nsub][lane]: G[k = 4 ks + lane%4, j1, n = 8 nsub + lane/4]
    const int NSB = L.kr_np / 8;
    const int64_t tile = static_cast<int64_t>(L.Kp) * L.kr_np;
    std::vector<double> bp(static_cast<size_t>(r1 * tile), 0.0);
    for (int j1 = 0; j1 < r1; ++j1)
      for (int ks = 0; ks < L.Kp / 4; ++ks)
        for (int ns = 0; ns < NSB; ++ns)
          for (int lane = 0; lane < 32; ++lane) {
            const int k = 4 * ks + (lane & 3);
            const int nn = 8 * ns + (lane >> 2);
            double v = 0.0;
            if (k < r0 && nn < L.Mout)
              v = core[static_cast<size_t>(k + static_cast<int64_t>(r0) * (j1 + static_cast<int64_t>(r1) * nn))];
            bp[static_cast<size_t>(j1 * tile + (ks * NSB + ns) * 32 + lane)] = v;
          }
    out.alloc(bp.size());
    FSTK_CUDA(cudaMemcpy(out.p, bp.data(), bp.size() * sizeof(double), cudaMemcpyHostToDevice));
    return;
  }
  const int NS = L.N1p / 8;
  const int64_t NT = static_cast<int64_t>(L.NC) * L.Mout;
  std::vector<double> bp(static_cast<size_t>(NT * L.btile_elems), 0.0);
  for (int64_t tt = 0; tt < NT; ++tt) {
    const int c = static_cast<int>(tt % L.NC);
    const int64_t mo = tt / L.NC;
    double* tile = bp.data() + tt * L.btile_elems;
    for (int ks = 0; ks < L.Kp / 4; ++ks)
      for (int ns = 0; ns < NS; ++ns)
        for (int lane = 0; lane < 32; ++lane) {
          const int k = 4 * ks + (lane & 3);
          const int j1 = c * L.N1p + 8 * ns + (lane >> 2);
          double v = 0.0;
          if (k < r0 && j1 < r1)
            v = core[static_cast<size_t>(k + static_cast<int64_t>(r0) * (j1 + static_cast<int64_t>(r1) * mo))];
          tile[(ks * NS + ns) * 32 + lane] = v;
        }
  }
  out.alloc(bp.size());
  FSTK_CUDA(cudaMemcpy(out.p, bp.data(), bp.size() * sizeof(double), cudaMemcpyHostToDevice));
}

static void pack_core(fstk_gpu_model* m) { pack_core_into(m, m->core.data(), m->d_bpack); }

static void upload_core(fstk_gpu_model* m) {
  FSTK_CUDA(cudaMemcpy(m->d_core.p, m->core.data(), m->core.size() * sizeof(double),
                       cudaMemcpyHostToDevice));
  pack_core(m);
}

[[noreturn]] void throw_domain(const fstk_gpu_model* m, int64_t row, const double* y) {
  Error e{FSTK_E_DOMAIN, "point outside basis domain"};
  e.index = row;
  for (int k = 0; k < m->d; ++k) {
    const ModeHost& mh = m->modes[k];
    const double span = mh.hi - mh.lo;
    const double slack = 1e-12 * span;
    if (!(y[k] >= mh.lo - slack && y[k] <= mh.hi + slack)) {
      e.mode = k;
      e.value = y[k];
      break;
    }
  }
  throw e;
}

// Evaluates n device-resident points in chunks of the model's workspace,
// optionally with a replacement core (host pointer, e.g. a refit result).
// Chunks alternate between the two workspace streams so the mode-table
// kernel of chunk i+1 runs concurrently with the DMMA contraction of chunk i
// (both are fp64-pipe bound with complementary stalls).  Chunk c records its
// lowest failing row in m->chunk_err[c]; the caller's stream `s` is joined
// at the end.
// Chunk begins of a q-point evaluation (the last entry is q): full chunks of
// CH, except that with `ramp` slabs of >= 4 chunks ramp their first and last
// chunks (CH/8, CH/4, CH/2 and back), so the work that cannot overlap
// another chunk -- the first upload or mode-table pass, the last read-back --
// is small.  Chunking never changes a point's value (position independence).
static std::vector<int64_t> chunk_begins(int64_t q, int64_t CH, bool ramp) {
  std::vector<int64_t> cb{0};
  const int64_t r8 = round_up(std::max<int64_t>(CH / 8, 128), 128);
  if (ramp && q >= 4 * CH && CH >= 1024) {
    const int64_t steps[3] = {r8, 2 * r8, 4 * r8};
    for (int64_t x : steps) cb.push_back(cb.back() + x);
    const int64_t mid_end = q - 7 * r8;
    while (cb.back() + CH <= mid_end) cb.push_back(cb.back() + CH);
    if (cb.back() < mid_end) cb.push_back(mid_end);
    for (int i = 2; i >= 0; --i) cb.push_back(cb.back() + steps[i]);
  } else {
    for (int64_t b = CH; b < q; b += CH) cb.push_back(b);
    cb.push_back(std::max<int64_t>(q, 0));
  }
  return cb;
}

// Allocates and zeroes the padded table workspaces of both chunk slots on
// first use (padding rows stay 0 afterwards).  Caller holds m->mu.
void ensure_chunk_workspace(const fstk_gpu_model* m) {
  for (auto& ck : m->chunk) {
    if (ck.tables.p) continue;
    int64_t toff[kMaxOrder], tot = 0;
    eval_table_offsets(m, round_up(m->chunk_points, 128), toff, &tot);
    ck.tables.alloc(static_cast<size_t>(tot));
    FSTK_CUDA(cudaMemsetAsync(ck.tables.p, 0, static_cast<size_t>(tot) * 8, ck.stream));
    ck.err.alloc(1);
    ck.points.alloc(static_cast<size_t>(m->d) * m->chunk_points);
    ck.out.alloc(static_cast<size_t>(m->chunk_points));
    FSTK_CUDA(cudaStreamSynchronize(ck.stream));
  }
}

// fstk_gpu_eval_serialize: every chunk on the first workspace stream, so the
// mode-table and contraction kernels never overlap (a measurement mode: their
// event durations are then the kernels' own, for the roofline).
static std::atomic<int> g_eval_serial{0};

void evaluate_device_core(const fstk_gpu_model* m, const double* core_host, const double* pts,
                          int64_t ldp, int64_t n, double* out, cudaStream_t s) {
  ensure_chunk_workspace(m);
  const int lanes = g_eval_serial.load() ? 1 : 2;
  const int64_t CH = m->chunk_points;
  int64_t toff[kMaxOrder], tot = 0;
  const int64_t ldt = round_up(CH, 128);
  eval_table_offsets(m, ldt, toff, &tot);
  DevBuf<double> bp, craw;
  if (core_host) {
    pack_core_into(m, core_host, bp);
    craw.alloc(m->R);
    FSTK_CUDA(cudaMemcpy(craw.p, core_host, m->R * 8, cudaMemcpyHostToDevice));
  }
  // Device-resident inputs: uniform chunks (a ramp measured no faster here;
  // the first two chunks' mode passes already run concurrently).
  const std::vector<int64_t> cb = chunk_begins(n, CH, false);
  const int64_t nchunks = std::max<int64_t>(1, static_cast<int64_t>(cb.size()) - 1);
  m->chunk_err.ensure(static_cast<size_t>(nchunks));
  FSTK_CUDA(cudaMemsetAsync(m->chunk_err.p, 0xff, nchunks * sizeof(unsigned long long), s));
  FSTK_CUDA(cudaEventRecord(m->fork_ev, s));
  for (auto& ck : m->chunk) FSTK_CUDA(cudaStreamWaitEvent(ck.stream, m->fork_ev, 0));
  for (int64_t c = 0; c + 1 < static_cast<int64_t>(cb.size()) && cb[c] < n; ++c) {
    Chunk& ck = m->chunk[c & 1];
    cudaStream_t cs = m->chunk[lanes == 1 ? 0 : (c & 1)].stream;
    const int64_t b = cb[c];
    const int64_t nb = cb[c + 1] - b;
    const int64_t nout = round_up(nb, 128);
    launch_mode_tables(m, pts + b, ldp, nb, nout, nullptr, ck.tables.p, toff, ldt, false,
                       m->chunk_err.p + c, cs);
    launch_contract(m, ck.tables.p, toff, ldt, nb, out + b, cs,
                    core_host ? bp.p : nullptr, core_host ? craw.p : nullptr);
  }
  for (auto& ck : m->chunk) {
    FSTK_CUDA(cudaEventRecord(ck.done, ck.stream));
    FSTK_CUDA(cudaStreamWaitEvent(s, ck.done, 0));
  }
  if (core_host) FSTK_CUDA(cudaStreamSynchronize(s));  // temporaries go out of scope
}

// Lowest failing row over the chunks of the last evaluate_device call (or -1);
// synchronises `s`.
int64_t evaluate_device_error(const fstk_gpu_model* m, int64_t n, cudaStream_t s) {
  const std::vector<int64_t> cb = chunk_begins(n, m->chunk_points, false);
  const int64_t nchunks = std::max<int64_t>(1, static_cast<int64_t>(cb.size()) - 1);
  std::vector<unsigned long long> bad(static_cast<size_t>(nchunks));
  FSTK_CUDA(cudaMemcpyAsync(bad.data(), m->chunk_err.p, nchunks * sizeof(unsigned long long),
                            cudaMemcpyDeviceToHost, s));
  FSTK_CUDA(cudaStreamSynchronize(s));
  for (int64_t c = 0; c < nchunks; ++c)
    if (bad[c] != ULLONG_MAX) return cb[c] + static_cast<int64_t>(bad[c]);
  return -1;
}

void evaluate_device(const fstk_gpu_model* m, const double* pts, int64_t ldp, int64_t n,
                     double* out, cudaStream_t s) {
  evaluate_device_core(m, nullptr, pts, ldp, n, out, s);
}

}  // namespace fstk_gpu

using namespace fstk_gpu;

fstk_gpu_model::~fstk_gpu_model() {
  for (auto& c : chunk) {
    if (c.stream) cudaStreamDestroy(c.stream);
    if (c.done) cudaEventDestroy(c.done);
    if (c.host_done) cudaEventDestroy(c.host_done);
    if (c.h_stage) cudaFreeHost(c.h_stage);
  }
  if (fork_ev) cudaEventDestroy(fork_ev);
}

// ================================================================= C-ABI ===
extern "C" {

int32_t fstk_gpu_abi_version(void) { return FSTK_GPU_ABI_VERSION; }

int32_t fstk_gpu_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

uint64_t fstk_gpu_launch_count(void) { return g_launches.load(); }

int32_t fstk_gpu_eval_serialize(int32_t on) { return g_eval_serial.exchange(on ? 1 : 0); }

int32_t fstk_gpu_set_device_cache(int32_t policy) {
  const int prev = device_cache_policy().exchange(policy <= 0 ? 0 : (policy >= 2 ? 2 : 1));
  if (policy <= 0 || (policy == 1 && device_cache_sessions().load() == 0)) device_cache_trim(-1);
  return prev;
}

uint64_t fstk_gpu_trim_device_cache(int32_t device) {
  DeviceCache& c = device_cache();
  size_t before;
  {
    std::lock_guard<std::mutex> lk(c.mu);
    before = c.cached;
  }
  device_cache_trim(device);
  std::lock_guard<std::mutex> lk(c.mu);
  return before - c.cached;
}

namespace fstk_gpu {
static void rethrow_stage_code(int32_t c, const fstk_gpu_error* err) {
  if (!c) return;
  Error e{c, err ? err->message : "stage failed"};
  throw e;
}
static std::mutex g_dev_mu;
static std::vector<int> g_devices;  // fstk_gpu_set_devices; empty = the current device
}  // namespace fstk_gpu

int32_t fstk_gpu_set_devices(int32_t n, const int32_t* ids, fstk_gpu_error* err) {
  using namespace fstk_gpu;
  return guarded(err, [&] {
    require(n >= 0 && (n == 0 || ids), FSTK_E_PARAMETER, "set_devices: bad device list");
    int count = 0;
    FSTK_CUDA(cudaGetDeviceCount(&count));
    std::vector<int> v;
    for (int i = 0; i < n; ++i) {
      require(ids[i] >= 0 && ids[i] < count, FSTK_E_PARAMETER, "set_devices: no such device");
      v.push_back(ids[i]);
    }
    std::lock_guard<std::mutex> lk(g_dev_mu);
    g_devices = v;
  });
}

int32_t fstk_gpu_model_create(const fstk_model_desc* desc, int32_t device, fstk_gpu_model** out,
                              fstk_gpu_error* err) {
  if (device < 0) {
    // The device list of fstk_gpu_set_devices: the model on the first device,
    // replicas on the others (a host evaluate_batch then splits across all).
    std::vector<int> ids;
    {
      std::lock_guard<std::mutex> lk(fstk_gpu::g_dev_mu);
      ids = fstk_gpu::g_devices;
    }
    if (ids.empty()) {
      int cur = 0;
      cudaGetDevice(&cur);
      ids.push_back(cur);
    }
    const int32_t rc = fstk_gpu_model_create(desc, ids[0], out, err);
    if (rc) return rc;
    for (size_t i = 1; i < ids.size(); ++i) {
      fstk_gpu_model* r = nullptr;
      const int32_t rc2 = fstk_gpu_model_create(desc, ids[i], &r, err);
      if (rc2) {
        fstk_gpu_model_destroy(*out);
        *out = nullptr;
        return rc2;
      }
      (*out)->replicas.push_back(r);
    }
    return 0;
  }
  return guarded(err, [&] {
    require(desc != nullptr && out != nullptr, FSTK_E_PARAMETER, "null argument");
    *out = nullptr;
    const int d = desc->d;
    // model.cpp:31-53 validate_structure + basis.cpp:30-47 validate.
    require(d >= 1 && d <= kMaxOrder, FSTK_E_SHAPE, "model: mode count does not match core order");
    auto m = std::make_unique<fstk_gpu_model>();
    m->device = device;
    m->d = d;
    m->ranks.assign(desc->ranks, desc->ranks + d);
    m->R = 1;
    for (int k = 0; k < d; ++k) {
      require(m->ranks[k] >= 1, FSTK_E_SHAPE, "model: empty mode");
      m->R *= m->ranks[k];
    }
    m->core.assign(desc->core, desc->core + m->R);
    m->modes.resize(d);
    size_t f = 0, c = 0;
    for (int k = 0; k < d; ++k) {
      ModeHost& mh = m->modes[k];
      mh.r = static_cast<int>(m->ranks[k]);
      mh.rowptr.push_back(0);
      for (int j = 0; j < mh.r; ++j, ++f) {
        const int fam = desc->family[f], deg = desc->degree[f], res = desc->resolution[f];
        const double lo = desc->lo[f], hi = desc->hi[f];
        require(deg >= 0 && deg <= kMaxDegree, FSTK_E_PARAMETER, "basis degree must be in [0, 64]");
        if (fam == 0) {
          require(res == 0, FSTK_E_PARAMETER, "Legendre basis has no resolution parameter");
        } else {
          require(res >= 0 && res <= 20, FSTK_E_PARAMETER, "wavelet resolution must be in [0, 20]");
          require((static_cast<long long>(deg + 1) << res) <= (1 << 24), FSTK_E_PARAMETER,
                  "basis dimension too large");
        }
        require(lo < hi, FSTK_E_PARAMETER, "basis domain must satisfy lo < hi");
        require(std::isfinite(lo) && std::isfinite(hi), FSTK_E_PARAMETER,
                "basis domain must be finite");
        if (j == 0) {
          mh.lo = lo;
          mh.hi = hi;
        }
        require(lo == mh.lo && hi == mh.hi, FSTK_E_SHAPE,
                "model: inconsistent domains within a mode");
        const int dim = fam == 0 ? deg + 1 : (deg + 1) << res;
        for (uint32_t s = 0; s < desc->nnz[f]; ++s, ++c) {
          require(static_cast<int>(desc->indices[c]) < dim, FSTK_E_SHAPE,
                  "model: coefficient index outside basis dimension");
          if (s > 0 && desc->indices[c] <= desc->indices[c - 1]) mh.sorted = false;
          mh.idx.push_back(desc->indices[c]);
          mh.coef.push_back(desc->coeffs[c]);
        }
        mh.rowptr.push_back(static_cast<int>(mh.idx.size()));
        mh.pmax = std::max(mh.pmax, deg);
        // distinct bases of the mode (mode_values evaluates each once, model.cpp:76-92)
        int sid = -1;
        for (size_t q2 = 0; q2 < mh.spec_family.size(); ++q2)
          if (mh.spec_family[q2] == fam && mh.spec_p[q2] == deg && mh.spec_s[q2] == res)
            sid = static_cast<int>(q2);
        if (sid < 0) {
          sid = static_cast<int>(mh.spec_family.size());
          mh.spec_family.push_back(fam);
          mh.spec_p.push_back(deg);
          mh.spec_s.push_back(res);
        }
        mh.fn_spec.push_back(sid);
        if (fam != 0) mh.general = true;
      }
    }
    DeviceGuard dg(device);
    static std::once_flag once[64];
    std::call_once(once[device & 63], [&] { upload_leg_constants(device); });
    m->num_sms = device_sm_count(device);
    m->d_core.alloc(m->R);
    // CSR tables, all modes concatenated.
    std::vector<int> rowptr;
    std::vector<uint32_t> idx;
    std::vector<double> coef;
    std::vector<size_t> rp_off(d), ix_off(d);
    for (int k = 0; k < d; ++k) {
      rp_off[k] = rowptr.size();
      ix_off[k] = idx.size();
      rowptr.insert(rowptr.end(), m->modes[k].rowptr.begin(), m->modes[k].rowptr.end());
      idx.insert(idx.end(), m->modes[k].idx.begin(), m->modes[k].idx.end());
      coef.insert(coef.end(), m->modes[k].coef.begin(), m->modes[k].coef.end());
    }
    if (idx.empty()) {
      idx.push_back(0);
      coef.push_back(0.0);
    }
    m->d_rowptr.alloc(rowptr.size());
    m->d_idx.alloc(idx.size());
    m->d_coef.alloc(coef.size());
    FSTK_CUDA(cudaMemcpy(m->d_rowptr.p, rowptr.data(), rowptr.size() * 4, cudaMemcpyHostToDevice));
    FSTK_CUDA(cudaMemcpy(m->d_idx.p, idx.data(), idx.size() * 4, cudaMemcpyHostToDevice));
    FSTK_CUDA(cudaMemcpy(m->d_coef.p, coef.data(), coef.size() * 8, cudaMemcpyHostToDevice));
    // Dense coefficient blocks (pmax+1) x ldc per mode, for the dense kernel.
    std::vector<double> dense;
    std::vector<size_t> dense_off(d);
    std::vector<int> jc(d), nch(d);
    for (int k = 0; k < d; ++k) {
      const ModeHost& mh = m->modes[k];
      jc[k] = static_cast<int>(std::min<int64_t>(round_up(mh.r, 8), 64));
      nch[k] = static_cast<int>(ceil_div(mh.r, jc[k]));
      const int ldc = jc[k] * nch[k];
      dense_off[k] = dense.size();
      if (mh.general) continue;  // wavelet modes use mode_general_kernel
      dense.resize(dense.size() + static_cast<size_t>(mh.pmax + 1) * ldc, 0.0);
      double* blk = dense.data() + dense_off[k];
      for (int j = 0; j < mh.r; ++j)
        for (int s2 = mh.rowptr[j]; s2 < mh.rowptr[j + 1]; ++s2)
          blk[static_cast<size_t>(mh.idx[s2]) * ldc + j] = mh.coef[s2];
    }
    if (dense.empty()) dense.push_back(0.0);
    m->d_dense.alloc(dense.size());
    FSTK_CUDA(cudaMemcpy(m->d_dense.p, dense.data(), dense.size() * 8, cudaMemcpyHostToDevice));
    m->h_dense = dense;
    m->modes_dev.d = d;
    for (int k = 0; k < d; ++k) {
      m->modes_dev.m[k].dense = m->d_dense.p + dense_off[k];
      m->modes_dev.m[k].h_dense = m->h_dense.data() + dense_off[k];
      m->modes_dev.m[k].jc = jc[k];
      m->modes_dev.m[k].nchunk = nch[k];
      m->modes_dev.m[k].ldc = jc[k] * nch[k];
    }
    for (int k = 0; k < d; ++k) {
      ModeDev& md = m->modes_dev.m[k];
      const ModeHost& mh = m->modes[k];
      md.lo = mh.lo;
      md.hi = mh.hi;
      md.span = mh.hi - mh.lo;
      md.slack = 1e-12 * md.span;
      md.r = mh.r;
      md.pmax = mh.pmax;
      md.rowptr = m->d_rowptr.p + rp_off[k];
      md.idx = m->d_idx.p + ix_off[k];
      md.coef = m->d_coef.p + ix_off[k];
    }
    // Wavelet-capable modes.
    {
      std::vector<int> fs;
      std::vector<size_t> fs_off(d);
      for (int k = 0; k < d; ++k) {
        fs_off[k] = fs.size();
        fs.insert(fs.end(), m->modes[k].fn_spec.begin(), m->modes[k].fn_spec.end());
      }
      m->d_fn_spec.alloc(std::max<size_t>(fs.size(), 1));
      FSTK_CUDA(cudaMemcpy(m->d_fn_spec.p, fs.data(), fs.size() * 4, cudaMemcpyHostToDevice));
      bool any = false;
      for (int k = 0; k < d; ++k) {
        const ModeHost& mh = m->modes[k];
        GenModeDev& G = m->gen[k];
        G = GenModeDev{};
        if (!mh.general) continue;
        any = true;
        const int nspec = static_cast<int>(mh.spec_family.size());
        require(nspec <= kMaxSpec, FSTK_E_PARAMETER,
                "GPU path: more than 8 distinct bases in one mode");
        G.md = m->modes_dev.m[k];
        G.nspec = nspec;
        G.fn_spec = m->d_fn_spec.p + fs_off[k];
        int voff = 0;
        for (int q2 = 0; q2 < nspec; ++q2) {
          SpecDev& sp = G.sp[q2];
          sp.family = mh.spec_family[q2];
          sp.p = mh.spec_p[q2];
          sp.s = sp.family == 0 ? 0 : mh.spec_s[q2];
          sp.voff = voff;
          const int n1 = sp.p + 1;
          voff += sp.family == 0 ? n1 : 2 * n1 + sp.s * (n1 + 1);
          sp.coords = nullptr;
          if (sp.family != 0) {
            auto mc = mother_coords_device(device, sp.p);
            m->mother_refs.push_back(mc);
            sp.coords = mc->p;
          }
        }
        G.vtot = voff;
        require(static_cast<size_t>(voff) * 64 * sizeof(double) <= 200 * 1024, FSTK_E_PARAMETER,
                "GPU path: wavelet basis too large for the per-point scratch "
                "(needs sum over bases of (p+1)(2+s) <= 400)");
      }
      if (any) upload_wavelet_constants(device);
    }
    plan_layout(m.get());
    // Padded table rows beyond r_k are zero-filled by construction: the mode
    // kernel writes r_k rows; padding rows are cleared once per workspace.
    upload_core(m.get());
    // ~1/8 GB of tables per chunk, but at least 64K points.
    int64_t per_pt = 0;
    for (int k = 0; k < d; ++k) per_pt += m->rp[k];
    // Chunks large enough that the last wave of tiles is a small fraction
    // (>= ~100 tiles per SM), capped near 2 GB of table workspace.
    static const int chunk_log2 = [] {
      const char* e = std::getenv("FSTK_EVAL_CHUNK_LOG2");
      return e ? std::min(24, std::max(16, std::atoi(e))) : 21;
    }();
    m->chunk_points = std::min<int64_t>(int64_t(1) << chunk_log2,
                                        std::max<int64_t>(int64_t(1) << 16,
                                                          (int64_t(1) << 31) / (per_pt * 8)));
    m->chunk_points = round_up(m->chunk_points, 128);
    FSTK_CUDA(cudaEventCreateWithFlags(&m->fork_ev, cudaEventDisableTiming));
    for (auto& ck : m->chunk) {
      FSTK_CUDA(cudaStreamCreateWithFlags(&ck.stream, cudaStreamNonBlocking));
      FSTK_CUDA(cudaEventCreateWithFlags(&ck.done, cudaEventDisableTiming));
      FSTK_CUDA(cudaEventCreateWithFlags(&ck.host_done, cudaEventDisableTiming));
    }
    // The chunk workspaces (up to ~2 GB of tables each) are allocated on the
    // first evaluation (ensure_chunk_workspace): a model used only for
    // mode_values / eval_basis / grids never holds them.
    FSTK_CUDA(cudaDeviceSynchronize());
    *out = m.release();
  });
}

void fstk_gpu_model_destroy(fstk_gpu_model* model) {
  if (!model) return;
  for (auto* r : model->replicas) fstk_gpu_model_destroy(r);
  model->replicas.clear();
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(model->device);
  cudaDeviceSynchronize();
  delete model;
  if (prev >= 0) cudaSetDevice(prev);
}

int32_t fstk_gpu_model_set_core(fstk_gpu_model* m, const double* core, fstk_gpu_error* err) {
  return guarded(err, [&] {
    require(m && core, FSTK_E_PARAMETER, "null argument");
    for (auto* r : m->replicas) rethrow_stage_code(fstk_gpu_model_set_core(r, core, err), err);
    std::lock_guard<std::mutex> lk(m->mu);
    DeviceGuard dg(m->device);
    FSTK_CUDA(cudaDeviceSynchronize());
    m->core.assign(core, core + m->R);
    upload_core(m);
  });
}

int32_t fstk_gpu_model_get_core(const fstk_gpu_model* m, double* core, fstk_gpu_error* err) {
  return guarded(err, [&] {
    require(m && core, FSTK_E_PARAMETER, "null argument");
    std::memcpy(core, m->core.data(), m->core.size() * sizeof(double));
  });
}

int32_t fstk_gpu_evaluate_batch_device(const fstk_gpu_model* m, const double* points, int64_t ld,
                                       int64_t q, int32_t d, double* out, void* stream,
                                       fstk_gpu_error* err) {
  return guarded(err, [&] {
    require(m != nullptr, FSTK_E_PARAMETER, "null model");
    require(d == m->d, FSTK_E_PARAMETER, "points must have one column per mode");
    require(q >= 0 && ld >= q, FSTK_E_PARAMETER, "bad point count or leading dimension");
    if (q == 0) return;
    std::lock_guard<std::mutex> lk(m->mu);
    DeviceGuard dg(m->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    evaluate_device(m, points, ld, q, out, s);
    const int64_t bad = evaluate_device_error(m, q, s);
    if (bad >= 0) {
      std::vector<double> y(d);
      for (int k = 0; k < d; ++k)
        FSTK_CUDA(cudaMemcpy(&y[k], points + k * ld + bad, 8, cudaMemcpyDeviceToHost));
      throw_domain(m, static_cast<int64_t>(bad), y.data());
    }
  });
}

// Host buffers: chunks double-buffered over two streams so the H2D copy of
// chunk i+1 and the D2H copy of chunk i-1 overlap the kernels of chunk i.
// Each chunk records its lowest failing row in its own device slot; one
// read-back at the end reports the globally lowest (deterministic) Domain error.
namespace fstk_gpu {
// Rows [r0, r0 + q) of a column-major points buffer with leading dimension
// ldp, on this model's device (chunked, two streams).  A Domain error reports
// the global row index.
// dst <- src (bytes) on up to 8 host threads (pageable <-> pinned staging).
// Host staging copies run on a persistent pool (up to 8 threads): spawning
// threads per copy cost several milliseconds per C2 evaluation.  A job is a
// list of segments whose concatenation is split into equal byte ranges.
struct CopySeg {
  void* dst;
  const void* src;
  size_t bytes;
};
class CopyPool {
 public:
  explicit CopyPool(int n) : nparts_(n) {
    for (int i = 1; i < n; ++i) std::thread([this, i] { worker(i); }).detach();
  }
  void run(const CopySeg* segs, int nseg) {
    size_t total = 0;
    for (int k = 0; k < nseg; ++k) total += segs[k].bytes;
    if (nparts_ <= 1 || total < (size_t(4) << 20)) {
      for (int k = 0; k < nseg; ++k) std::memcpy(segs[k].dst, segs[k].src, segs[k].bytes);
      return;
    }
    std::lock_guard<std::mutex> one(run_mu_);  // one job at a time
    {
      std::lock_guard<std::mutex> lk(mu_);
      segs_ = segs;
      nseg_ = nseg;
      total_ = total;
      remaining_ = nparts_ - 1;
      ++gen_;
    }
    cv_.notify_all();
    part(segs, nseg, total, 0, nparts_);
    std::unique_lock<std::mutex> lk(mu_);
    done_.wait(lk, [&] { return remaining_ == 0; });
  }

 private:
  static void part(const CopySeg* segs, int nseg, size_t total, int i, int np) {
    size_t lo = total * i / np, hi = total * (i + 1) / np, base = 0;
    for (int k = 0; k < nseg && lo < hi; ++k) {
      const size_t b = segs[k].bytes;
      if (lo < base + b) {
        const size_t off = lo - base, n = std::min(hi, base + b) - lo;
        std::memcpy(static_cast<char*>(segs[k].dst) + off, static_cast<const char*>(segs[k].src) + off, n);
        lo += n;
      }
      base += b;
    }
  }
  void worker(int i) {
    uint64_t seen = 0;
    for (;;) {
      std::unique_lock<std::mutex> lk(mu_);
      cv_.wait(lk, [&] { return gen_ != seen; });
      seen = gen_;
      const CopySeg* segs = segs_;
      const int nseg = nseg_;
      const size_t total = total_;
      lk.unlock();
      part(segs, nseg, total, i, nparts_);
      lk.lock();
      if (--remaining_ == 0) done_.notify_one();
    }
  }
  const int nparts_;
  std::mutex run_mu_, mu_;
  std::condition_variable cv_, done_;
  const CopySeg* segs_ = nullptr;
  int nseg_ = 0;
  size_t total_ = 0;
  int remaining_ = 0;
  uint64_t gen_ = 0;
};
static CopyPool& copy_pool() {
  static CopyPool* p = new CopyPool(
      static_cast<int>(std::max(1u, std::min(8u, std::thread::hardware_concurrency()))));
  return *p;  // leaked: its detached workers live for the process
}
static void host_copy(void* dst, const void* src, size_t bytes) {
  const CopySeg seg{dst, src, bytes};
  copy_pool().run(&seg, 1);
}

static bool is_pinned(const void* p) {
  cudaPointerAttributes a{};
  const bool ok = cudaPointerGetAttributes(&a, p) == cudaSuccess;
  cudaGetLastError();
  return ok && a.type != cudaMemoryTypeUnregistered;
}

static void eval_host_slab(const fstk_gpu_model* m, const double* points, int64_t ldp,
                           int64_t r0, int64_t q, int d, double* out) {
  if (q == 0) return;
  std::lock_guard<std::mutex> lk(m->mu);
  DeviceGuard dg(m->device);
  ensure_chunk_workspace(m);
  const int64_t CH = m->chunk_points;
  // Pageable caller buffers (the reference's Eigen/numpy arrays): stage each
  // chunk through a pinned double buffer, the host copies of chunk c+1 (and
  // the results of c-1) overlapping the GPU work of chunk c.  Pinned buffers
  // go straight to the DMA engines.
  const bool stage = q >= (int64_t(1) << 16) && !(is_pinned(points) && is_pinned(out));
  if (stage)
    for (auto& ck : m->chunk)
      if (!ck.h_stage)
        FSTK_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&ck.h_stage),
                                static_cast<size_t>(d + 1) * CH * sizeof(double),
                                cudaHostAllocDefault));
  // Long pinned slabs ramp their end chunks; the staged (pageable) path is
  // bound by its host copies, where small end chunks measured slower (3.2e8
  // -> 2.8e8 pts/s at C2) while the pinned path gained (3.70e8 -> 3.74e8).
  const std::vector<int64_t> cb = chunk_begins(q, CH, !stage);
  int64_t pend[2] = {-1, -1};  // chunk whose outputs wait in each staging slot
  auto drain = [&](int slot) {
    if (pend[slot] < 0) return;
    Chunk& ck = m->chunk[slot];
    FSTK_CUDA(cudaEventSynchronize(ck.host_done));
    const int64_t b = cb[pend[slot]], nb = cb[pend[slot] + 1] - b;
    host_copy(out + r0 + b, ck.h_stage + static_cast<int64_t>(d) * CH, nb * sizeof(double));
    pend[slot] = -1;
  };
  const int64_t ldt = round_up(CH, 128);
  int64_t toff[kMaxOrder], tot = 0;
  eval_table_offsets(m, ldt, toff, &tot);
  const int64_t nchunks = static_cast<int64_t>(cb.size()) - 1;
  m->chunk_err.ensure(static_cast<size_t>(nchunks));
  FSTK_CUDA(cudaMemsetAsync(m->chunk_err.p, 0xff, nchunks * sizeof(unsigned long long),
                            m->chunk[0].stream));
  FSTK_CUDA(cudaEventRecord(m->chunk[0].done, m->chunk[0].stream));
  FSTK_CUDA(cudaStreamWaitEvent(m->chunk[1].stream, m->chunk[0].done, 0));
  for (int64_t c = 0; c < nchunks; ++c) {
    const int slot = static_cast<int>(c & 1);
    Chunk& ck = m->chunk[slot];
    const int64_t b = cb[c];
    const int64_t nb = cb[c + 1] - b;
    if (stage) {
      drain(slot);  // chunk c-2 is done with this slot: its outputs go to the caller
      CopySeg segs[kMaxOrder];
      for (int k = 0; k < d; ++k)
        segs[k] = {ck.h_stage + static_cast<int64_t>(k) * CH, points + k * ldp + r0 + b,
                   static_cast<size_t>(nb) * sizeof(double)};
      copy_pool().run(segs, d);
      FSTK_CUDA(cudaMemcpyAsync(ck.points.p, ck.h_stage, static_cast<size_t>(d) * CH * sizeof(double),
                                cudaMemcpyHostToDevice, ck.stream));
    } else {
      for (int k = 0; k < d; ++k)
        FSTK_CUDA(cudaMemcpyAsync(ck.points.p + k * CH, points + k * ldp + r0 + b,
                                  nb * sizeof(double), cudaMemcpyHostToDevice, ck.stream));
    }
    launch_mode_tables(m, ck.points.p, CH, nb, round_up(nb, 128), nullptr, ck.tables.p, toff,
                       ldt, false, m->chunk_err.p + c, ck.stream);
    launch_contract(m, ck.tables.p, toff, ldt, nb, ck.out.p, ck.stream, nullptr, nullptr);
    if (stage) {
      FSTK_CUDA(cudaMemcpyAsync(ck.h_stage + static_cast<int64_t>(d) * CH, ck.out.p,
                                nb * sizeof(double), cudaMemcpyDeviceToHost, ck.stream));
      FSTK_CUDA(cudaEventRecord(ck.host_done, ck.stream));
      pend[slot] = c;
    } else {
      FSTK_CUDA(cudaMemcpyAsync(out + r0 + b, ck.out.p, nb * sizeof(double),
                                cudaMemcpyDeviceToHost, ck.stream));
    }
  }
  if (stage) {
    drain(static_cast<int>((nchunks - 2) & 1));
    drain(static_cast<int>((nchunks - 1) & 1));
  }
  FSTK_CUDA(cudaStreamSynchronize(m->chunk[1].stream));
  FSTK_CUDA(cudaStreamSynchronize(m->chunk[0].stream));
  std::vector<unsigned long long> bad(static_cast<size_t>(nchunks));
  FSTK_CUDA(cudaMemcpyAsync(bad.data(), m->chunk_err.p, nchunks * sizeof(unsigned long long),
                            cudaMemcpyDeviceToHost, m->chunk[0].stream));
  FSTK_CUDA(cudaStreamSynchronize(m->chunk[0].stream));
  for (int64_t c = 0; c < nchunks; ++c) {
    if (bad[c] != ULLONG_MAX) {
      const int64_t row = r0 + cb[c] + static_cast<int64_t>(bad[c]);
      std::vector<double> y(d);
      for (int k = 0; k < d; ++k) y[k] = points[k * ldp + row];
      throw_domain(m, row, y.data());
    }
  }
}
}  // namespace fstk_gpu

int32_t fstk_gpu_evaluate_batch(const fstk_gpu_model* m, const double* points, int64_t q,
                                int32_t d, double* out, fstk_gpu_error* err) {
  return guarded(err, [&] {
    require(m != nullptr, FSTK_E_PARAMETER, "null model");
    require(d == m->d, FSTK_E_PARAMETER, "points must have one column per mode");
    require(q >= 0, FSTK_E_PARAMETER, "negative point count");
    if (q == 0) return;
    require(points && out, FSTK_E_PARAMETER, "null buffer");
    if (m->replicas.empty()) {
      eval_host_slab(m, points, q, 0, q, d, out);
      return;
    }
    // One host thread per device: contiguous slabs, concurrently.  Errors
    // are the reference's: the Domain error with the lowest point index wins.
    std::vector<const fstk_gpu_model*> dev{m};
    for (const auto* r : m->replicas) dev.push_back(r);
    const int64_t G = static_cast<int64_t>(dev.size());
    std::vector<Error> errs(dev.size());
    std::vector<char> failed(dev.size(), 0);
    std::vector<std::thread> th;
    for (int64_t g = 0; g < G; ++g) {
      th.emplace_back([&, g] {
        try {
          eval_host_slab(dev[g], points, q, q * g / G, q * (g + 1) / G - q * g / G, d, out);
        } catch (const Error& e) {
          errs[g] = e;
          failed[g] = 1;
        } catch (const std::exception& e) {
          errs[g] = Error{FSTK_E_COMPUTE, e.what()};
          failed[g] = 1;
        }
      });
    }
    for (auto& t : th) t.join();
    int first = -1;
    for (int64_t g = 0; g < G; ++g) {
      if (!failed[g]) continue;
      if (first < 0) first = static_cast<int>(g);
      const bool dom = errs[g].code == FSTK_E_DOMAIN, fdom = errs[first].code == FSTK_E_DOMAIN;
      if (dom && (!fdom || errs[g].index < errs[first].index)) first = static_cast<int>(g);
    }
    if (first >= 0) throw errs[first];
  });
}

int32_t fstk_gpu_evaluate(const fstk_gpu_model* m, const double* y, int32_t d, double* out,
                          fstk_gpu_error* err) {
  if (!m) {
    return guarded(err, [&] { fail(FSTK_E_PARAMETER, "null model"); });
  }
  if (d != m->d) {
    return guarded(err, [&] { fail(FSTK_E_PARAMETER, "evaluation point has wrong dimension"); });
  }
  // A single point is a batch of one, column-major Q=1 (bit-identical to the batch path).
  return fstk_gpu_evaluate_batch(m, y, 1, d, out, err);
}

int32_t fstk_gpu_mode_values(const fstk_gpu_model* m, int32_t mode, const double* x, int64_t n,
                             double* out, fstk_gpu_error* err) {
  return guarded(err, [&] {
    require(m != nullptr, FSTK_E_PARAMETER, "null model");
    require(mode >= 0 && mode < m->d, FSTK_E_PARAMETER, "mode out of range");
    require(n >= 0, FSTK_E_PARAMETER, "negative count");
    if (n == 0) return;
    std::lock_guard<std::mutex> lk(m->mu);
    DeviceGuard dg(m->device);
    const int r = static_cast<int>(m->ranks[mode]);
    DevBuf<double> dx(n), dout(static_cast<size_t>(n) * r);
    DevBuf<unsigned long long> derr(1);
    cudaStream_t s = m->chunk[0].stream;
    FSTK_CUDA(cudaMemsetAsync(derr.p, 0xff, 8, s));
    FSTK_CUDA(cudaMemcpyAsync(dx.p, x, n * 8, cudaMemcpyHostToDevice, s));
    launch_mode_table_one(m, mode, dx.p, n, dout.p, n, true, derr.p, s);
    unsigned long long bad = 0;
    FSTK_CUDA(cudaMemcpyAsync(&bad, derr.p, 8, cudaMemcpyDeviceToHost, s));
    FSTK_CUDA(cudaMemcpyAsync(out, dout.p, static_cast<size_t>(n) * r * 8,
                              cudaMemcpyDeviceToHost, s));
    FSTK_CUDA(cudaStreamSynchronize(s));
    if (bad != ULLONG_MAX) {
      Error e{FSTK_E_DOMAIN, "point outside basis domain"};
      e.index = static_cast<int64_t>(bad);
      e.mode = mode;
      e.value = x[bad];
      throw e;
    }
  });
}

}  // extern "C"
