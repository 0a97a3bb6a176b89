// CRT helpers shared by the int8 Gram kernels (fstk_gram.cu, fstk_syrk.cu):
// the moduli, Garner's reconstruction of an exact integer sum from residues
// congruent to it, and its power-of-two scaling.  See fstk_gram.cu for the
// scheme (an Ozaki-II-style modular split of A^T A).
#pragma once
#include <cstdint>

namespace fstk_gpu {
namespace {

// Pairwise coprime moduli <= 255 (residues fit int8 in symmetric form).
__host__ __device__ constexpr int kmod(int i) {
  constexpr int t[20] = {255, 254, 253, 251, 247, 241, 239, 233, 229, 227,
                         223, 211, 199, 197, 193, 191, 181, 179, 173, 167};
  return t[i];
}
constexpr int kMaxModuli = 20;
constexpr int cx_inv(int a, int m) {  // a^-1 mod m (gcd(a, m) = 1)
  for (int x = 1; x < m; ++x)
    if ((static_cast<long long>(a) * x) % m == 1) return x;
  return 0;
}
struct CrtTables {
  int pmod[kMaxModuli][kMaxModuli];  // (prod_{l<j} m_l) mod m_i, j < i
  int inv[kMaxModuli];               // (prod_{l<i} m_l)^-1 mod m_i
  int q[kMaxModuli][kMaxModuli];     // pmod[l][i] inv[i] mod m_i (Garner, one reduction per digit)
};
constexpr CrtTables make_crt_tables() {
  CrtTables t{};
  for (int i = 0; i < kMaxModuli; ++i) {
    long long p = 1;  // prod_{l<j} m_l mod m_i, built up over j
    for (int j = 0; j < kMaxModuli; ++j) {
      t.pmod[j][i] = static_cast<int>(p);
      if (j < i) p = (p * kmod(j)) % kmod(i);
    }
    t.inv[i] = i == 0 ? 1 : cx_inv(static_cast<int>(p % kmod(i)), kmod(i));
    for (int j = 0; j < kMaxModuli; ++j)
      t.q[j][i] = static_cast<int>((static_cast<long long>(t.pmod[j][i]) * t.inv[i]) % kmod(i));
  }
  return t;
}
__constant__ CrtTables c_crt = make_crt_tables();

// P_s = prod_{t<s} m_t, and the split of an NM-digit Garner value into two
// halves that are exact in fp64: the smallest s with prod_{s<=t<NM} m_t and
// P_s both below 2^53 (0 = none; then the 128-bit path).
__host__ __device__ constexpr unsigned long long crt_prefix(int s) {
  unsigned long long p = 1;
  for (int t = 0; t < s; ++t) p *= static_cast<unsigned long long>(kmod(t));
  return p;
}
__host__ __device__ constexpr int crt_split(int nm) {
  constexpr unsigned long long lim = 1ull << 53;
  for (int s = 1; s < nm; ++s) {
    unsigned long long q = 1;
    bool ok = true;
    for (int t = s; t < nm; ++t) {
      if (q > lim / static_cast<unsigned long long>(kmod(t))) { ok = false; break; }
      q *= static_cast<unsigned long long>(kmod(t));
    }
    if (ok && q < lim && crt_prefix(s) < lim) return s;
  }
  return 0;
}
static_assert(crt_split(9) > 0 && crt_split(11) > 0 && crt_split(12) > 0, "CRT split");

// 128-bit integer -> double on the magnitude: exact whenever the value is
// representable (both 64-bit halves then carry <= 53 significant bits and the
// fused sum is exact), otherwise within one ulp.
__device__ __forceinline__ double i128_to_double(__int128 v) {
  const bool neg = v < 0;
  const unsigned __int128 u = neg ? static_cast<unsigned __int128>(0) - static_cast<unsigned __int128>(v)
                                  : static_cast<unsigned __int128>(v);
  const double hi = static_cast<double>(static_cast<unsigned long long>(u >> 64));
  const double lo = static_cast<double>(static_cast<unsigned long long>(u));
  const double d = fma(hi, 18446744073709551616.0, lo);
  return neg ? -d : d;
}

// Exact integer from NM values congruent to it modulo m_t (|value| < M/2,
// M = prod m_t), rounded once to fp64.  REDUCED: the inputs are already
// symmetric residues (|r| <= m_t / 2), so the first reduction is skipped --
// same digits either way.  Garner, one reduction per digit: y_t = (r_t inv_t
// - sum_{l<t} y_l q_{l,t}) mod m_t (|.| < 2^19 for residues, 2^31-safe for
// int32 sums after the first % m_t).
template <int NM, bool REDUCED>
__device__ __forceinline__ double crt_value(const int (&r)[NM]) {
  int y[NM];  // symmetric mixed-radix digits
#pragma unroll
  for (int t = 0; t < NM; ++t) {
    const int mt = kmod(t);
    int a = (REDUCED ? r[t] : r[t] % mt) * c_crt.inv[t];
#pragma unroll
    for (int l = 0; l < t; ++l) a -= y[l] * c_crt.q[l][t];
    int v = a % mt;
    if (v < 0) v += mt;
    if (v > mt / 2) v -= mt;
    y[t] = v;
  }
  constexpr int SPLIT = crt_split(NM);
  if constexpr (SPLIT > 0) {
    // V = V_lo + P_s V_hi with both halves and P_s below 2^53 (exact int64
    // Horner, exact doubles); one fma rounds V once: correctly rounded, so
    // exact whenever V is representable, like the 128-bit evaluation.
    long long hi = y[NM - 1];
#pragma unroll
    for (int t = NM - 2; t >= SPLIT; --t) hi = hi * kmod(t) + y[t];
    long long lo = y[SPLIT - 1];
#pragma unroll
    for (int t = SPLIT - 2; t >= 0; --t) lo = lo * kmod(t) + y[t];
    return fma(static_cast<double>(hi), static_cast<double>(crt_prefix(SPLIT)), static_cast<double>(lo));
  } else {
    __int128 acc = y[NM - 1];
#pragma unroll
    for (int t = NM - 2; t >= 0; --t) acc = acc * kmod(t) + y[t];
    return i128_to_double(acc);
  }
}

// v 2^e, correctly rounded (one multiplication by an exact power of two when
// 2^e is a normal double -- the same single rounding ldexp performs).
__device__ __forceinline__ double crt_scale(double v, int e) {
  if (e > -1023 && e < 1024) return v * __longlong_as_double(static_cast<long long>(e + 1023) << 52);
  return ldexp(v, e);
}

}  // namespace
}  // namespace fstk_gpu
