// TEST INFRASTRUCTURE ONLY.  C entry points over the reference's own
// Eigen-free sources (proj/src/rng.cpp, transforms.cpp, parallel.cpp), which
// oracle/Makefile compiles AS-IS from /root/reference into
// oracle/_ref/libfstk_ref.so.  Used to pin the oracle restatement
// (tests/test_oracle_pins.py) and to generate tests/golden/ fixtures.
#include <complex>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "fstk/error.hpp"
#include "fstk/parallel.hpp"
#include "fstk/rng.hpp"
#include "fstk/transforms.hpp"

namespace {
thread_local std::string g_err;
template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const fstk::Error& e) {
    g_err = e.what();
    return static_cast<int>(e.kind()) + 1;
  }
}
}  // namespace

extern "C" {
const char* ref_last_error() { return g_err.c_str(); }
std::uint64_t ref_mix_seed(std::uint64_t s, std::uint64_t t) { return fstk::mix_seed(s, t); }
std::uint64_t ref_next_pow2(std::uint64_t n) { return fstk::next_pow2(n); }
void ref_u64_stream(std::uint64_t seed, std::uint64_t n, std::uint64_t* out) {
  fstk::Rng r(seed);
  for (std::uint64_t i = 0; i < n; ++i) out[i] = r.next_u64();
}
void ref_sign_stream(std::uint64_t seed, std::uint64_t n, double* out) {
  fstk::Rng r(seed);
  for (std::uint64_t i = 0; i < n; ++i) out[i] = r.sign();
}
int ref_uniform_index_stream(std::uint64_t seed, std::uint64_t bound, std::uint64_t n,
                             std::uint64_t* out) {
  return guarded([&] {
    fstk::Rng r(seed);
    for (std::uint64_t i = 0; i < n; ++i) out[i] = r.uniform_index(bound);
  });
}
void ref_sample_without_replacement(std::uint64_t seed, std::uint64_t n, std::uint64_t k,
                                    std::uint64_t* out) {
  fstk::Rng r(seed);
  const auto v = r.sample_without_replacement(n, k);
  std::memcpy(out, v.data(), v.size() * sizeof(std::uint64_t));
}
// make_plan order (randls.cpp:67-71): all q_pad signs first, then the sample.
void ref_plan_stream(std::uint64_t seed, std::uint64_t q_pad, std::uint64_t s, double* signs,
                     std::uint64_t* rows) {
  fstk::Rng r(seed);
  for (std::uint64_t i = 0; i < q_pad; ++i) signs[i] = r.sign();
  const auto v = r.sample_without_replacement(q_pad, s);
  std::memcpy(rows, v.data(), v.size() * sizeof(std::uint64_t));
}
int ref_fft_pow2(double* x, std::uint64_t n, int inverse) {
  return guarded([&] { fstk::fft_pow2(reinterpret_cast<std::complex<double>*>(x), n, inverse); });
}
int ref_unitary_fft(double* x, std::uint64_t n, int inverse) {
  return guarded([&] { fstk::unitary_fft(reinterpret_cast<std::complex<double>*>(x), n, inverse); });
}
int ref_dct2(double* x, std::uint64_t n) { return guarded([&] { fstk::dct2_orthonormal(x, n); }); }
int ref_wht(double* x, std::uint64_t n) { return guarded([&] { fstk::wht_orthonormal(x, n); }); }
// parallel_for chunking check: records which chunk each index landed in.
void ref_parallel_chunks(std::uint64_t n, int threads, std::uint64_t* begin_of) {
  fstk::set_max_threads(threads);
  fstk::parallel_for(n, [&](std::size_t b, std::size_t e) {
    for (std::size_t i = b; i < e; ++i) begin_of[i] = b;
  });
  fstk::set_max_threads(0);
}
}
