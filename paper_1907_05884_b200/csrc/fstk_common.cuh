// Shared device/host helpers for the fstk B200 library (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <chrono>
#include <cstdlib>
#include <mutex>
#include <vector>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>

#include "fstk_gpu.h"

namespace fstk_gpu {

// ------------------------------------------------------------ errors ------
// Host-side exception carrying an fstk ErrorKind (+1 = status code); caught
// at the C-ABI and converted to a status, never thrown across it.
struct Error {
  int code;
  std::string msg;
  int mode = -1;
  int64_t index = -1;
  double value = 0.0;
};

[[noreturn]] inline void fail(int code, const std::string& m) { throw Error{code, m}; }
inline void require(bool c, int code, const char* m) {
  if (!c) fail(code, m);
}

#define FSTK_CUDA(call)                                                       \
  do {                                                                        \
    cudaError_t e_ = (call);                                                  \
    if (e_ != cudaSuccess)                                                    \
      ::fstk_gpu::fail(FSTK_E_COMPUTE, std::string("CUDA: ") + #call + ": " + \
                                           cudaGetErrorString(e_));           \
  } while (0)

extern std::atomic<uint64_t> g_launches;
inline void count_launch(uint64_t n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }
inline void check_launch(const char* what) {
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) fail(FSTK_E_COMPUTE, std::string("launch ") + what + ": " + cudaGetErrorString(e));
}

template <typename F>
int32_t guarded(fstk_gpu_error* err, F&& f) {
  if (err) {
    err->kind = 0;
    err->mode = -1;
    err->index = -1;
    err->value = 0.0;
    err->message[0] = 0;
  }
  try {
    f();
    return FSTK_OK;
  } catch (const Error& e) {
    if (err) {
      err->kind = e.code;
      err->mode = e.mode;
      err->index = e.index;
      err->value = e.value;
      std::snprintf(err->message, sizeof(err->message), "%s", e.msg.c_str());
    }
    return e.code;
  } catch (const std::bad_alloc&) {
    if (err) {
      err->kind = FSTK_E_COMPUTE;
      std::snprintf(err->message, sizeof(err->message), "host allocation failed");
    }
    return FSTK_E_COMPUTE;
  } catch (const std::exception& e) {
    if (err) {
      err->kind = FSTK_E_COMPUTE;
      std::snprintf(err->message, sizeof(err->message), "%s", e.what());
    }
    return FSTK_E_COMPUTE;
  }
}

// Scoped device selection (restores the caller's current device).
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) FSTK_CUDA(cudaSetDevice(dev));
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// ------------------------------------------------ large-block device cache ---
// Refit sessions allocate ~80 GB at C2 (A alone is 68.7 GB) and used to hand
// it back to the driver on close.  Re-mapping that much memory every session
// left some refits' HBM-bound stages (sketch, blocked Cholesky) up to 1.8x
// slower at full SM clocks (tools/refit_clocks.py).  Blocks of >= 256 MB are
// therefore kept per device after release and reused by the next request of
// the same size class (<= 1/8 larger), up to 3/4 of the device's memory
// (least recently released blocks are freed first; C2's ~97 GB session fits).
// A failed cudaMalloc returns cached blocks, oldest first, until the request
// fits; fstk_gpu_trim_device_cache() returns all of them on demand.
//
// Policy (fstk_gpu_set_device_cache, or FSTK_DEVICE_CACHE=0/1/2):
//   0 off: plain cudaMalloc/cudaFree;
//   1 session (default): blocks are cached only while a refit session is
//     open; when the last one ends, every cached block goes back to the
//     driver, so reestimate_core returns holding no idle HBM;
//   2 persistent: blocks stay cached across sessions (repeated refits of the
//     same size, e.g. bench.py) until trimmed.
struct CachedBlock {
  void* p;
  size_t bytes;
  int device;
};
struct DeviceCache {
  std::mutex mu;
  std::vector<CachedBlock> free_blocks;
  size_t cached = 0;
  size_t cached_small = 0;  // of which blocks below kCacheMinBytes
};
inline DeviceCache& device_cache() {
  static DeviceCache* c = new DeviceCache();  // leaked: no teardown-order hazards at exit
  return *c;
}
constexpr size_t kCacheMinBytes = size_t(256) << 20;
inline std::atomic<int>& device_cache_policy() {
  static std::atomic<int> pol{[] {
    const char* e = std::getenv("FSTK_DEVICE_CACHE");
    if (!e || !e[0]) return 1;
    const int v = std::atoi(e);
    return v <= 0 ? 0 : (v >= 2 ? 2 : 1);
  }()};
  return pol;
}
// Open refit sessions (policy 1 keeps released blocks only while > 0).
inline std::atomic<int>& device_cache_sessions() {
  static std::atomic<int> n{0};
  return n;
}
inline bool device_cache_enabled() { return device_cache_policy().load() != 0; }
inline bool device_cache_keeps() {
  const int p = device_cache_policy().load();
  return p == 2 || (p == 1 && device_cache_sessions().load() > 0);
}
// Frees the cached blocks of `device` (all devices when < 0).
inline void device_cache_trim(int device) {
  DeviceCache& c = device_cache();
  std::lock_guard<std::mutex> lk(c.mu);
  int prev = -1;
  cudaGetDevice(&prev);
  for (size_t i = 0; i < c.free_blocks.size();) {
    CachedBlock& b = c.free_blocks[i];
    if (device >= 0 && b.device != device) {
      ++i;
      continue;
    }
    cudaSetDevice(b.device);
    cudaFree(b.p);
    c.cached -= b.bytes;
    if (b.bytes < kCacheMinBytes) c.cached_small -= b.bytes;
    c.free_blocks.erase(c.free_blocks.begin() + i);
  }
  if (prev >= 0) cudaSetDevice(prev);
}
// RAII marker of an open refit session; the last one to close under policy
// 1 returns the session's cached blocks to the driver.
struct DeviceCacheSession {
  DeviceCacheSession() { device_cache_sessions().fetch_add(1); }
  ~DeviceCacheSession() {
    if (device_cache_sessions().fetch_sub(1) == 1 && device_cache_policy().load() == 1)
      device_cache_trim(-1);
  }
  DeviceCacheSession(const DeviceCacheSession&) = delete;
  DeviceCacheSession& operator=(const DeviceCacheSession&) = delete;
};
// Driver-call accounting of the large-block path (FSTK_DEBUG_TIMING prints it).
struct DriverAllocStats {
  std::atomic<uint64_t> mallocs{0}, frees{0}, ns{0};
  std::atomic<uint64_t> small_calls{0}, small_ns{0};  // blocks below the cache's size class
};
inline DriverAllocStats& driver_alloc_stats() {
  static DriverAllocStats st;
  return st;
}
struct DriverCallTimer {
  bool small;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  explicit DriverCallTimer(bool sm = false) : small(sm) {}
  ~DriverCallTimer() {
    (small ? driver_alloc_stats().small_ns : driver_alloc_stats().ns) += static_cast<uint64_t>(
        std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count());
  }
};
// FSTK_DEBUG_TIMING: cumulative driver calls of the large-block path so far.
inline void debug_alloc_report(const char* tag) {
  static const bool on = std::getenv("FSTK_DEBUG_TIMING") != nullptr;
  if (!on) return;
  DriverAllocStats& st = driver_alloc_stats();
  size_t fb = 0, tb = 0;
  cudaMemGetInfo(&fb, &tb);
  std::fprintf(stderr,
               "fstk alloc @%s: cudaMalloc %llu cudaFree %llu driver %.1f ms; small blocks %llu calls %.1f ms; "
               "free %.1f GB\n",
               tag, static_cast<unsigned long long>(st.mallocs.load()),
               static_cast<unsigned long long>(st.frees.load()), st.ns.load() * 1e-6,
               static_cast<unsigned long long>(st.small_calls.load()), st.small_ns.load() * 1e-6, fb * 1e-9);
}
inline cudaError_t timed_malloc(void** p, size_t bytes, bool small = false) {
  DriverCallTimer t(small);
  ++(small ? driver_alloc_stats().small_calls : driver_alloc_stats().mallocs);
  return cudaMalloc(p, bytes);
}
inline void timed_free(void* p, bool small = false) {
  DriverCallTimer t(small);
  ++(small ? driver_alloc_stats().small_calls : driver_alloc_stats().frees);
  cudaFree(p);
}
// Small blocks (below the large-block size class) are cached in power-of-two
// size buckets: a refit makes ~50 of them (scratch, index tables, solver
// workspaces), and their cudaMalloc/cudaFree calls cost 30-100 ms per C2
// refit in the driver -- up to 90 ms for a single cudaFree inside the blocked
// Cholesky (FSTK_DEBUG_TIMING), the cause of its 0.2 -> 0.7 s outliers.
constexpr size_t kSmallCacheCap = size_t(4) << 30;  // cached small blocks per process
inline size_t small_bucket(size_t bytes) {
  size_t b = 256;
  while (b < bytes) b <<= 1;
  return b;
}
inline cudaError_t device_alloc(void** p, size_t bytes, size_t* got) {
  int dev = 0;
  cudaGetDevice(&dev);
  const bool small = bytes < kCacheMinBytes;
  if (small && device_cache_enabled()) bytes = small_bucket(bytes);
  *got = bytes;
  if (device_cache_enabled()) {
    DeviceCache& c = device_cache();
    std::lock_guard<std::mutex> lk(c.mu);
    int best = -1;
    for (size_t i = 0; i < c.free_blocks.size(); ++i) {
      const CachedBlock& b = c.free_blocks[i];
      if (b.device != dev) continue;
      const bool fits = small ? b.bytes == bytes : (b.bytes >= bytes && b.bytes - bytes <= bytes / 8);
      if (fits && (best < 0 || b.bytes < c.free_blocks[best].bytes)) best = static_cast<int>(i);
    }
    if (best >= 0) {
      *p = c.free_blocks[best].p;
      *got = c.free_blocks[best].bytes;
      c.cached -= c.free_blocks[best].bytes;
      if (small) c.cached_small -= c.free_blocks[best].bytes;
      c.free_blocks.erase(c.free_blocks.begin() + best);  // keep release order (oldest first)
      return cudaSuccess;
    }
  }
  if (!small && device_cache_enabled()) {
    // A block beyond the cache's cap (C4's 137 GB sketch) means this
    // session's working set cannot stay cached: return everything now, once,
    // rather than evicting block by block inside the timed stages later.
    size_t fb = 0, tb = 0;
    if (cudaMemGetInfo(&fb, &tb) == cudaSuccess && bytes > tb / 4 * 3) device_cache_trim(dev);
    cudaGetLastError();
  }
  cudaError_t e = timed_malloc(p, bytes, small);
  // Out of memory: return cached blocks of this device to the driver, least
  // recently released first, one at a time until the request fits.
  while (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    bool freed = false;
    {
      DeviceCache& c = device_cache();
      std::lock_guard<std::mutex> lk(c.mu);
      for (size_t i = 0; i < c.free_blocks.size(); ++i) {
        if (c.free_blocks[i].device != dev) continue;
        const bool sm = c.free_blocks[i].bytes < kCacheMinBytes;
        timed_free(c.free_blocks[i].p, sm);
        c.cached -= c.free_blocks[i].bytes;
        if (sm) c.cached_small -= c.free_blocks[i].bytes;
        c.free_blocks.erase(c.free_blocks.begin() + i);
        freed = true;
        break;
      }
    }
    if (!freed) break;
    e = timed_malloc(p, bytes, small);
  }
  return e;
}
// cudaMemGetInfo for sizing decisions: the current device's cached blocks
// count as free (an allocation that needs them trims the cache and retries),
// so cached memory never shrinks a later session's segment or batch sizes.
inline cudaError_t device_mem_info(size_t* free_b, size_t* total_b) {
  const cudaError_t e = cudaMemGetInfo(free_b, total_b);
  if (e != cudaSuccess) return e;
  int dev = 0;
  cudaGetDevice(&dev);
  DeviceCache& c = device_cache();
  std::lock_guard<std::mutex> lk(c.mu);
  for (const CachedBlock& b : c.free_blocks)
    if (b.device == dev) *free_b += b.bytes;
  return e;
}
inline void device_free(void* p, size_t bytes) {
  if (!p) return;
  cudaPointerAttributes at{};
  const bool small = bytes < kCacheMinBytes;
  // Small blocks are cached only in their bucket sizes (allocated while the cache was on).
  const bool cacheable = !small || (bytes & (bytes - 1)) == 0;
  if (cacheable && device_cache_keeps() && cudaPointerGetAttributes(&at, p) == cudaSuccess &&
      at.type == cudaMemoryTypeDevice) {
    int prev = -1;
    cudaGetDevice(&prev);
    if (prev != at.device) cudaSetDevice(at.device);
    size_t cap = kSmallCacheCap;
    if (!small) {
      size_t total = 0, freeb = 0;
      cudaMemGetInfo(&freeb, &total);
      cap = total / 4 * 3;
    }
    DeviceCache& c = device_cache();
    const bool keep = bytes <= cap;
    // cudaFree would have synchronised the device; a cached block must
    // likewise be idle before the next owner's stream touches it.  (Outside
    // the cache's lock: other host threads keep allocating meanwhile.)
    if (keep) cudaDeviceSynchronize();
    std::unique_lock<std::mutex> lk(c.mu);
    if (keep) {
      // Least recently released blocks go first, so the latest session's
      // working set is what stays cached.  Large blocks are capped per
      // device, small ones by their total.
      size_t held = 0;
      for (const CachedBlock& b : c.free_blocks)
        if (small ? b.bytes < kCacheMinBytes : (b.device == at.device && b.bytes >= kCacheMinBytes))
          held += b.bytes;
      for (size_t i = 0; held + bytes > cap && i < c.free_blocks.size();) {
        const CachedBlock& b = c.free_blocks[i];
        const bool same_class = small ? b.bytes < kCacheMinBytes
                                      : (b.device == at.device && b.bytes >= kCacheMinBytes);
        if (!same_class) {
          ++i;
          continue;
        }
        if (b.device != at.device) cudaSetDevice(b.device);
        timed_free(b.p, small);
        if (b.device != at.device) cudaSetDevice(at.device);
        held -= b.bytes;
        c.cached -= b.bytes;
        if (small) c.cached_small -= b.bytes;
        c.free_blocks.erase(c.free_blocks.begin() + i);
      }
      c.free_blocks.push_back({p, bytes, at.device});
      c.cached += bytes;
      if (small) c.cached_small += bytes;
    }
    lk.unlock();
    if (prev >= 0 && prev != at.device) cudaSetDevice(prev);
    if (keep) return;
  }
  cudaGetLastError();
  timed_free(p, small);
}

// RAII device buffer.
template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  size_t bytes = 0;  // of the block actually held (a cached block may be larger)
  DevBuf() = default;
  explicit DevBuf(size_t count) { alloc(count); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n), bytes(o.bytes) { o.p = nullptr; o.n = 0; o.bytes = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) { release(); p = o.p; n = o.n; bytes = o.bytes; o.p = nullptr; o.n = 0; o.bytes = 0; }
    return *this;
  }
  void alloc(size_t count) {
    release();
    if (count == 0) return;
    cudaError_t e = device_alloc(reinterpret_cast<void**>(&p), count * sizeof(T), &bytes);
    if (e != cudaSuccess) {
      p = nullptr;
      cudaGetLastError();
      fail(FSTK_E_COMPUTE, "device allocation of " + std::to_string(count * sizeof(T)) +
                               " bytes failed: " + cudaGetErrorString(e));
    }
    n = count;
  }
  void ensure(size_t count) {
    if (count > n) alloc(count);
  }
  void release() {
    if (p) device_free(p, bytes);
    p = nullptr;
    n = 0;
    bytes = 0;
  }
  ~DevBuf() { release(); }
};

// ------------------------------------------------- exact fp64 arithmetic ---
// The reference is compiled for x86-64 without FMA (proj/CMakeLists.txt,
// Release, no -march); where the product must reproduce its bits, every
// product and sum is rounded separately (no contraction).
__device__ __forceinline__ double xmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double xadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double xsub(double a, double b) { return __dsub_rn(a, b); }
// Correctly rounded a / b for b a small positive integer, given rcp =
// RN(1/b): Markstein's correction q1 = RN(q0 + RN?(a - b q0) * rcp).
__device__ __forceinline__ double xdiv_small(double a, double b, double rcp) {
  const double q0 = __dmul_rn(a, rcp);
  const double r = __fma_rn(-q0, b, a);
  return __fma_rn(r, rcp, q0);
}

// ------------------------------------------------ mbarrier + bulk copy ---
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
// 1-D bulk copy global -> shared (TMA engine, UBLKCP), completion counted in
// bytes on the mbarrier.  bytes % 16 == 0, both addresses 16-byte aligned.
__device__ __forceinline__ void bulk_g2s(void* smem_dst, const void* gsrc, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem_dst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// ---------------------------------------------------------------- DMMA ---
// D(8x8) += A(8x4, row) * B(4x8, col), fp64 tensor-core MMA (SASS DMMA.8x8x4).
// Fragments (lane = 4*g + t): a = A[g][t], b = B[t][g], c0/c1 = C[g][2t], C[g][2t+1].
__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// Optional per-launch event timing (fstk_gpu_profile_enable).
extern std::atomic<int> g_prof_on;
void prof_record(int kind, cudaEvent_t a, cudaEvent_t b);
struct ProfScope {
  int kind;
  cudaStream_t s;
  cudaEvent_t a = nullptr, b = nullptr;
  ProfScope(int k, cudaStream_t st) : kind(k), s(st) {
    if (g_prof_on.load(std::memory_order_relaxed)) {
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a, s);
    }
  }
  ~ProfScope() {
    if (a) {
      cudaEventRecord(b, s);
      prof_record(kind, a, b);
    }
  }
};

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

}  // namespace fstk_gpu
