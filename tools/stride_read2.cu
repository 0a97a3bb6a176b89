// Probe 2: the 32-byte-run strided read (sketch last pass) with a large
// shared-memory carve-out (small L1), by load flavour.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/stride_read2 tools/stride_read2.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

template <int MODE>
__device__ __forceinline__ double2 ld(const double2* p) {
  double2 v;
  if (MODE == 0) return __ldcs(p);
  if (MODE == 1) return __ldcg(p);
  if (MODE == 2) {
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
  }
  if (MODE == 3) {
    asm volatile("ld.relaxed.gpu.global.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
  }
  return *p;
}

template <int MODE, int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 1) probe(const double2* __restrict__ buf, int ncols, int ysplit,
                                                      double* out) {
  extern __shared__ double2 sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = lane >> 4, ap = lane & 15;
  const int group = warp >> 1, wg = warp & 1;
  constexpr int NG = WARPS / 2;
  const int lo0 = (blockIdx.x % 512) * 2;
  const int y = blockIdx.x / 512;
  double acc = 0.0;
  if (threadIdx.x == 0) sm[0] = make_double2(0, 0);
  for (int cc = y * NG + group; cc < ncols; cc += ysplit * NG) {
    const double2* src = buf + (size_t)cc * (1 << 20) + lo0 + c + (size_t)(512 * wg + 32 * ap) * 1024;
    if (MODE == 5) {
      // cp.async.cg 16 B into shared memory (bypasses L1 and registers)
      double2* dst = sm + warp * 1056 + lane * 33;
#pragma unroll
      for (int b = 0; b < 32; ++b) {
        const unsigned d = (unsigned)__cvta_generic_to_shared(dst + b);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src + (size_t)b * 1024) : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_all;" ::: "memory");
      __syncwarp();
#pragma unroll
      for (int b = 0; b < 32; ++b) acc += dst[b].x;
    } else if (MODE == 4) {
      // 256-bit loads: a lane takes both classes' elements (one whole sector)
      const double2* s32 = buf + (size_t)cc * (1 << 20) + lo0 + (size_t)(512 * wg + 16 * lane) * 1024;
      unsigned long long q[16][4];
#pragma unroll
      for (int b = 0; b < 16; ++b)
        asm volatile("ld.global.L1::no_allocate.L2::evict_first.v4.b64 {%0,%1,%2,%3}, [%4];"
                     : "=l"(q[b][0]), "=l"(q[b][1]), "=l"(q[b][2]), "=l"(q[b][3])
                     : "l"(s32 + (size_t)b * 1024));
#pragma unroll
      for (int b = 0; b < 16; ++b)
        acc += __longlong_as_double(q[b][0]) + __longlong_as_double(q[b][1]) + __longlong_as_double(q[b][2]) +
               __longlong_as_double(q[b][3]);
    } else {
      double2 v[32];
#pragma unroll
      for (int b = 0; b < 32; ++b) v[b] = ld<MODE>(src + (size_t)b * 1024);
#pragma unroll
      for (int b = 0; b < 32; ++b) acc += v[b].x + v[b].y;
    }
  }
  if (acc == 12345.678) out[0] = acc + sm[0].x;
}

template <class F>
static void timeit(const char* name, F&& f, double bytes) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 2; ++i) f();
  cudaEventRecord(a);
  const int reps = 5;
  for (int i = 0; i < reps; ++i) f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  ms /= reps;
  printf("%-44s %8.3f ms  %7.1f GB/s  (%s)\n", name, ms, bytes / ms * 1e-6, cudaGetErrorString(cudaGetLastError()));
}

template <int MODE>
static void run(const char* name, const double2* buf, double* out, double bytes) {
  for (int smem_kb : {1, 100, 160, 215}) {
    auto k = probe<MODE, 10>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    const size_t sm = MODE == 5 ? std::max<size_t>(smem_kb * 1024, 10 * 1056 * 16) : (size_t)smem_kb * 1024;
    char nm[128];
    snprintf(nm, sizeof nm, "%s smem %zu KB", name, sm / 1024);
    timeit(nm, [&] { k<<<1024, 320, sm>>>(buf, 256, 2, out); }, bytes);
  }
}

int main() {
  const size_t n = (size_t)256 << 20;
  double2* buf;
  double* out;
  cudaMalloc(&buf, n * sizeof(double2));
  cudaMalloc(&out, 8);
  cudaMemset(buf, 0, n * sizeof(double2));
  const double bytes = (double)n * 16;
  run<0>("ld.cs", buf, out, bytes);
  run<1>("ld.cg", buf, out, bytes);
  run<2>("ld.nc.L1::no_allocate", buf, out, bytes);
  run<3>("ld.relaxed.gpu", buf, out, bytes);
  run<4>("ld.v4.b64 (256-bit) no_allocate", buf, out, bytes);
  run<5>("cp.async.cg -> smem", buf, out, bytes);
  return 0;
}
