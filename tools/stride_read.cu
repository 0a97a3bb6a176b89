// Probe: DRAM read rate of the sketch's last-pass access pattern.  A batch of
// 256 columns x 2^20 complex (4 GiB); a warp reads, for G adjacent position
// classes, elements t*1024 + lo (16 B each, G*16-byte runs at 16 KB stride),
// 32 loads per lane in flight, as the warp-level last pass would.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/stride_read tools/stride_read.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

template <int G, int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 1) probe(const double2* __restrict__ buf, int ncols, int ysplit,
                                                      double* out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int LPC = 32 / G;            // lanes per class
  const int c = lane / LPC, ap = lane % LPC;
  const int group = warp / G, wg = warp % G;  // G warps cover one column's G classes
  constexpr int NG = WARPS / G;
  const int lo0 = (blockIdx.x % (1024 / G)) * G;
  const int y = blockIdx.x / (1024 / G);
  double acc = 0.0;
  for (int cc = y * NG + group; cc < ncols; cc += ysplit * NG) {
    const double2* src = buf + (size_t)cc * (1 << 20) + lo0 + c + (size_t)((1024 / G) * wg + 32 * ap) * 1024;
    double2 v[32];
#pragma unroll
    for (int b = 0; b < 32; ++b) v[b] = __ldcs(src + (size_t)b * 1024);
#pragma unroll
    for (int b = 0; b < 32; ++b) acc += v[b].x + v[b].y;
  }
  if (acc == 12345.678) out[0] = acc;
}

__global__ void contiguous(const double2* __restrict__ buf, size_t n, double* out) {
  double acc = 0.0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const double2 v = __ldcs(buf + i);
    acc += v.x + v.y;
  }
  if (acc == 12345.678) out[0] = acc;
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
  printf("%-28s %8.3f ms  %7.1f GB/s  (%s)\n", name, ms, bytes / ms * 1e-6, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const int ncols = 256;
  const size_t n = (size_t)ncols << 20;
  double2* buf;
  double* out;
  cudaMalloc(&buf, n * sizeof(double2));
  cudaMalloc(&out, 8);
  cudaMemset(buf, 0, n * sizeof(double2));
  const double bytes = (double)n * 16;
  timeit("contiguous", [&] { contiguous<<<148 * 8, 256>>>(buf, n, out); }, bytes);
  timeit("G=2 (32 B runs) 10 warps y2", [&] { probe<2, 10><<<512 * 2, 320>>>(buf, ncols, 2, out); }, bytes);
  timeit("G=2 (32 B runs) 12 warps y2", [&] { probe<2, 12><<<512 * 2, 384>>>(buf, ncols, 2, out); }, bytes);
  timeit("G=2 (32 B runs) 16 warps y2", [&] { probe<2, 16><<<512 * 2, 512>>>(buf, ncols, 2, out); }, bytes);
  timeit("G=4 (64 B runs) 12 warps y4", [&] { probe<4, 12><<<256 * 4, 384>>>(buf, ncols, 4, out); }, bytes);
  timeit("G=4 (64 B runs) 8 warps y4", [&] { probe<4, 8><<<256 * 4, 256>>>(buf, ncols, 4, out); }, bytes);
  timeit("G=8 (128 B runs) 8 warps y8", [&] { probe<8, 8><<<128 * 8, 256>>>(buf, ncols, 8, out); }, bytes);
  timeit("G=8 (128 B runs) 16 warps y8", [&] { probe<8, 16><<<128 * 8, 512>>>(buf, ncols, 8, out); }, bytes);
  return 0;
}
