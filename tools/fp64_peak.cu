// Microbenchmark: fp64 DFMA vs DMMA (mma.sync m8n8k4 f64) throughput on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters, double s) {
  double a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = fma(a[i], s, 1e-9);
  }
  double r = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) r += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

__global__ void dmma_kernel(double* out, int iters, double s) {
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = 0; c[i][1] = 0; }
  double av = threadIdx.x * 1e-3 + s, bv = 1.0 - threadIdx.x * 1e-4;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(av), "d"(bv));
  }
  double r = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) r += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

// Mixed: every warp issues DMMA chains and DFMA chains that are independent.
// If the tensor (DMMA) and FMA (DFMA) fp64 paths were separate, the combined
// rate would exceed either alone.
__global__ void mixed_kernel(double* out, int iters, double s, int nf) {
  double c[8][2];
  double a[16];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = 0; c[i][1] = 0; }
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3 + i;
  double av = threadIdx.x * 1e-3 + s, bv = 1.0 - threadIdx.x * 1e-4;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(av), "d"(bv));
    for (int r = 0; r < nf; ++r) {
#pragma unroll
      for (int i = 0; i < 16; ++i) a[i] = fma(a[i], s, 1e-9);
    }
  }
  double r = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) r += c[i][0] + c[i][1];
#pragma unroll
  for (int i = 0; i < 16; ++i) r += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

int main() {
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, sizeof(double) * sms * 8 * 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int threads : {256, 512, 1024}) {
    for (int bps : {1, 2, 4}) {
      int blocks = sms * bps; if (threads * bps > 2048) continue;
      int iters = 20000;
      dfma_kernel<<<blocks, threads>>>(out, 100, 0.999);
      cudaEventRecord(e0);
      dfma_kernel<<<blocks, threads>>>(out, iters, 0.999);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double fl = 2.0 * 16 * iters * (double)blocks * threads;
      printf("DFMA threads=%d blocks=%d : %.2f TFLOP/s\n", threads, blocks, fl / ms / 1e9);
      dmma_kernel<<<blocks, threads>>>(out, 100, 0.5);
      cudaEventRecord(e0);
      dmma_kernel<<<blocks, threads>>>(out, iters / 4, 0.5);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      fl = 2.0 * 256 * 8 * (iters / 4) * (double)blocks * (threads / 32);
      printf("DMMA threads=%d blocks=%d : %.2f TFLOP/s\n", threads, blocks, fl / ms / 1e9);
    }
  }
  for (int nf : {1, 2, 4, 8}) {
    const int threads = 512, blocks = sms * 2, iters = 5000;
    mixed_kernel<<<blocks, threads>>>(out, 50, 0.5, nf);
    cudaEventRecord(e0);
    mixed_kernel<<<blocks, threads>>>(out, iters, 0.5, nf);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double fm = 2.0 * 256 * 8 * iters * (double)blocks * (threads / 32);
    const double ff = 2.0 * 16 * nf * iters * (double)blocks * threads;
    printf("MIXED nf=%d: DMMA %.2f + DFMA %.2f = %.2f TFLOP/s (%.3f ms)\n", nf, fm / ms / 1e9,
           ff / ms / 1e9, (fm + ff) / ms / 1e9, ms);
  }
  cudaError_t err = cudaGetLastError();
  printf("err=%s\n", cudaGetErrorString(err));
  return 0;
}
