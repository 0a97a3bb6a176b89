// fstk B200 library — measurement hooks: per-launch event timing and the
// fp64 tensor-core peak probe used as the roofline denominator.
#include <mutex>
#include <vector>

#include "fstk_internal.h"

namespace fstk_gpu {

std::atomic<int> g_prof_on{0};
static std::mutex g_prof_mu;
struct ProfRec {
  int kind;
  cudaEvent_t a, b;
};
static std::vector<ProfRec> g_prof;

void prof_record(int kind, cudaEvent_t a, cudaEvent_t b) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_prof.push_back({kind, a, b});
}

// DMMA throughput probe: 8 independent accumulator chains per warp.
__global__ void __launch_bounds__(512) dmma_peak_kernel(double* out, int iters, double s) {
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  const double a = threadIdx.x * 1e-3 + s, b = 1.0 - threadIdx.x * 1e-4;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) dmma_8x8x4(c[i][0], c[i][1], a, b);
  }
  double r = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) r += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

__global__ void __launch_bounds__(512) dfma_peak_kernel(double* out, int iters, double s) {
  double a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = fma(a[i], s, 1e-9);
  }
  double r = 0.0;
#pragma unroll
  for (int i = 0; i < 16; ++i) r += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

}  // namespace fstk_gpu

using namespace fstk_gpu;

extern "C" {

void fstk_gpu_profile_enable(int32_t enable) { g_prof_on.store(enable ? 1 : 0); }

int32_t fstk_gpu_profile_read(double* ms, uint64_t* launches, fstk_gpu_error* err) {
  return guarded(err, [&] {
    std::vector<ProfRec> recs;
    {
      std::lock_guard<std::mutex> lk(g_prof_mu);
      recs.swap(g_prof);
    }
    for (int k = 0; k < FSTK_PROF_KINDS; ++k) {
      if (ms) ms[k] = 0.0;
      if (launches) launches[k] = 0;
    }
    for (auto& r : recs) {
      FSTK_CUDA(cudaEventSynchronize(r.b));
      float t = 0.f;
      FSTK_CUDA(cudaEventElapsedTime(&t, r.a, r.b));
      if (r.kind >= 0 && r.kind < FSTK_PROF_KINDS) {
        if (ms) ms[r.kind] += t;
        if (launches) launches[r.kind] += 1;
      }
      cudaEventDestroy(r.a);
      cudaEventDestroy(r.b);
    }
  });
}

int32_t fstk_gpu_fp64_peak(int32_t device, double* dmma_tflops, double* dfma_tflops,
                           fstk_gpu_error* err) {
  return guarded(err, [&] {
    DeviceGuard dg(device);
    const int sms = device_sm_count(device);
    const int threads = 512, blocks = sms * 2;
    DevBuf<double> out(static_cast<size_t>(blocks) * threads);
    cudaEvent_t a, b;
    FSTK_CUDA(cudaEventCreate(&a));
    FSTK_CUDA(cudaEventCreate(&b));
    const int iters = 20000;
    double best_mma = 0, best_fma = 0;
    for (int rep = 0; rep < 3; ++rep) {
      dmma_peak_kernel<<<blocks, threads>>>(out.p, 64, 0.5);
      check_launch("dmma_peak_kernel");
      FSTK_CUDA(cudaEventRecord(a));
      dmma_peak_kernel<<<blocks, threads>>>(out.p, iters / 4, 0.5);
      check_launch("dmma_peak_kernel");
      FSTK_CUDA(cudaEventRecord(b));
      FSTK_CUDA(cudaEventSynchronize(b));
      float ms = 0;
      FSTK_CUDA(cudaEventElapsedTime(&ms, a, b));
      const double fl = 2.0 * 256 * 8 * (iters / 4) * double(blocks) * (threads / 32);
      best_mma = std::max(best_mma, fl / (ms * 1e-3) / 1e12);
      FSTK_CUDA(cudaEventRecord(a));
      dfma_peak_kernel<<<blocks, threads>>>(out.p, iters, 0.999);
      check_launch("dfma_peak_kernel");
      FSTK_CUDA(cudaEventRecord(b));
      FSTK_CUDA(cudaEventSynchronize(b));
      FSTK_CUDA(cudaEventElapsedTime(&ms, a, b));
      const double fl2 = 2.0 * 16 * iters * double(blocks) * threads;
      best_fma = std::max(best_fma, fl2 / (ms * 1e-3) / 1e12);
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    if (dmma_tflops) *dmma_tflops = best_mma;
    if (dfma_tflops) *dfma_tflops = best_fma;
  });
}

}  // extern "C"
