// fstk B200 library — multi-device core refit behind the C-ABI.
//
// reestimate_core (randls.cpp:360-383) is ONE least-squares problem.  With a
// model created after fstk_gpu_set_devices(n > 1) (a model plus n - 1
// replicas), fstk_gpu_reestimate_core runs it sharded over the n devices in
// this process, so the reference's C++ caller (pipeline.cpp:473) reaches the
// multi-GPU path through the same call:
//  1. every device runs the (bit-identical) host plan and sketches ITS
//     column block of the R design columns + rhs for all S sample rows
//     (fstk_gpu_refit_begin_columns; one host thread per device);
//  2. one all-to-all turns column blocks into row slabs (grouped
//     ncclSend/ncclRecv, or peer copies) -- adopt_rows;
//  3. each device forms its partial A^T A (the int8 tcgen05 SYRK) and A^T b;
//  4. the lower triangles are packed (R(R+1)/2 + R values: 4.3 GB at C2, not
//     the 8.6 GB square) and ONE reduce sums them on the solver device;
//  5. the solver device factors; every refinement step broadcasts x, each
//     device computes its rows' correction A_g^T (b_g - A_g x), and one
//     reduce sums them (R values); escalation re-forms and re-reduces the
//     Gram; the rank question (certify, else streaming TSQR of every slab
//     stacked on the solver, pivoted QR with Eigen's threshold, COD) follows
//     fstk_gpu_refit_solve / dist.refine_distributed step for step, so every
//     decision is taken once.
// Transport: NCCL (dlopen'ed libnccl.so.2, ncclCommInitAll over the
// distinct devices; grouped ncclSend/ncclRecv for the all-to-all, ncclReduce
// and ncclBroadcast) when every device is distinct and NCCL loads, else peer
// copies (cudaMemcpyPeerAsync over NVLink, or plain device copies for
// replicas on one GPU -- how the single-GPU test pool exercises this path).
// $FSTK_MULTI_TRANSPORT=p2p forces the peer-copy transport.
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "fstk_common.cuh"
#include "fstk_internal.h"

namespace fstk_gpu {
namespace {

// ------------------------------------------------------------ kernels ---
// packed[off(j) + i - j] = G[i + j n] for i >= j, off(j) = j n - j (j - 1) / 2.
// (Columns strided over gridDim.y, so any n fits the 65,535 grid limit.)
__global__ void pack_lower_kernel(const double* __restrict__ g, int64_t n, double* __restrict__ packed) {
  for (int64_t j = blockIdx.y; j < n; j += gridDim.y) {
    const int64_t i = j + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) packed[j * n - j * (j - 1) / 2 + (i - j)] = g[i + j * n];
  }
}
__global__ void unpack_lower_kernel(const double* __restrict__ packed, int64_t n, double* __restrict__ g) {
  for (int64_t j = blockIdx.y; j < n; j += gridDim.y) {
    const int64_t i = j + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) g[i + j * n] = packed[j * n - j * (j - 1) / 2 + (i - j)];
  }
}
__global__ void add_kernel(double* __restrict__ y, const double* __restrict__ x, int64_t n) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    y[i] += x[i];
}

void pack_lower(const double* g, int64_t n, double* packed, cudaStream_t s) {
  dim3 grid(static_cast<unsigned>(ceil_div(n, 256)), static_cast<unsigned>(std::min<int64_t>(n, 65535)));
  pack_lower_kernel<<<grid, 256, 0, s>>>(g, n, packed);
  check_launch("pack_lower_kernel");
}
void unpack_lower(const double* packed, int64_t n, double* g, cudaStream_t s) {
  dim3 grid(static_cast<unsigned>(ceil_div(n, 256)), static_cast<unsigned>(std::min<int64_t>(n, 65535)));
  unpack_lower_kernel<<<grid, 256, 0, s>>>(packed, n, g);
  check_launch("unpack_lower_kernel");
}

// ---------------------------------------------------------- transports ---
struct Transport {
  explicit Transport(std::vector<int> devs) : dev(std::move(devs)), streams(dev.size()) {
    for (size_t g = 0; g < dev.size(); ++g) {
      DeviceGuard dg(dev[g]);
      FSTK_CUDA(cudaStreamCreateWithFlags(&streams[g], cudaStreamNonBlocking));
    }
  }
  virtual ~Transport() {
    for (size_t g = 0; g < dev.size(); ++g) {
      DeviceGuard dg(dev[g]);
      cudaStreamDestroy(streams[g]);
    }
  }
  virtual const char* name() const = 0;
  // send[g] holds, in peer order, sc[g][h] elements for peer h; recv[h]
  // receives, in source order, rc[h][g] elements from source g.
  virtual void alltoallv(const std::vector<double*>& send, const std::vector<std::vector<int64_t>>& sc,
                         const std::vector<double*>& recv, const std::vector<std::vector<int64_t>>& rc) = 0;
  // buf[root] = sum_g buf[g] (count elements); other buffers may be clobbered.
  virtual void reduce(const std::vector<double*>& buf, int64_t count, int root) = 0;
  // buf[g] = buf[root] for every g.
  virtual void broadcast(const std::vector<double*>& buf, int64_t count, int root) = 0;
  void sync_all() {
    for (size_t g = 0; g < dev.size(); ++g) {
      DeviceGuard dg(dev[g]);
      FSTK_CUDA(cudaStreamSynchronize(streams[g]));
    }
  }
  std::vector<int> dev;
  std::vector<cudaStream_t> streams;
};

// Peer copies (cudaMemcpyPeerAsync: NVLink between devices, a device copy
// within one).  The reduce streams each peer's buffer into the root in
// chunks and adds it there.
struct P2PTransport : Transport {
  explicit P2PTransport(std::vector<int> devs) : Transport(std::move(devs)) {
    for (size_t a = 0; a < dev.size(); ++a)
      for (size_t b = 0; b < dev.size(); ++b) {
        if (dev[a] == dev[b]) continue;
        int ok = 0;
        cudaDeviceCanAccessPeer(&ok, dev[a], dev[b]);
        if (ok) {
          DeviceGuard dg(dev[a]);
          const cudaError_t e = cudaDeviceEnablePeerAccess(dev[b], 0);
          if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) fail(FSTK_E_COMPUTE, "peer access");
          cudaGetLastError();
        }
      }
  }
  const char* name() const override { return "p2p"; }
  void alltoallv(const std::vector<double*>& send, const std::vector<std::vector<int64_t>>& sc,
                 const std::vector<double*>& recv, const std::vector<std::vector<int64_t>>& rc) override {
    const int G = static_cast<int>(dev.size());
    for (int g = 0; g < G; ++g) {
      int64_t so = 0;
      for (int h = 0; h < G; ++h) {
        int64_t ro = 0;
        for (int s = 0; s < g; ++s) ro += rc[h][s];
        if (sc[g][h] != rc[h][g]) fail(FSTK_E_COMPUTE, "internal: all-to-all count mismatch");
        if (sc[g][h]) {
          DeviceGuard dg(dev[g]);
          FSTK_CUDA(cudaMemcpyPeerAsync(recv[h] + ro, dev[h], send[g] + so, dev[g], sc[g][h] * 8, streams[g]));
        }
        so += sc[g][h];
      }
    }
    sync_all();
  }
  void reduce(const std::vector<double*>& buf, int64_t count, int root) override {
    const int64_t chunk = std::min<int64_t>(count, int64_t(32) << 20);  // 256 MB
    DeviceGuard dg(dev[root]);
    DevBuf<double> tmp(chunk);
    for (size_t g = 0; g < dev.size(); ++g) {
      if (static_cast<int>(g) == root) continue;
      for (int64_t o = 0; o < count; o += chunk) {
        const int64_t c = std::min(chunk, count - o);
        FSTK_CUDA(cudaMemcpyPeerAsync(tmp.p, dev[root], buf[g] + o, dev[g], c * 8, streams[root]));
        add_kernel<<<static_cast<unsigned>(std::min<int64_t>(ceil_div(c, 256), 4096)), 256, 0, streams[root]>>>(
            buf[root] + o, tmp.p, c);
        check_launch("add_kernel");
      }
    }
    FSTK_CUDA(cudaStreamSynchronize(streams[root]));
  }
  void broadcast(const std::vector<double*>& buf, int64_t count, int root) override {
    DeviceGuard dg(dev[root]);
    for (size_t g = 0; g < dev.size(); ++g)
      if (static_cast<int>(g) != root && buf[g] != buf[root])
        FSTK_CUDA(cudaMemcpyPeerAsync(buf[g], dev[g], buf[root], dev[root], count * 8, streams[root]));
    FSTK_CUDA(cudaStreamSynchronize(streams[root]));
  }
};

// NCCL, loaded at run time (single-GPU users never need it).
struct Nccl {
  using Comm = void*;
  int (*CommInitAll)(Comm*, int, const int*) = nullptr;
  int (*CommDestroy)(Comm) = nullptr;
  int (*GroupStart)() = nullptr;
  int (*GroupEnd)() = nullptr;
  int (*Send)(const void*, size_t, int, int, Comm, cudaStream_t) = nullptr;
  int (*Recv)(void*, size_t, int, int, Comm, cudaStream_t) = nullptr;
  int (*Reduce)(const void*, void*, size_t, int, int, int, Comm, cudaStream_t) = nullptr;
  int (*Broadcast)(const void*, void*, size_t, int, int, Comm, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
  static constexpr int kFloat64 = 8, kSum = 0;
  static Nccl* load() {
    static Nccl* lib = [] () -> Nccl* {
      const char* env = std::getenv("FSTK_NCCL_LIB");
      void* h = dlopen(env ? env : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
      if (!h) return nullptr;
      auto* n = new Nccl();
      bool ok = true;
      auto sym = [&](auto& fp, const char* name) {
        fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(h, name));
        ok = ok && fp != nullptr;
      };
      sym(n->CommInitAll, "ncclCommInitAll");
      sym(n->CommDestroy, "ncclCommDestroy");
      sym(n->GroupStart, "ncclGroupStart");
      sym(n->GroupEnd, "ncclGroupEnd");
      sym(n->Send, "ncclSend");
      sym(n->Recv, "ncclRecv");
      sym(n->Reduce, "ncclReduce");
      sym(n->Broadcast, "ncclBroadcast");
      sym(n->GetErrorString, "ncclGetErrorString");
      if (!ok) {
        delete n;
        return nullptr;
      }
      return n;
    }();
    return lib;
  }
  void check(int r, const char* what) const {
    if (r != 0) fail(FSTK_E_COMPUTE, std::string("NCCL ") + what + ": " + GetErrorString(r));
  }
};

struct NcclTransport : Transport {
  NcclTransport(Nccl* lib, std::vector<int> devs) : Transport(std::move(devs)), n(lib), comms(dev.size()) {
    n->check(n->CommInitAll(comms.data(), static_cast<int>(dev.size()), dev.data()), "CommInitAll");
  }
  ~NcclTransport() override {
    for (auto c : comms) n->CommDestroy(c);
  }
  const char* name() const override { return "nccl"; }
  void alltoallv(const std::vector<double*>& send, const std::vector<std::vector<int64_t>>& sc,
                 const std::vector<double*>& recv, const std::vector<std::vector<int64_t>>& rc) override {
    const int G = static_cast<int>(dev.size());
    n->check(n->GroupStart(), "GroupStart");
    for (int g = 0; g < G; ++g) {
      int64_t so = 0, ro = 0;
      for (int h = 0; h < G; ++h) {
        if (sc[g][h]) n->check(n->Send(send[g] + so, sc[g][h], Nccl::kFloat64, h, comms[g], streams[g]), "Send");
        if (rc[g][h]) n->check(n->Recv(recv[g] + ro, rc[g][h], Nccl::kFloat64, h, comms[g], streams[g]), "Recv");
        so += sc[g][h];
        ro += rc[g][h];
      }
    }
    n->check(n->GroupEnd(), "GroupEnd");
    sync_all();
  }
  void reduce(const std::vector<double*>& buf, int64_t count, int root) override {
    n->check(n->GroupStart(), "GroupStart");
    for (size_t g = 0; g < dev.size(); ++g)
      n->check(n->Reduce(buf[g], buf[g], count, Nccl::kFloat64, Nccl::kSum, root, comms[g], streams[g]), "Reduce");
    n->check(n->GroupEnd(), "GroupEnd");
    sync_all();
  }
  void broadcast(const std::vector<double*>& buf, int64_t count, int root) override {
    n->check(n->GroupStart(), "GroupStart");
    for (size_t g = 0; g < dev.size(); ++g)
      n->check(n->Broadcast(buf[g], buf[g], count, Nccl::kFloat64, root, comms[g], streams[g]), "Broadcast");
    n->check(n->GroupEnd(), "GroupEnd");
    sync_all();
  }
  Nccl* n;
  std::vector<Nccl::Comm> comms;
};

std::unique_ptr<Transport> make_transport(const std::vector<int>& devs) {
  const char* e = std::getenv("FSTK_MULTI_TRANSPORT");
  const bool force_p2p = e && std::string(e) == "p2p";
  std::vector<int> sorted = devs;
  std::sort(sorted.begin(), sorted.end());
  const bool distinct = std::adjacent_find(sorted.begin(), sorted.end()) == sorted.end();
  if (!force_p2p && distinct) {
    if (Nccl* n = Nccl::load()) {
      try {
        return std::make_unique<NcclTransport>(n, devs);
      } catch (const Error&) {
        // NCCL present but unusable here (e.g. no P2P topology): peer copies.
      }
    }
  }
  return std::make_unique<P2PTransport>(devs);
}

// Runs f(g) for every device g on its own host thread; rethrows the first
// (lowest-g) error.
void on_all(int G, const std::function<void(int)>& f) {
  std::vector<std::exception_ptr> ex(G);
  std::vector<std::thread> th;
  for (int g = 0; g < G; ++g)
    th.emplace_back([&, g] {
      try {
        f(g);
      } catch (...) {
        ex[g] = std::current_exception();
      }
    });
  for (auto& t : th) t.join();
  for (auto& x : ex)
    if (x) std::rethrow_exception(x);
}

void stage(int32_t c, const fstk_gpu_error& e) {
  if (!c) return;
  Error x{c, e.message};
  x.index = e.index;
  x.mode = e.mode;
  x.value = e.value;
  throw x;
}

double wall_s(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace

int32_t reestimate_core_multi(const fstk_gpu_model* m, const double* points, const double* values,
                              int64_t q, int32_t d, const fstk_sketch_cfg* cfg, double* core_out,
                              fstk_reestimate_info* info, fstk_gpu_error* err) {
  std::vector<const fstk_gpu_model*> models{m};
  for (auto* r : m->replicas) models.push_back(r);
  const int G = static_cast<int>(models.size());
  std::vector<fstk_gpu_refit*> rf(G, nullptr);
  fstk_reestimate_info local{};
  fstk_reestimate_info* inf = info ? info : &local;
  std::memset(inf, 0, sizeof(*inf));
  const int32_t rc = guarded(err, [&] {
    require(core_out, FSTK_E_PARAMETER, "null argument");
    std::vector<int> devs(G);
    for (int g = 0; g < G; ++g) devs[g] = models[g]->device;
    std::vector<fstk_reestimate_info> ginf(G);
    std::vector<fstk_gpu_error> gerr(G);
    // 1. Plan + column-sharded sketch on every device.
    on_all(G, [&](int g) {
      stage(fstk_gpu_refit_begin_columns(models[g], points, values, q, d, cfg, g, G, &rf[g], &ginf[g], &gerr[g]),
            gerr[g]);
    });
    *inf = ginf[0];
    for (int g = 1; g < G; ++g) {
      inf->t_prepare = std::max(inf->t_prepare, ginf[g].t_prepare);
      inf->t_sketch = std::max(inf->t_sketch, ginf[g].t_sketch);
      inf->t_alloc = std::max(inf->t_alloc, ginf[g].t_alloc);
    }
    auto tp = make_transport(devs);
    const int64_t R = refit_order(rf[0]);
    // 2. Column blocks -> row slabs (transform = none generates rows locally).
    auto t0 = std::chrono::steady_clock::now();
    if (refit_awaits_exchange(rf[0])) {
      std::vector<double*> send(G), recv(G);
      std::vector<std::vector<int64_t>> sc(G, std::vector<int64_t>(G)), rcnt(G, std::vector<int64_t>(G));
      for (int g = 0; g < G; ++g)
        stage(fstk_gpu_refit_exchange_layout(rf[g], &send[g], sc[g].data(), &recv[g], rcnt[g].data(), &gerr[g]),
              gerr[g]);
      tp->alltoallv(send, sc, recv, rcnt);
      for (int g = 0; g < G; ++g) stage(fstk_gpu_refit_adopt_rows(rf[g], &gerr[g]), gerr[g]);
    }
    inf->t_exchange = wall_s(t0);
    // 3-4. Partial normal equations, packed, reduced on device 0.
    const int64_t npack = R * (R + 1) / 2 + R;
    std::vector<DevBuf<double>> gram(G), rhs(G), packed(G);
    for (int g = 0; g < G; ++g) {
      DeviceGuard dg(devs[g]);
      gram[g].alloc(static_cast<size_t>(R) * R);
      rhs[g].alloc(R);
      packed[g].alloc(npack);
    }
    auto reduce_system = [&](int level) {
      std::vector<fstk_reestimate_info> li(G);
      on_all(G, [&](int g) {
        if (level < 0)
          stage(fstk_gpu_refit_normal_equations(rf[g], gram[g].p, rhs[g].p, &li[g], &gerr[g]), gerr[g]);
        else
          stage(fstk_gpu_refit_normal_equations_level(rf[g], level, gram[g].p, rhs[g].p, &li[g], &gerr[g]),
                gerr[g]);
        DeviceGuard dg(devs[g]);
        cudaStream_t s = tp->streams[g];
        pack_lower(gram[g].p, R, packed[g].p, s);
        FSTK_CUDA(cudaMemcpyAsync(packed[g].p + R * (R + 1) / 2, rhs[g].p, R * 8, cudaMemcpyDeviceToDevice, s));
        FSTK_CUDA(cudaStreamSynchronize(s));
      });
      double tg = 0.0, ops = 0.0;
      for (int g = 0; g < G; ++g) {
        tg = std::max(tg, li[g].t_gram);
        ops += li[g].gram_int8_ops;
      }
      inf->t_gram += tg;
      inf->gram_int8_ops += ops;
      inf->gram_slices = refit_gram_used(rf[0]);
      const auto tr = std::chrono::steady_clock::now();
      std::vector<double*> pb(G);
      for (int g = 0; g < G; ++g) pb[g] = packed[g].p;
      tp->reduce(pb, npack, 0);
      DeviceGuard dg(devs[0]);
      unpack_lower(packed[0].p, R, gram[0].p, tp->streams[0]);
      FSTK_CUDA(cudaMemcpyAsync(rhs[0].p, packed[0].p + R * (R + 1) / 2, R * 8, cudaMemcpyDeviceToDevice,
                                tp->streams[0]));
      FSTK_CUDA(cudaStreamSynchronize(tp->streams[0]));
      inf->t_reduce += wall_s(tr);
    };
    reduce_system(-1);
    // 5. Solve on device 0 with sharded refinement (fstk_gpu_refit_solve's
    // ladder; dist.refine_distributed's collectives).
    const auto ts = std::chrono::steady_clock::now();
    std::vector<DevBuf<double>> xs(G), sv(G);
    for (int g = 0; g < G; ++g) {
      DeviceGuard dg(devs[g]);
      xs[g].alloc(R);
      sv[g].alloc(R);
    }
    auto factor = [&]() {
      stage(fstk_gpu_refit_factor(rf[0], gram[0].p, rhs[0].p, xs[0].p, inf, &gerr[0]), gerr[0]);
      return refit_is_factored(rf[0]);
    };
    auto escalate_until_factored = [&]() {
      while (true) {
        const int used = refit_gram_used(rf[0]);
        if (used == 0) return false;
        reduce_system(used < kGramUpgradeSlices ? kGramUpgradeSlices : 0);
        if (factor()) return true;
      }
    };
    bool ok = factor();
    if (!ok) ok = escalate_until_factored();
    bool need_qr = !ok;
    int steps = 0;
    std::vector<double*> xb(G), sb(G);
    for (int g = 0; g < G; ++g) {
      xb[g] = xs[g].p;
      sb[g] = sv[g].p;
    }
    double prev = 1e300;
    for (int it = 0; ok && it < 8; ++it) {
      tp->broadcast(xb, R, 0);
      on_all(G, [&](int g) { stage(fstk_gpu_refit_correction(rf[g], xs[g].p, sv[g].p, &gerr[g]), gerr[g]); });
      tp->reduce(sb, R, 0);
      double step = 0.0;
      stage(fstk_gpu_refit_apply(rf[0], sv[0].p, xs[0].p, &step, &gerr[0]), gerr[0]);
      ++steps;
      if (step <= 1e-15) break;
      // converged by extrapolation (see fstk_gpu_refit_solve)
      if (it >= 1 && step < 0.1 * prev && step * (step / prev) <= kDoneFloor) break;
      constexpr double kStallFloor = 1e-11;
      const bool flat = it >= 1 && step > 0.5 * prev;
      if (flat && step <= kStallFloor) break;
      const int used = refit_gram_used(rf[0]);
      const bool slow = used > 0 && it >= 1 && step > kStallFloor && step > 0.1 * prev;
      const bool last = it == 7 && step > kStallFloor;
      if (flat || slow || last) {
        if (used > 0) {
          if (!escalate_until_factored()) {
            need_qr = true;
            break;
          }
          prev = 1e300;
          it = -1;
          continue;
        }
        need_qr = true;  // no contraction on the native Gram
        break;
      }
      prev = step;
    }
    inf->refine_steps = steps;
    if (!need_qr) {
      int32_t cert = 0;
      double ratio = 0.0;
      stage(fstk_gpu_refit_certify(rf[0], gram[0].p, &ratio, &cert, &gerr[0]), gerr[0]);
      inf->sigma_ratio = ratio;
      need_qr = !cert;
    }
    if (need_qr) {
      // Streaming TSQR of every slab, stacked on device 0 in shard order.
      const int64_t n1 = R + 1;
      std::vector<DevBuf<double>> raug(G);
      for (int g = 0; g < G; ++g) {
        DeviceGuard dg(devs[g]);
        raug[g].alloc(static_cast<size_t>(n1) * n1);
      }
      on_all(G, [&](int g) { stage(fstk_gpu_refit_local_qr(rf[g], raug[g].p, &gerr[g]), gerr[g]); });
      DeviceGuard dg(devs[0]);
      DevBuf<double> other(static_cast<size_t>(n1) * n1);
      for (int g = 1; g < G; ++g) {
        FSTK_CUDA(cudaMemcpyPeerAsync(other.p, devs[0], raug[g].p, devs[g], n1 * n1 * 8, tp->streams[0]));
        FSTK_CUDA(cudaStreamSynchronize(tp->streams[0]));
        stage(fstk_gpu_qr_stack(raug[0].p, other.p, n1, devs[0], tp->streams[0], &gerr[0]), gerr[0]);
      }
      FSTK_CUDA(cudaStreamSynchronize(tp->streams[0]));
      stage(fstk_gpu_refit_qr_solve(rf[0], raug[0].p, xs[0].p, inf, &gerr[0]), gerr[0]);
      inf->qr_path = 1;
    } else {
      inf->rank_deficient = 0;
    }
    inf->t_solve = wall_s(ts);
    stage(fstk_gpu_refit_finish(rf[0], xs[0].p, core_out, inf, &gerr[0]), gerr[0]);
    inf->devices = G;
    inf->multi_transport = std::string(tp->name()) == "nccl" ? 1 : 2;
  });
  for (auto* r : rf)
    if (r) fstk_gpu_refit_end(r);
  return rc;
}

}  // namespace fstk_gpu

// Packed normal equations for callers that reduce them themselves (the
// one-process-per-GPU torch.distributed path, dist.py): the lower triangle of
// G (n x n, column-major) and rhs (n) into R(R+1)/2 + R values, and back.
extern "C" int32_t fstk_gpu_pack_normal_equations(const double* gram, const double* rhs, int64_t n, double* packed,
                                                  int32_t unpack, void* stream, fstk_gpu_error* err) {
  using namespace fstk_gpu;
  return guarded(err, [&] {
    require(gram && rhs && packed && n > 0, FSTK_E_PARAMETER, "null argument");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int64_t tri = n * (n + 1) / 2;
    if (unpack) {
      unpack_lower(packed, n, const_cast<double*>(gram), s);
      FSTK_CUDA(cudaMemcpyAsync(const_cast<double*>(rhs), packed + tri, n * 8, cudaMemcpyDeviceToDevice, s));
    } else {
      pack_lower(gram, n, packed, s);
      FSTK_CUDA(cudaMemcpyAsync(packed + tri, rhs, n * 8, cudaMemcpyDeviceToDevice, s));
    }
  });
}
