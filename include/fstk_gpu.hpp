// fstk_gpu.hpp — header-only C++ shim over the C-ABI (fstk_gpu.h) that
// re-exposes the reference's hot-path signatures, so the reference's callers
// (pipeline.cpp:387,415,473,519,558,633,781-784,821; module.cpp:216-223,
// 271-294) switch by changing one call.  Errors come back as exceptions
// carrying the reference ErrorKind (error.hpp:11-19); the caller's own
// fstk::Error can be rebuilt from kind()/what().
//
// flatten() adapts ANY model type with the reference's interface
// (fstk::FunctionalSparseTuckerModel, model.hpp:33-59: order(), ranks(),
// core().data(), modes()[k][j].fit.{basis, coeffs}) without depending on it.
#ifndef FSTK_GPU_HPP_
#define FSTK_GPU_HPP_

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "fstk_gpu.h"

namespace fstk_gpu_shim {

class Error : public std::runtime_error {
 public:
  Error(int32_t status, const fstk_gpu_error& e)
      : std::runtime_error(e.message), status_(status), index_(e.index), mode_(e.mode),
        value_(e.value) {}
  // fstk::ErrorKind value (Parameter = 0 ... Compute = 6).
  int kind() const noexcept { return status_ - 1; }
  int64_t index() const noexcept { return index_; }
  int mode() const noexcept { return mode_; }
  double value() const noexcept { return value_; }

 private:
  int32_t status_;
  int64_t index_;
  int mode_;
  double value_;
};

inline void check(int32_t rc, const fstk_gpu_error& e) {
  if (rc != FSTK_OK) throw Error(rc, e);
}

// Owning flat copy of a model, convertible to fstk_model_desc.
struct FlatModel {
  int32_t d = 0;
  std::vector<int64_t> ranks;
  std::vector<double> core;
  std::vector<int32_t> family, degree, resolution;
  std::vector<double> lo, hi;
  std::vector<uint32_t> nnz, indices;
  std::vector<double> coeffs;

  fstk_model_desc desc() const {
    fstk_model_desc m{};
    m.d = d;
    m.ranks = ranks.data();
    m.core = core.data();
    m.family = family.data();
    m.degree = degree.data();
    m.resolution = resolution.data();
    m.lo = lo.data();
    m.hi = hi.data();
    m.nnz = nnz.data();
    m.indices = indices.data();
    m.coeffs = coeffs.data();
    return m;
  }
};

// RefModel: anything shaped like fstk::FunctionalSparseTuckerModel.
template <class RefModel>
FlatModel flatten(const RefModel& model) {
  FlatModel f;
  f.d = static_cast<int32_t>(model.order());
  for (auto r : model.ranks()) f.ranks.push_back(static_cast<int64_t>(r));
  int64_t total = 1;
  for (auto r : f.ranks) total *= r;
  f.core.assign(model.core().data(), model.core().data() + total);
  for (const auto& mode : model.modes()) {
    for (const auto& fn : mode) {
      const auto& b = fn.fit.basis;
      f.family.push_back(static_cast<int32_t>(b.family));
      f.degree.push_back(static_cast<int32_t>(b.degree));
      f.resolution.push_back(static_cast<int32_t>(b.resolution));
      f.lo.push_back(b.lo);
      f.hi.push_back(b.hi);
      f.nnz.push_back(static_cast<uint32_t>(fn.fit.coeffs.size()));
      for (const auto& ic : fn.fit.coeffs) {
        f.indices.push_back(static_cast<uint32_t>(ic.first));
        f.coeffs.push_back(static_cast<double>(ic.second));
      }
    }
  }
  return f;
}

// Device-resident model (owns an fstk_gpu_model*).
class Model {
 public:
  explicit Model(const fstk_model_desc& desc, int32_t device = 0) {
    fstk_gpu_error e{};
    check(fstk_gpu_model_create(&desc, device, &h_, &e), e);
  }
  template <class RefModel>
  static Model from_reference(const RefModel& m, int32_t device = 0) {
    const FlatModel f = flatten(m);
    return Model(f.desc(), device);
  }
  Model(const Model&) = delete;
  Model& operator=(const Model&) = delete;
  Model(Model&& o) noexcept : h_(o.h_) { o.h_ = nullptr; }
  Model& operator=(Model&& o) noexcept {
    std::swap(h_, o.h_);
    return *this;
  }
  ~Model() { fstk_gpu_model_destroy(h_); }
  fstk_gpu_model* get() const { return h_; }

  // evaluate_batch (model.cpp:208-227): points Q x d column-major.
  void evaluate_batch(const double* points, int64_t q, int32_t d, double* out) const {
    fstk_gpu_error e{};
    check(fstk_gpu_evaluate_batch(h_, points, q, d, out, &e), e);
  }
  std::vector<double> evaluate_batch(const double* points, int64_t q, int32_t d) const {
    std::vector<double> out(static_cast<size_t>(q));
    evaluate_batch(points, q, d, out.data());
    return out;
  }
  // evaluate (model.cpp:195-206).
  double evaluate(const std::vector<double>& y) const {
    double v = 0.0;
    fstk_gpu_error e{};
    check(fstk_gpu_evaluate(h_, y.data(), static_cast<int32_t>(y.size()), &v, &e), e);
    return v;
  }
  // mode_values (model.cpp:71-94) for n coordinates: out n x r_mode column-major.
  void mode_values(int32_t mode, const double* x, int64_t n, double* out) const {
    fstk_gpu_error e{};
    check(fstk_gpu_mode_values(h_, mode, x, n, out, &e), e);
  }
  // with_core (model.cpp:62-69), in place on the device copy.
  void set_core(const double* core) {
    fstk_gpu_error e{};
    check(fstk_gpu_model_set_core(h_, core, &e), e);
  }

 private:
  fstk_gpu_model* h_ = nullptr;
};

// reestimate_core (randls.cpp:360-383): returns the new core (mode-0 fastest);
// the caller builds the new model with with_core(), as the reference does.
inline std::vector<double> reestimate_core(const Model& m, const double* points,
                                           const double* values, int64_t q, int32_t d,
                                           const fstk_sketch_cfg& cfg, int64_t core_size,
                                           fstk_reestimate_info* info = nullptr) {
  std::vector<double> core(static_cast<size_t>(core_size));
  fstk_gpu_error e{};
  check(fstk_gpu_reestimate_core(m.get(), points, values, q, d, &cfg, core.data(), info, &e), e);
  return core;
}

// interpolate_to_grid (ingest.cpp:265-383): points Q x d column-major,
// values Q, the cloud box (nullptr = the points' own), the grid sizes and
// intervals; returns prod(sizes) values, mode-0 fastest (DenseTensor order).
inline std::vector<double> interpolate_to_grid(const double* points, const double* values, int64_t q,
                                               int32_t d, const double* box_lo, const double* box_hi,
                                               const std::vector<int64_t>& sizes,
                                               const std::vector<double>& lo, const std::vector<double>& hi,
                                               int32_t neighbors = 0, double power = 2.0,
                                               fstk_interp_report* report = nullptr, int32_t device = 0) {
  int64_t n = 1;
  for (auto s : sizes) n *= s;
  std::vector<double> out(static_cast<size_t>(n > 0 ? n : 0));
  fstk_gpu_error e{};
  check(fstk_gpu_interpolate_to_grid(points, values, q, d, box_lo, box_hi, sizes.data(), lo.data(), hi.data(),
                                     neighbors, power, out.data(), report, nullptr, device, &e),
        e);
  return out;
}

inline fstk_sketch_cfg default_sketch_config() {  // randls.hpp:15-24 defaults
  fstk_sketch_cfg c{};
  c.seed = 0;
  c.working_subset = uint64_t(1) << 20;
  c.sample_rows = 0;
  c.transform = FSTK_TRANSFORM_DCT;
  c.validation_fraction = 0.05;
  return c;
}

}  // namespace fstk_gpu_shim

#endif  // FSTK_GPU_HPP_
