#pragma once
// Binding of the reference-shaped C++ API to the sm_100a engine (C ABI in
// include/cvgram_b200.h): per-thread default context, status -> exception
// translation, and the device-backed core/fast.hpp functions.

#include <cstdlib>
#include <memory>
#include <string>
#include <vector>

#include "cvgram/core.hpp"
#include "cvgram_b200.h"

namespace cvgram {

/// The engine could not run (no sm_100 device, CUDA failure, out of memory).
struct device_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

namespace detail {

[[noreturn]] inline void throw_status(int rc, const char* msg) {
  switch (rc) {
    case CVG_E_DIMENSION: throw dimension_error(msg);
    case CVG_E_PARTITION: throw partition_error(msg);
    case CVG_E_SCALABILITY: throw scalability_error(msg);
    case CVG_E_INVALID_ARG: throw std::invalid_argument(msg);
    default: throw device_error(msg);
  }
}

inline void check(int rc, const char* err) {
  if (rc != CVG_OK) throw_status(rc, err);
}

/// One context per thread (contexts are not internally thread-safe), bound to
/// device CVG_DEVICE / LOCAL_RANK / 0 -- or, with CVG_DEVICES="0,1,2,3", to several
/// devices (cvg_context_create_multi): run_all_folds then shards the folds across
/// them with the same results, bit for bit (threading.hpp:8-10's n_threads contract,
/// as GPUs).
class Context {
 public:
  static cvg_context* get() {
    thread_local Context c;
    return c.h_;
  }
  ~Context() {
    if (h_) cvg_context_destroy(h_);
  }

 private:
  Context() {
    char err[512] = {0};
    if (const char* list = std::getenv("CVG_DEVICES")) {
      std::vector<int> ids;
      for (const char* p = list; *p;) {
        char* end = nullptr;
        const long v = std::strtol(p, &end, 10);
        if (end == p) break;
        ids.push_back(static_cast<int>(v));
        p = *end == ',' ? end + 1 : end;
      }
      if (!ids.empty()) {
        check(cvg_context_create_multi(static_cast<int>(ids.size()), ids.data(), &h_, err, sizeof err), err);
        return;
      }
    }
    const char* d = std::getenv("CVG_DEVICE");
    if (!d) d = std::getenv("LOCAL_RANK");
    check(cvg_context_create(d ? std::atoi(d) : 0, &h_, err, sizeof err), err);
  }
  cvg_context* h_ = nullptr;
};

}  // namespace detail

/// Device state kept alive by a GlobalCache (the shifted-basis whole-data Gram).
struct DeviceGlobal {
  cvg_global* h = nullptr;
  const double* x_data = nullptr;  // identity of the DatasetPair it was built from
  Index n = 0, k = 0, m = 0;
  ~DeviceGlobal() {
    if (h) cvg_global_destroy(h);
  }
};

inline std::shared_ptr<DeviceGlobal> make_device_global(const DatasetPair& data) {
  auto g = std::make_shared<DeviceGlobal>();
  char err[512] = {0};
  detail::check(cvg_global_create(detail::Context::get(), CVG_DTYPE_F64, data.x().data(), data.y().data(),
                                  data.n_rows(), data.n_features(), data.n_responses(), &g->h, err, sizeof err),
                err);
  g->x_data = data.x().data();
  g->n = data.n_rows();
  g->k = data.n_features();
  g->m = data.n_responses();
  return g;
}

/// Entry (i,j) of the result is m(i,j) / (left(i) * right(j)) (core.hpp:114-130), on the device.
inline Matrix hadamard_outer_divide(const Matrix& m, const Vector& left, const Vector& right) {
  Matrix out(m.rows(), m.cols());
  char err[512] = {0};
  detail::check(cvg_hadamard_outer_divide(detail::Context::get(), m.data(), m.rows(), m.cols(), left.data(),
                                          left.size(), right.data(), right.size(), out.data(), err, sizeof err),
                err);
  return out;
}

}  // namespace cvgram
