// extern "C" boundary of the cvgram B200 engine (declared in include/cvgram_b200.h).
//
// Host-side validation runs first, in the reference's order and with its
// messages (fast.hpp:137-141; partition.hpp:21-58; core.hpp:37-45), so the
// error behaviour is identical for every binding (C++ header, Python, FFI).
// Every compute entry point then runs on the device; there is no host path.
#include <algorithm>
#include <cmath>
#include <initializer_list>
#include <cstring>
#include <new>
#include <mutex>
#include <map>
#include <random>
#include <string>
#include <thread>

#include <sys/mman.h>
#include <vector>

#include "../../include/cvgram_b200.h"
#include "engine.cuh"
#include "multi.cuh"

using cvg::Status;

namespace {

int report(const Status& s, char* err, size_t errlen) {
  if (!s.ok() && err && errlen) {
    std::strncpy(err, s.msg.c_str(), errlen - 1);
    err[errlen - 1] = 0;
  }
  return s.code;
}

template <typename F>
int guarded(char* err, size_t errlen, F&& f) {
  try {
    return report(f(), err, errlen);
  } catch (const std::bad_alloc&) {
    return report(Status::Err(CVG_E_OOM, "host allocation failed"), err, errlen);
  } catch (const std::exception& e) {
    return report(Status::Err(CVG_E_INVALID_ARG, e.what()), err, errlen);
  }
}

Status validate_partitioning(const int32_t* labels, int64_t n, int32_t p, std::vector<int64_t>* counts) {
  if (p < 2) return Status::Err(CVG_E_PARTITION, "fold count must be at least 2, got " + std::to_string(p));
  if ((int64_t)p > n)
    return Status::Err(CVG_E_PARTITION,
                       "fold count " + std::to_string(p) + " exceeds sample count " + std::to_string(n));
  std::vector<int64_t> c(p, 0);
  for (int64_t i = 0; i < n; ++i) {
    const int32_t l = labels[i];
    if (l < 1 || l > p)
      return Status::Err(CVG_E_PARTITION, "label " + std::to_string(l) + " at sample " + std::to_string(i + 1) +
                                              " is outside {1.." + std::to_string(p) + "}");
    ++c[l - 1];
  }
  for (int32_t f = 0; f < p; ++f)
    if (!c[f]) return Status::Err(CVG_E_PARTITION, "fold " + std::to_string(f + 1) + " is empty");
  if (counts) *counts = std::move(c);
  return Status::Ok();
}

Status check_scalable(const std::vector<int64_t>& counts, int64_t n) {
  for (size_t f = 0; f < counts.size(); ++f)
    if (n - counts[f] < 2)
      return Status::Err(CVG_E_SCALABILITY, "fold " + std::to_string(f + 1) + " leaves a training partition of " +
                                                std::to_string(n - counts[f]) + " rows; scaling needs at least 2");
  return Status::Ok();
}

bool any_scale(const uint32_t* cfgs, int32_t n) {
  for (int32_t i = 0; i < n; ++i)
    if (cfgs[i] & (CVG_SCALE_X | CVG_SCALE_Y)) return true;
  return false;
}

size_t elt(int dtype) { return dtype == CVG_DTYPE_F32 ? 4 : 8; }

Status d2h(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  if (!dst || !bytes) return Status::Ok();
  return cvg::cuda_status(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s), "device-to-host copy");
}

// Large device -> pageable host copies (the caller's fresh output arrays): the driver's pageable path runs at
// ~10 GB/s and slower still into untouched pages (configs' 84 MB of C7 outputs: 21 ms into np.empty, 4.7 ms into
// pinned memory).  Here the bytes go through two pinned 32 MB staging chunks (the device copy of chunk i
// overlaps the host copy of chunk i - 1) and each chunk is copied out by up to 8 host threads, which also
// spreads the first-touch page faults.  Pinned destinations are copied directly.
Status d2h_large(cvg_context* ctx, void* dst, const void* src, size_t bytes) {
  cudaStream_t st = ctx->stream;
  if (!dst || !bytes) return Status::Ok();
  cudaPointerAttributes pa;
  const bool pinned = cudaPointerGetAttributes(&pa, dst) == cudaSuccess && pa.type == cudaMemoryTypeHost;
  cudaGetLastError();
  constexpr size_t kChunk = size_t(32) << 20;
  if (pinned || bytes <= kChunk / 4)
    return cvg::cuda_status(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st), "device-to-host copy");
  cvg::HostScratch& sc = *ctx->scratch;
  if (!sc.stage) {
    void* p = nullptr;
    Status s = cvg::cuda_status(cudaHostAlloc(&p, 2 * kChunk, cudaHostAllocDefault), "pinned staging");
    if (!s.ok()) return s;
    sc.stage = p;
    for (auto& e : sc.stage_ev)
      if (!(s = cvg::cuda_status(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event")).ok()) return s;
  }
  {  // fresh caller pages fault in 4 KB steps; ask for transparent huge pages over the destination's interior
    const uintptr_t a = (reinterpret_cast<uintptr_t>(dst) + 4095) & ~uintptr_t(4095);
    const uintptr_t b = (reinterpret_cast<uintptr_t>(dst) + bytes) & ~uintptr_t(4095);
    if (b > a) madvise(reinterpret_cast<void*>(a), b - a, MADV_HUGEPAGE);
  }
  const unsigned hw = std::thread::hardware_concurrency();
  const int nthreads = (int)std::max(1u, std::min(8u, hw ? hw : 1u));
  auto host_copy = [&](char* d, const char* s2, size_t len) {
    const size_t per = (len + nthreads - 1) / nthreads;
    std::vector<std::thread> th;
    for (int t = 1; t < nthreads && (size_t)t * per < len; ++t)
      th.emplace_back([=] { std::memcpy(d + t * per, s2 + t * per, std::min(per, len - t * per)); });
    std::memcpy(d, s2, std::min(per, len));
    for (auto& x : th) x.join();
  };
  const size_t nch = (bytes + kChunk - 1) / kChunk;
  char* stage = static_cast<char*>(sc.stage);
  for (size_t i = 0; i <= nch; ++i) {
    if (i < nch) {
      const size_t len = std::min(kChunk, bytes - i * kChunk);
      Status s = cvg::cuda_status(cudaMemcpyAsync(stage + (i & 1) * kChunk, static_cast<const char*>(src) + i * kChunk,
                                                  len, cudaMemcpyDeviceToHost, st), "device-to-host copy");
      if (!s.ok()) return s;
      if (!(s = cvg::cuda_status(cudaEventRecord(sc.stage_ev[i & 1], st), "event record")).ok()) return s;
    }
    if (i >= 1) {  // chunk i - 1 has landed in its staging half: copy it out while chunk i transfers
      const size_t j = i - 1, len = std::min(kChunk, bytes - j * kChunk);
      Status s = cvg::cuda_status(cudaEventSynchronize(sc.stage_ev[j & 1]), "event synchronize");
      if (!s.ok()) return s;
      host_copy(static_cast<char*>(dst) + j * kChunk, stage + (j & 1) * kChunk, len);
    }
  }
  return Status::Ok();
}

template <typename Launch>
Status small_vector_op(cvg_context* ctx, std::initializer_list<std::pair<const double*, int64_t>> ins, double* out,
                       int64_t out_len, Launch&& launch) {
  Status s = cvg::cuda_status(cudaSetDevice(ctx->device), "cudaSetDevice");
  if (!s.ok()) return s;
  std::vector<cvg::DevBuf> bufs(ins.size() + 1);
  std::vector<const double*> dptr;
  size_t i = 0;
  for (auto& in : ins) {
    if (!(s = bufs[i].ensure(sizeof(double) * std::max<int64_t>(in.second, 1))).ok()) return s;
    if (in.second)
      if (!(s = cvg::cuda_status(cudaMemcpyAsync(bufs[i].as<void>(), in.first, sizeof(double) * in.second,
                                                 cudaMemcpyHostToDevice, ctx->stream),
                                 "H2D"))
               .ok())
        return s;
    dptr.push_back(bufs[i].as<double>());
    ++i;
  }
  if (!(s = bufs[i].ensure(sizeof(double) * std::max<int64_t>(out_len, 1))).ok()) return s;
  launch(dptr, bufs[i].as<double>());
  ctx->launches += 1;
  if (!(s = cvg::cuda_status(cudaGetLastError(), "kernel launch")).ok()) return s;
  if (!(s = d2h(out, bufs[i].as<void>(), sizeof(double) * out_len, ctx->stream)).ok()) return s;
  return cvg::cuda_status(cudaStreamSynchronize(ctx->stream), "stream synchronize");
}

// One fold of the baseline engine: training rows t_rows of (d_x, d_y), two
// Gram passes (any shift -> training means; then the exact-mean basis), the
// direct epilogue per configuration.  Device outputs for this fold:
// xtx[c] at xtx + c*cstride_xx, xty likewise; stats [k|m] (may be null).
Status baseline_rows(cvg_context* ctx, int dtype, const void* d_x, const void* d_y, int64_t n, int64_t k, int64_t m,
                     const std::vector<int64_t>& t_rows, const uint32_t* cfgs, int32_t ncfg, double* d_xtx,
                     int64_t cstride_xx, double* d_xty, int64_t cstride_xy, double* d_mx, double* d_my,
                     double* d_sx, double* d_sy, cvg::DevBuf& mean_buf) {
  cvg::Plan pl;
  const int64_t nt = (int64_t)t_rows.size();
  Status s = pl.create(ctx, dtype, std::max<int64_t>(nt, 2), k, m, 1, 0, 1, false);
  if (!s.ok()) return s;
  if (!(s = pl.bind_rows(t_rows.data(), nt, n)).ok()) return s;
  if (!(s = pl.gram(d_x, k, d_y, m, nullptr, nullptr)).ok()) return s;  // pass 1: means
  if (!(s = mean_buf.ensure(sizeof(double) * (k + m))).ok()) return s;
  if (!(s = pl.direct_means(mean_buf.as<double>())).ok()) return s;
  if (!(s = pl.gram(d_x, k, d_y, m, nullptr, mean_buf.as<double>())).ok()) return s;  // pass 2: centered
  for (int32_t c = 0; c < ncfg; ++c) {
    const bool first = c == 0;
    if (!(s = pl.finish_direct(&cfgs[c], 1, d_xtx + c * cstride_xx, d_xty + c * cstride_xy, first ? d_mx : nullptr,
                               first ? d_my : nullptr, first ? d_sx : nullptr, first ? d_sy : nullptr))
             .ok())
      return s;
  }
  return Status::Ok();
}

}  // namespace

extern "C" {

int cvg_version(void) { return 1; }

struct cvg_rng {
  std::mt19937_64 eng;
};

cvg_rng* cvg_rng_create(uint64_t seed) { return new (std::nothrow) cvg_rng{std::mt19937_64(seed)}; }
void cvg_rng_destroy(cvg_rng* rng) { delete rng; }
uint64_t cvg_rng_next(cvg_rng* rng) { return rng->eng(); }
double cvg_uniform01_bits(uint64_t draw) { return static_cast<double>(draw >> 11) * 0x1.0p-53; }
double cvg_rng_uniform01(cvg_rng* rng) { return cvg_uniform01_bits(rng->eng()); }

void cvg_random_dataset_fn(cvg_next_fn next, void* state, int64_t n, int64_t k, int64_t m, double* x, double* y) {
  for (int64_t i = 0; i < n * k; ++i) x[i] = cvg_uniform01_bits(next(state));
  for (int64_t i = 0; i < n * m; ++i) y[i] = cvg_uniform01_bits(next(state));
}

void cvg_random_partitioning_fn(cvg_next_fn next, void* state, int64_t n, int32_t p, int32_t* labels) {
  for (int64_t i = 0; i < n; ++i) labels[i] = 1 + static_cast<int32_t>(i % p);
  for (int64_t i = n - 1; i > 0; --i) {
    const int64_t j = static_cast<int64_t>(next(state) % static_cast<uint64_t>(i + 1));
    std::swap(labels[i], labels[j]);
  }
}

static uint64_t rng_next_tramp(void* st) { return static_cast<cvg_rng*>(st)->eng(); }

void cvg_random_dataset(cvg_rng* rng, int64_t n, int64_t k, int64_t m, double* x, double* y) {
  cvg_random_dataset_fn(rng_next_tramp, rng, n, k, m, x, y);
}

void cvg_random_partitioning(cvg_rng* rng, int64_t n, int32_t p, int32_t* labels) {
  cvg_random_partitioning_fn(rng_next_tramp, rng, n, p, labels);
}

int cvg_context_create(int device, cvg_context** out, char* err, size_t errlen) {
  return guarded(err, errlen, [&]() -> Status {
    if (!out) return Status::Err(CVG_E_INVALID_ARG, "null output pointer");
    *out = nullptr;
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0) {
      cudaGetLastError();
      return Status::Err(CVG_E_CUDA, "no CUDA device available (the cvgram engine has no CPU path)");
    }
    if (device < 0 || device >= count) return Status::Err(CVG_E_CUDA, "device ordinal out of range");
    cudaDeviceProp prop;
    Status s = cvg::cuda_status(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
    if (!s.ok()) return s;
    if (prop.major != 10 || prop.minor != 0)
      return Status::Err(CVG_E_CUDA, std::string("the cvgram engine is built for sm_100a (B200); device is ") +
                                         prop.name + " sm_" + std::to_string(prop.major * 10 + prop.minor));
    s = cvg::cuda_status(cudaSetDevice(device), "cudaSetDevice");
    if (!s.ok()) return s;
    auto* ctx = new cvg_context();
    ctx->device = device;
    s = cvg::cuda_status(cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking), "cudaStreamCreate");
    if (!s.ok()) {
      delete ctx;
      return s;
    }
    ctx->stream = ctx->own_stream;
    *out = ctx;
    return Status::Ok();
  });
}

int cvg_context_create_multi(int n_gpus, const int* dev_ids, cvg_context** out, char* err, size_t errlen) {
  return guarded(err, errlen, [&]() -> Status {
    if (!out) return Status::Err(CVG_E_INVALID_ARG, "null output pointer");
    *out = nullptr;
    if (n_gpus < 1 || !dev_ids) return Status::Err(CVG_E_INVALID_ARG, "need at least one device id");
    cvg_context* ctx = nullptr;
    char e2[256] = {0};
    const int rc = cvg_context_create(dev_ids[0], &ctx, e2, sizeof e2);
    if (rc != CVG_OK) return Status::Err(rc, e2);
    Status s = cvg::multi_init(ctx, dev_ids, n_gpus);
    if (!s.ok()) {
      cvg_context_destroy(ctx);
      return s;
    }
    *out = ctx;
    return Status::Ok();
  });
}

int cvg_context_device_count(const cvg_context* ctx) {
  if (!ctx) return 0;
  return ctx->ranks.empty() ? 1 : (int)ctx->ranks.size();
}

int cvg_context_exchange(const cvg_context* ctx) {
  if (!ctx || ctx->ranks.empty()) return 0;
  return ctx->nccl ? 1 : 2;
}

void cvg_context_destroy(cvg_context* ctx) {
  if (!ctx) return;
  cvg::multi_destroy(ctx);
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  ctx->clear_recs();
  for (cudaEvent_t e : ctx->event_pool) cudaEventDestroy(e);
  if (ctx->copy_stream) cudaStreamSynchronize(ctx->copy_stream);
  for (cudaEvent_t e : ctx->sync_events) cudaEventDestroy(e);
  if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
  if (ctx->aux_stream) {
    cudaStreamSynchronize(ctx->aux_stream);
    cudaStreamDestroy(ctx->aux_stream);
  }
  ctx->scratch.reset();
  if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
  delete ctx;
}

int cvg_context_set_stream(cvg_context* ctx, void* stream) {
  if (!ctx) return CVG_E_INVALID_ARG;
  ctx->stream = stream ? static_cast<cudaStream_t>(stream) : ctx->own_stream;
  return CVG_OK;
}

int64_t cvg_context_launch_count(const cvg_context* ctx) {
  if (!ctx) return 0;
  int64_t n = ctx->launches;
  for (const cvg_context* r : ctx->ranks) n += r->launches;
  return n;
}

int cvg_context_enable_timing(cvg_context* ctx, int enable) {
  if (!ctx) return CVG_E_INVALID_ARG;
  cudaStreamSynchronize(ctx->stream);
  ctx->clear_recs();
  ctx->timing = enable != 0;
  return CVG_OK;
}

int cvg_context_kernel_times(cvg_context* ctx, double* ms, int64_t* launches) {
  if (!ctx) return CVG_E_INVALID_ARG;
  for (int i = 0; i < CVG_KERNEL_CLASSES; ++i) {
    if (ms) ms[i] = 0.0;
    if (launches) launches[i] = 0;
  }
  for (auto& r : ctx->recs) {
    if (cudaEventSynchronize(r.b) != cudaSuccess) return CVG_E_CUDA;
    float t = 0.f;
    if (cudaEventElapsedTime(&t, r.a, r.b) != cudaSuccess) return CVG_E_CUDA;
    if (ms) ms[r.cls] += t;
    if (launches) launches[r.cls] += 1;
  }
  return CVG_OK;
}

int cvg_validate_dataset(const double* x, const double* y, int64_t n, int64_t k, int64_t m, int64_t y_rows,
                         char* err, size_t errlen) {
  return guarded(err, errlen, [&]() -> Status {
    if (n != y_rows) return Status::Err(CVG_E_DIMENSION, "x and y must have the same number of rows");
    if (n < 2) return Status::Err(CVG_E_DIMENSION, "need at least 2 samples");
    if (k < 1 || m < 1) return Status::Err(CVG_E_DIMENSION, "x and y must each have at least one column");
    for (int64_t i = 0; i < n * k; ++i)
      if (!std::isfinite(x[i])) return Status::Err(CVG_E_DIMENSION, "x and y entries must be finite");
    for (int64_t i = 0; i < n * m; ++i)
      if (!std::isfinite(y[i])) return Status::Err(CVG_E_DIMENSION, "x and y entries must be finite");
    return Status::Ok();
  });
}

int cvg_validate_partitioning(const int32_t* labels, int64_t n, int32_t p, char* err, size_t errlen) {
  return guarded(err, errlen, [&]() { return validate_partitioning(labels, n, p, nullptr); });
}

int cvg_check_scalable(const int32_t* labels, int64_t n, int32_t p, char* err, size_t errlen) {
  return guarded(err, errlen, [&]() -> Status {
    std::vector<int64_t> c(p > 0 ? p : 0, 0);
    for (int64_t i = 0; i < n; ++i)
      if (labels[i] >= 1 && labels[i] <= p) ++c[labels[i] - 1];
    return check_scalable(c, n);
  });
}

int cvg_fold_range(int32_t p, int32_t rank, int32_t world, int32_t* begin, int32_t* end) {
  if (world < 1 || rank < 0 || rank >= world || p < 0 || !begin || !end) return CVG_E_INVALID_ARG;
  int32_t lo = 0, hi = world, a = 0, b = p;
  while (hi - lo > 1) {
    const int32_t rmid = lo + (hi - lo) / 2, fmid = a + (b - a) / 2;
    if (rank < rmid) {
      hi = rmid;
      b = fmid;
    } else {
      lo = rmid;
      a = fmid;
    }
  }
  *begin = a;
  *end = b;
  return CVG_OK;
}

int cvg_run_all_folds(cvg_context* ctx, int dtype, const void* x, const void* y, int64_t n, int64_t k, int64_t m,
                      const int32_t* labels, int64_t n_labels, int32_t p, const uint32_t* cfg_masks, int32_t n_cfg,
                      double* xtx, double* xty, double* mean_x, double* mean_y, double* std_x, double* std_y,
                      int64_t* n_train, int64_t* n_val, char* err, size_t errlen) {
  return guarded(err, errlen, [&]() -> Status {
    if (!ctx) return Status::Err(CVG_E_INVALID_ARG, "null context");
    if (dtype != CVG_DTYPE_F64 && dtype != CVG_DTYPE_F32) return Status::Err(CVG_E_INVALID_ARG, "unsupported dtype");
    if (n < 2) return Status::Err(CVG_E_DIMENSION, "need at least 2 samples");
    if (k < 1 || m < 1) return Status::Err(CVG_E_DIMENSION, "x and y must each have at least one column");
    if (n_cfg < 1 || !cfg_masks) return Status::Err(CVG_E_INVALID_ARG, "need at least one configuration");
    for (int32_t c = 0; c < n_cfg; ++c)
      if (cfg_masks[c] > 15u) return Status::Err(CVG_E_INVALID_ARG, "configuration mask outside 0..15");
    // run_all_folds validation order, fast.hpp:137-141
    if (n_labels != n) return Status::Err(CVG_E_DIMENSION, "partitioning length does not match sample count");
    std::vector<int64_t> counts;
    Status s = validate_partitioning(labels, n, p, &counts);
    if (!s.ok()) return s;
    const bool scal = any_scale(cfg_masks, n_cfg);
    if (scal) {
      s = check_scalable(counts, n);
      if (!s.ok()) return s;
    }
    // several devices (cvg_context_create_multi) -- except when every fold is tiny (<= 32 rows, e.g. leave-one-out):
    // one device's small-fold mode forms the fold Grams in the epilogue, a summation order rank plans do not share,
    // so such runs stay on the first device and keep returning one device's bits
    if (!ctx->ranks.empty() && !cvg::Plan::small_fold_mode(dtype, counts)) {
      s = cvg::run_all_folds_multi(ctx, dtype, x, y, n, k, m, labels, p, cfg_masks, n_cfg, counts, scal, xtx, xty,
                                   mean_x, mean_y, std_x, std_y);
      if (!s.ok()) return s;
      for (int32_t f = 0; f < p; ++f) {
        if (n_train) n_train[f] = n - counts[f];
        if (n_val) n_val[f] = counts[f];
      }
      return Status::Ok();
    }
    s = cvg::cuda_status(cudaSetDevice(ctx->device), "cudaSetDevice");
    if (!s.ok()) return s;
    if (!ctx->scratch) ctx->scratch.reset(new cvg::HostScratch());
    cvg::HostScratch& sc = *ctx->scratch;
    cudaStream_t st = ctx->stream;
    const size_t e = elt(dtype);
#define TRY(expr)        \
  do {                   \
    s = (expr);          \
    if (!s.ok()) return s; \
  } while (0)
    TRY(sc.x.ensure(e * n * k));
    TRY(sc.y.ensure(e * n * m));
    TRY(sc.labels.ensure(sizeof(int32_t) * n));
    TRY(cvg::cuda_status(cudaMemcpyAsync(sc.labels.as<void>(), labels, sizeof(int32_t) * n, cudaMemcpyHostToDevice, st),
                         "H2D labels"));
    TRY(sc.plan.create(ctx, dtype, n, k, m, p, 0, p, true));
    TRY(sc.plan.bind_labels(sc.labels.as<int32_t>(), true, scal));
    // shift = row 0 of (x | y), read on the host; x and y stream in by column slabs
    std::vector<double> shift(k + m);
    for (int64_t c = 0; c < k + m; ++c) {
      const void* src = c < k ? x : y;
      const int64_t i = c < k ? c : c - k;
      shift[c] = dtype == CVG_DTYPE_F32 ? (double)static_cast<const float*>(src)[i] : static_cast<const double*>(src)[i];
    }
    TRY(sc.plan.gram_host(x, y, sc.x.as<void>(), sc.y.as<void>(), shift.data()));
    const size_t nxx = (size_t)n_cfg * p * k * k, nxy = (size_t)n_cfg * p * k * m;
    TRY(sc.xtx.ensure(sizeof(double) * nxx));
    TRY(sc.xty.ensure(sizeof(double) * nxy));
    TRY(sc.mx.ensure(sizeof(double) * p * k));
    TRY(sc.my.ensure(sizeof(double) * p * m));
    TRY(sc.sx.ensure(sizeof(double) * p * k));
    TRY(sc.sy.ensure(sizeof(double) * p * m));
    TRY(sc.plan.finish(nullptr, 1, nullptr, cfg_masks, n_cfg, sc.xtx.as<double>(), sc.xty.as<double>(),
                       sc.mx.as<double>(), sc.my.as<double>(), sc.sx.as<double>(), sc.sy.as<double>()));
    TRY(d2h_large(ctx, xtx, sc.xtx.as<void>(), sizeof(double) * nxx));
    TRY(d2h_large(ctx, xty, sc.xty.as<void>(), sizeof(double) * nxy));
    // FoldStats fill rules, core.hpp:95-105: means iff any flag, stds iff that side is scaled.
    for (int32_t c = 0; c < n_cfg; ++c) {
      const uint32_t cf = cfg_masks[c];
      if (cf) {
        if (mean_x) TRY(d2h(mean_x + (size_t)c * p * k, sc.mx.as<void>(), sizeof(double) * p * k, st));
        if (mean_y) TRY(d2h(mean_y + (size_t)c * p * m, sc.my.as<void>(), sizeof(double) * p * m, st));
      }
      if ((cf & CVG_SCALE_X) && std_x) TRY(d2h(std_x + (size_t)c * p * k, sc.sx.as<void>(), sizeof(double) * p * k, st));
      if ((cf & CVG_SCALE_Y) && std_y) TRY(d2h(std_y + (size_t)c * p * m, sc.sy.as<void>(), sizeof(double) * p * m, st));
    }
    TRY(cvg::cuda_status(cudaStreamSynchronize(st), "stream synchronize"));
    for (int32_t f = 0; f < p; ++f) {
      if (n_train) n_train[f] = n - counts[f];
      if (n_val) n_val[f] = counts[f];
    }
#undef TRY
    return Status::Ok();
  });
}

int cvg_run_all_folds_stream(cvg_context* ctx, int dtype, const void* x, const void* y, int64_t n, int64_t k, int64_t m,
                             const int32_t* labels, int64_t n_labels, int32_t p, const uint32_t* cfg_masks,
                             int32_t n_cfg, int32_t batch, cvg_fold_batch_fn fn, void* user, char* err, size_t errlen) {
  return guarded(err, errlen, [&]() -> Status {
    if (!ctx) return Status::Err(CVG_E_INVALID_ARG, "null context");
    if (!fn) return Status::Err(CVG_E_INVALID_ARG, "null fold callback");
    if (batch < 1) return Status::Err(CVG_E_INVALID_ARG, "batch must be at least 1 fold");
    if (dtype != CVG_DTYPE_F64 && dtype != CVG_DTYPE_F32) return Status::Err(CVG_E_INVALID_ARG, "unsupported dtype");
    if (n < 2) return Status::Err(CVG_E_DIMENSION, "need at least 2 samples");
    if (k < 1 || m < 1) return Status::Err(CVG_E_DIMENSION, "x and y must each have at least one column");
    if (n_cfg < 1 || !cfg_masks) return Status::Err(CVG_E_INVALID_ARG, "need at least one configuration");
    for (int32_t c = 0; c < n_cfg; ++c)
      if (cfg_masks[c] > 15u) return Status::Err(CVG_E_INVALID_ARG, "configuration mask outside 0..15");
    if (n_labels != n) return Status::Err(CVG_E_DIMENSION, "partitioning length does not match sample count");
    std::vector<int64_t> counts;
    Status s = validate_partitioning(labels, n, p, &counts);
    if (!s.ok()) return s;
    const bool scal = any_scale(cfg_masks, n_cfg);
    if (scal && !(s = check_scalable(counts, n)).ok()) return s;
    if (!(s = cvg::cuda_status(cudaSetDevice(ctx->device), "cudaSetDevice")).ok()) return s;
    if (!ctx->scratch) ctx->scratch.reset(new cvg::HostScratch());
    cvg::HostScratch& sc = *ctx->scratch;
    cudaStream_t st = ctx->stream;
    const size_t e = elt(dtype);
    if (!(s = sc.x.ensure(e * n * k)).ok() || !(s = sc.y.ensure(e * n * m)).ok() ||
        !(s = sc.labels.ensure(sizeof(int32_t) * n)).ok())
      return s;
    if (!(s = cvg::cuda_status(cudaMemcpyAsync(sc.labels.as<void>(), labels, sizeof(int32_t) * n,
                                               cudaMemcpyHostToDevice, st),
                               "H2D labels"))
             .ok())
      return s;
    if (!(s = sc.plan.create(ctx, dtype, n, k, m, p, 0, p, true)).ok()) return s;
    if (!(s = sc.plan.bind_labels(sc.labels.as<int32_t>(), true, scal)).ok()) return s;
    std::vector<double> shift(k + m);
    for (int64_t c = 0; c < k + m; ++c) {
      const void* src = c < k ? x : y;
      const int64_t i = c < k ? c : c - k;
      shift[c] = dtype == CVG_DTYPE_F32 ? (double)static_cast<const float*>(src)[i] : static_cast<const double*>(src)[i];
    }
    if (!(s = sc.plan.gram_host(x, y, sc.x.as<void>(), sc.y.as<void>(), shift.data())).ok()) return s;
    // one batch of outputs on the device and in pinned host memory, reused
    const int32_t nb = std::min<int32_t>(batch, p);
    const size_t nxx = (size_t)n_cfg * nb * k * k, nxy = (size_t)n_cfg * nb * k * m;
    cvg::DevBuf dxx, dxy, dvec;
    if (!(s = dxx.ensure(sizeof(double) * nxx)).ok() || !(s = dxy.ensure(sizeof(double) * nxy)).ok() ||
        !(s = dvec.ensure(sizeof(double) * 2 * nb * (k + m))).ok())
      return s;
    struct Pinned {
      void* p = nullptr;
      ~Pinned() {
        if (p) cudaFreeHost(p);
      }
    } host;
    const size_t hbytes = sizeof(double) * (nxx + nxy + 2 * (size_t)nb * (k + m)) + 2 * sizeof(int64_t) * nb;
    if (!(s = cvg::cuda_status(cudaHostAlloc(&host.p, hbytes, cudaHostAllocDefault), "pinned batch buffer")).ok())
      return s;
    double* hxx = static_cast<double*>(host.p);
    double* hxy = hxx + nxx;
    double* hmx = hxy + nxy;
    double* hmy = hmx + (size_t)nb * k;
    double* hsx = hmy + (size_t)nb * m;
    double* hsy = hsx + (size_t)nb * k;
    int64_t* hnt = reinterpret_cast<int64_t*>(hsy + (size_t)nb * m);
    int64_t* hnv = hnt + nb;
    double* dmx = dvec.as<double>();
    double* dmy = dmx + (size_t)nb * k;
    double* dsx = dmy + (size_t)nb * m;
    double* dsy = dsx + (size_t)nb * k;
    for (int32_t lo = 0; lo < p; lo += nb) {
      const int32_t hi = std::min<int32_t>(p, lo + nb), cnt = hi - lo;
      if (!(s = sc.plan.finish(nullptr, 1, nullptr, cfg_masks, n_cfg, dxx.as<double>(), dxy.as<double>(), dmx, dmy,
                               dsx, dsy, lo, hi))
               .ok())
        return s;
      // packed for cnt folds: [n_cfg][cnt][k][k] etc.
      if (!(s = d2h(hxx, dxx.as<void>(), sizeof(double) * n_cfg * cnt * k * k, st)).ok() ||
          !(s = d2h(hxy, dxy.as<void>(), sizeof(double) * n_cfg * cnt * k * m, st)).ok() ||
          !(s = d2h(hmx, dmx, sizeof(double) * cnt * k, st)).ok() || !(s = d2h(hmy, dmy, sizeof(double) * cnt * m, st)).ok() ||
          !(s = d2h(hsx, dsx, sizeof(double) * cnt * k, st)).ok() || !(s = d2h(hsy, dsy, sizeof(double) * cnt * m, st)).ok())
        return s;
      if (!(s = cvg::cuda_status(cudaStreamSynchronize(st), "stream synchronize")).ok()) return s;
      for (int32_t f = 0; f < cnt; ++f) {
        hnt[f] = n - counts[lo + f];
        hnv[f] = counts[lo + f];
      }
      if (fn(lo, hi, hxx, hxy, hmx, hmy, hsx, hsy, hnt, hnv, user)) break;
    }
    return Status::Ok();
  });
}

int cvg_baseline_fold_products(cvg_context* ctx, int dtype, const void* x, const void* y, int64_t n, int64_t k,
                               int64_t m, const int32_t* labels, int64_t n_labels, int32_t p,
                               const uint32_t* cfg_masks, int32_t n_cfg, double* xtx, double* xty, double* mean_x,
                               double* mean_y, double* std_x, double* std_y, int64_t* n_train, int64_t* n_val,
                               char* err, size_t errlen) {
  return guarded(err, errlen, [&]() -> Status {
    if (!ctx) return Status::Err(CVG_E_INVALID_ARG, "null context");
    if (n < 2) return Status::Err(CVG_E_DIMENSION, "need at least 2 samples");
    if (k < 1 || m < 1) return Status::Err(CVG_E_DIMENSION, "x and y must each have at least one column");
    if (n_cfg < 1 || !cfg_masks) return Status::Err(CVG_E_INVALID_ARG, "need at least one configuration");
    for (int32_t c = 0; c < n_cfg; ++c)
      if (cfg_masks[c] > 15u) return Status::Err(CVG_E_INVALID_ARG, "configuration mask outside 0..15");
    // baseline.hpp:82-87
    if (n_labels != n) return Status::Err(CVG_E_DIMENSION, "partitioning length does not match sample count");
    std::vector<int64_t> counts;
    Status s = validate_partitioning(labels, n, p, &counts);
    if (!s.ok()) return s;
    if (any_scale(cfg_masks, n_cfg) && !(s = check_scalable(counts, n)).ok()) return s;
    if (!(s = cvg::cuda_status(cudaSetDevice(ctx->device), "cudaSetDevice")).ok()) return s;
    if (!ctx->scratch) ctx->scratch.reset(new cvg::HostScratch());
    cvg::HostScratch& sc = *ctx->scratch;
    cudaStream_t st = ctx->stream;
    const size_t e = elt(dtype);
    if (!(s = sc.x.ensure(e * n * k)).ok() || !(s = sc.y.ensure(e * n * m)).ok()) return s;
    if (!(s = cvg::cuda_status(cudaMemcpyAsync(sc.x.as<void>(), x, e * n * k, cudaMemcpyHostToDevice, st), "H2D x"))
             .ok() ||
        !(s = cvg::cuda_status(cudaMemcpyAsync(sc.y.as<void>(), y, e * n * m, cudaMemcpyHostToDevice, st), "H2D y"))
             .ok())
      return s;
    const size_t nxx = (size_t)n_cfg * p * k * k, nxy = (size_t)n_cfg * p * k * m;
    if (!(s = sc.xtx.ensure(sizeof(double) * nxx)).ok() || !(s = sc.xty.ensure(sizeof(double) * nxy)).ok() ||
        !(s = sc.mx.ensure(sizeof(double) * p * k)).ok() || !(s = sc.my.ensure(sizeof(double) * p * m)).ok() ||
        !(s = sc.sx.ensure(sizeof(double) * p * k)).ok() || !(s = sc.sy.ensure(sizeof(double) * p * m)).ok())
      return s;
    // per-fold training rows (complement_rows, partition.hpp:71-83): host index bookkeeping
    std::vector<std::vector<int64_t>> t_rows(p);
    for (int32_t f = 0; f < p; ++f) t_rows[f].reserve(n - counts[f]);
    for (int64_t i = 0; i < n; ++i)
      for (int32_t f = 0; f < p; ++f)
        if (labels[i] != f + 1) t_rows[f].push_back(i);
    cvg::DevBuf mean_buf;
    for (int32_t f = 0; f < p; ++f) {
      s = baseline_rows(ctx, dtype, sc.x.as<void>(), sc.y.as<void>(), n, k, m, t_rows[f], cfg_masks, n_cfg,
                        sc.xtx.as<double>() + (size_t)f * k * k, (int64_t)p * k * k,
                        sc.xty.as<double>() + (size_t)f * k * m, (int64_t)p * k * m, sc.mx.as<double>() + f * k,
                        sc.my.as<double>() + f * m, sc.sx.as<double>() + f * k, sc.sy.as<double>() + f * m, mean_buf);
      if (!s.ok()) return s;
    }
    if (!(s = d2h(xtx, sc.xtx.as<void>(), sizeof(double) * nxx, st)).ok()) return s;
    if (!(s = d2h(xty, sc.xty.as<void>(), sizeof(double) * nxy, st)).ok()) return s;
    for (int32_t c = 0; c < n_cfg; ++c) {
      const uint32_t cf = cfg_masks[c];
      if (cf) {
        if (mean_x && !(s = d2h(mean_x + (size_t)c * p * k, sc.mx.as<void>(), sizeof(double) * p * k, st)).ok()) return s;
        if (mean_y && !(s = d2h(mean_y + (size_t)c * p * m, sc.my.as<void>(), sizeof(double) * p * m, st)).ok()) return s;
      }
      if ((cf & CVG_SCALE_X) && std_x &&
          !(s = d2h(std_x + (size_t)c * p * k, sc.sx.as<void>(), sizeof(double) * p * k, st)).ok())
        return s;
      if ((cf & CVG_SCALE_Y) && std_y &&
          !(s = d2h(std_y + (size_t)c * p * m, sc.sy.as<void>(), sizeof(double) * p * m, st)).ok())
        return s;
    }
    if (!(s = cvg::cuda_status(cudaStreamSynchronize(st), "stream synchronize")).ok()) return s;
    for (int32_t f = 0; f < p; ++f) {
      if (n_train) n_train[f] = n - counts[f];
      if (n_val) n_val[f] = counts[f];
    }
    return Status::Ok();
  });
}

int cvg_baseline_single_fold(cvg_context* ctx, int dtype, const void* x, const void* y, int64_t n, int64_t k,
                             int64_t m, const int64_t* v_rows, int64_t n_val, uint32_t cfg, double* xtx_t,
                             double* xty_t, double* mean_x_t, double* mean_y_t, double* std_x_t, double* std_y_t,
                             int64_t* n_train, char* err, size_t errlen) {
  return guarded(err, errlen, [&]() -> Status {
    if (!ctx) return Status::Err(CVG_E_INVALID_ARG, "null context");
    if (cfg > 15u) return Status::Err(CVG_E_INVALID_ARG, "configuration mask outside 0..15");
    for (int64_t i = 0; i < n_val; ++i)
      if (v_rows[i] < 0 || v_rows[i] >= n || (i && v_rows[i] <= v_rows[i - 1]))
        return Status::Err(CVG_E_INVALID_ARG, "v_rows must be ascending row indices in [0, n)");
    std::vector<int64_t> t_rows;  // complement_rows, partition.hpp:71-83
    for (int64_t i = 0, next = 0; i < n; ++i) {
      if (next < n_val && v_rows[next] == i)
        ++next;
      else
        t_rows.push_back(i);
    }
    // baseline.hpp:47-50
    if (n_val == 0 || t_rows.empty())
      return Status::Err(CVG_E_PARTITION, "a fold needs both validation and training rows");
    if ((cfg & (CVG_SCALE_X | CVG_SCALE_Y)) && t_rows.size() < 2)
      return Status::Err(CVG_E_SCALABILITY, "scaling needs at least 2 training rows");
    Status s = cvg::cuda_status(cudaSetDevice(ctx->device), "cudaSetDevice");
    if (!s.ok()) return s;
    const size_t e = elt(dtype);
    cvg::DevBuf dx, dy, oxx, oxy, ost, mean_buf;
    if (!(s = dx.ensure(e * n * k)).ok() || !(s = dy.ensure(e * n * m)).ok() ||
        !(s = oxx.ensure(sizeof(double) * k * k)).ok() || !(s = oxy.ensure(sizeof(double) * k * m)).ok() ||
        !(s = ost.ensure(sizeof(double) * 2 * (k + m))).ok())
      return s;
    cudaStream_t st = ctx->stream;
    if (!(s = cvg::cuda_status(cudaMemcpyAsync(dx.as<void>(), x, e * n * k, cudaMemcpyHostToDevice, st), "H2D x"))
             .ok() ||
        !(s = cvg::cuda_status(cudaMemcpyAsync(dy.as<void>(), y, e * n * m, cudaMemcpyHostToDevice, st), "H2D y"))
             .ok())
      return s;
    double* stv = ost.as<double>();
    const int64_t w = k + m;
    if (!(s = baseline_rows(ctx, dtype, dx.as<void>(), dy.as<void>(), n, k, m, t_rows, &cfg, 1, oxx.as<double>(), 0,
                            oxy.as<double>(), 0, stv, stv + k, stv + w, stv + w + k, mean_buf))
             .ok())
      return s;
    if (!(s = d2h(xtx_t, oxx.as<void>(), sizeof(double) * k * k, st)).ok()) return s;
    if (!(s = d2h(xty_t, oxy.as<void>(), sizeof(double) * k * m, st)).ok()) return s;
    if (cfg & 15u) {
      if (!(s = d2h(mean_x_t, stv, sizeof(double) * k, st)).ok()) return s;
      if (!(s = d2h(mean_y_t, stv + k, sizeof(double) * m, st)).ok()) return s;
    }
    if ((cfg & CVG_SCALE_X) && !(s = d2h(std_x_t, stv + w, sizeof(double) * k, st)).ok()) return s;
    if ((cfg & CVG_SCALE_Y) && !(s = d2h(std_y_t, stv + w + k, sizeof(double) * m, st)).ok()) return s;
    if (n_train) *n_train = (int64_t)t_rows.size();
    return cvg::cuda_status(cudaStreamSynchronize(st), "stream synchronize");
  });
}

int cvg_plan_create(cvg_context* ctx, int dtype, int64_t n, int64_t k, int64_t m, int32_t p, int32_t fold_begin,
                    int32_t fold_end, cvg_plan** out, char* err, size_t errlen) {
  return guarded(err, errlen, [&]() -> Status {
    if (!ctx || !out) return Status::Err(CVG_E_INVALID_ARG, "null argument");
    *out = nullptr;
    auto* pl = new cvg_plan();
    Status s = pl->plan.create(ctx, dtype, n, k, m, p, fold_begin, fold_end, true);
    if (!s.ok()) {
      delete pl;
      return s;
    }
    *out = pl;
    return Status::Ok();
  });
}

int cvg_plan_create_rank(cvg_context* ctx, int dtype, int64_t n, int64_t k, int64_t m, int32_t p, int32_t rank,
                         int32_t world, cvg_plan** out, char* err, size_t errlen) {
  return guarded(err, errlen, [&]() -> Status {
    if (!ctx || !out) return Status::Err(CVG_E_INVALID_ARG, "null argument");
    *out = nullptr;
    auto* pl = new cvg_plan();
    Status s = pl->plan.create_rank(ctx, dtype, n, k, m, p, rank, world);
    if (!s.ok()) {
      delete pl;
      return s;
    }
    *out = pl;
    return Status::Ok();
  });
}

int cvg_plan_assignment(const cvg_plan* plan, int32_t* fold_begin, int32_t* fold_end) {
  if (!plan || !fold_begin || !fold_end) return CVG_E_INVALID_ARG;
  *fold_begin = plan->plan.fold_begin();
  *fold_end = plan->plan.fold_end();
  return CVG_OK;
}

void cvg_plan_destroy(cvg_plan* plan) {
  if (!plan) return;
  cudaStreamSynchronize(plan->plan.ctx()->stream);
  delete plan;
}

int cvg_plan_bind_labels(cvg_plan* plan, const int32_t* d_labels, int require_scalable, char* err, size_t errlen) {
  return guarded(err, errlen, [&]() -> Status {
    if (!plan) return Status::Err(CVG_E_INVALID_ARG, "null plan");
    Status dev = cvg::cuda_status(cudaSetDevice(plan->plan.ctx()->device), "cudaSetDevice");
    if (!dev.ok()) return dev;
    return plan->plan.bind_labels(d_labels, true, require_scalable != 0);
  });
}

int cvg_plan_gram(cvg_plan* plan, const void* d_x, int64_t ldx, const void* d_y, int64_t ldy, const double* shift,
                  char* err, size_t errlen) {
  return guarded(err, errlen, [&]() -> Status {
    if (!plan) return Status::Err(CVG_E_INVALID_ARG, "null plan");
    Status dev = cvg::cuda_status(cudaSetDevice(plan->plan.ctx()->device), "cudaSetDevice");
    if (!dev.ok()) return dev;
    return plan->plan.gram(d_x, ldx, d_y, ldy, shift, nullptr);
  });
}

int cvg_plan_gram_mapped(cvg_plan* plan, const void* d_x, int64_t ldx, const void* d_y, int64_t ldy,
                         const int64_t* d_row_map, int64_t n_compact, const double* shift, char* err, size_t errlen) {
  return guarded(err, errlen, [&]() -> Status {
    if (!plan || !d_row_map) return Status::Err(CVG_E_INVALID_ARG, "null plan or row map");
    Status dev = cvg::cuda_status(cudaSetDevice(plan->plan.ctx()->device), "cudaSetDevice");
    if (!dev.ok()) return dev;
    if (!shift) return Status::Err(CVG_E_INVALID_ARG, "cvg_plan_gram_mapped needs an explicit shift");
    if (n_compact < 0) return Status::Err(CVG_E_INVALID_ARG, "negative compact row count");
    return plan->plan.gram(d_x, ldx, d_y, ldy, shift, nullptr, d_row_map, n_compact);
  });
}

int cvg_plan_partial(cvg_plan* plan, double* d_dst, int64_t* count) {
  if (!plan || !count) return CVG_E_INVALID_ARG;
  *count = plan->plan.partial_count();
  if (!d_dst) return CVG_OK;
  if (cudaSetDevice(plan->plan.ctx()->device) != cudaSuccess) return CVG_E_CUDA;
  const cudaError_t e = cudaMemcpyAsync(d_dst, plan->plan.local(), sizeof(double) * (*count),
                                        cudaMemcpyDeviceToDevice, plan->plan.ctx()->stream);
  return e == cudaSuccess ? CVG_OK : CVG_E_CUDA;
}

int cvg_plan_finish(cvg_plan* plan, const double* d_rank_partials, int32_t n_ranks, const uint32_t* cfg_masks,
                    int32_t n_cfg, double* d_xtx, double* d_xty, double* d_mean_x, double* d_mean_y,
                    double* d_std_x, double* d_std_y, char* err, size_t errlen) {
  return guarded(err, errlen, [&]() -> Status {
    if (!plan) return Status::Err(CVG_E_INVALID_ARG, "null plan");
    Status dev = cvg::cuda_status(cudaSetDevice(plan->plan.ctx()->device), "cudaSetDevice");
    if (!dev.ok()) return dev;
    for (int32_t c = 0; c < n_cfg; ++c)
      if (cfg_masks[c] > 15u) return Status::Err(CVG_E_INVALID_ARG, "configuration mask outside 0..15");
    return plan->plan.finish(d_rank_partials, n_ranks, nullptr, cfg_masks, n_cfg, d_xtx, d_xty, d_mean_x, d_mean_y,
                             d_std_x, d_std_y);
  });
}

int cvg_plan_finish_range(cvg_plan* plan, const double* d_rank_partials, int32_t n_ranks, const uint32_t* cfg_masks,
                          int32_t n_cfg, int32_t fold_lo, int32_t fold_hi, double* d_xtx, double* d_xty,
                          double* d_mean_x, double* d_mean_y, double* d_std_x, double* d_std_y, char* err,
                          size_t errlen) {
  return guarded(err, errlen, [&]() -> Status {
    if (!plan) return Status::Err(CVG_E_INVALID_ARG, "null plan");
    Status dev = cvg::cuda_status(cudaSetDevice(plan->plan.ctx()->device), "cudaSetDevice");
    if (!dev.ok()) return dev;
    for (int32_t c = 0; c < n_cfg; ++c)
      if (cfg_masks[c] > 15u) return Status::Err(CVG_E_INVALID_ARG, "configuration mask outside 0..15");
    const int32_t fb = plan->plan.fold_begin(), fe = plan->plan.fold_end();
    if (fold_lo < fb || fold_hi > fe || fold_lo > fold_hi)
      return Status::Err(CVG_E_INVALID_ARG, "fold range outside the plan's emitted folds");
    return plan->plan.finish(d_rank_partials, n_ranks, nullptr, cfg_masks, n_cfg, d_xtx, d_xty, d_mean_x, d_mean_y,
                             d_std_x, d_std_y, fold_lo - fb, fold_hi - fb);
  });
}

int cvg_plan_fold_counts(const cvg_plan* plan, int64_t* counts) {
  if (!plan || !counts) return CVG_E_INVALID_ARG;
  const auto& c = plan->plan.counts();
  if (c.empty()) return CVG_E_INVALID_ARG;
  std::memcpy(counts, c.data(), sizeof(int64_t) * c.size());
  return CVG_OK;
}

int cvg_global_create(cvg_context* ctx, int dtype, const void* x, const void* y, int64_t n, int64_t k, int64_t m,
                      cvg_global** out, char* err, size_t errlen) {
  return guarded(err, errlen, [&]() -> Status {
    if (!ctx || !out) return Status::Err(CVG_E_INVALID_ARG, "null argument");
    *out = nullptr;
    if (n < 2) return Status::Err(CVG_E_DIMENSION, "need at least 2 samples");
    if (k < 1 || m < 1) return Status::Err(CVG_E_DIMENSION, "x and y must each have at least one column");
    Status s = cvg::cuda_status(cudaSetDevice(ctx->device), "cudaSetDevice");
    if (!s.ok()) return s;
    auto* g = new cvg_global();
    g->ctx = ctx;
    g->dtype = dtype;
    g->n = n;
    g->k = k;
    g->m = m;
    const size_t e = elt(dtype);
    auto fail = [&](Status st) {
      delete g;
      return st;
    };
    if (!(s = g->x.ensure(e * n * k)).ok()) return fail(s);
    if (!(s = g->y.ensure(e * n * m)).ok()) return fail(s);
    s = cvg::cuda_status(cudaMemcpyAsync(g->x.as<void>(), x, e * n * k, cudaMemcpyHostToDevice, ctx->stream), "H2D x");
    if (!s.ok()) return fail(s);
    s = cvg::cuda_status(cudaMemcpyAsync(g->y.as<void>(), y, e * n * m, cudaMemcpyHostToDevice, ctx->stream), "H2D y");
    if (!s.ok()) return fail(s);
    if (!(s = g->all.create(ctx, dtype, n, k, m, 1, 0, 1, false)).ok()) return fail(s);
    std::vector<int64_t> rows(n);
    for (int64_t i = 0; i < n; ++i) rows[i] = i;
    if (!(s = g->all.bind_rows(rows.data(), n)).ok()) return fail(s);
    if (!(s = g->all.gram(g->x.as<void>(), k, g->y.as<void>(), m, nullptr, nullptr)).ok()) return fail(s);
    s = cvg::cuda_status(cudaStreamSynchronize(ctx->stream), "stream synchronize");
    if (!s.ok()) return fail(s);
    *out = g;
    return Status::Ok();
  });
}

void cvg_global_destroy(cvg_global* g) {
  if (!g) return;
  cudaStreamSynchronize(g->ctx->stream);
  delete g;
}

int cvg_global_export(cvg_global* g, uint32_t cfg, double* xtx, double* xty, double* sum_x, double* sum_y,
                      double* mean_x, double* mean_y, double* sum_sq_x, double* sum_sq_y, char* err,
                      size_t errlen) {
  return guarded(err, errlen, [&]() -> Status {
    if (!g) return Status::Err(CVG_E_INVALID_ARG, "null global");
    if (cudaSetDevice(g->ctx->device) != cudaSuccess) return Status::Err(CVG_E_CUDA, "cudaSetDevice failed");
    const int64_t k = g->k, m = g->m, w = k + m;
    cudaStream_t st = g->ctx->stream;
    Status s;
    if (!(s = g->out_xtx.ensure(sizeof(double) * k * k)).ok()) return s;
    if (!(s = g->out_xty.ensure(sizeof(double) * k * m)).ok()) return s;
    if (!(s = g->out_vec.ensure(sizeof(double) * 3 * w)).ok()) return s;
    double* vec = g->out_vec.as<double>();
    cvg::launch_unshift_global(g->all.local(), g->n, k, m, g->all.kp(), g->all.shift(), g->out_xtx.as<double>(),
                               g->out_xty.as<double>(), vec, vec + w, vec + 2 * w, st);
    g->ctx->launches += 1;
    if (!(s = cvg::cuda_status(cudaGetLastError(), "unshift kernel")).ok()) return s;
    if (!(s = d2h(xtx, g->out_xtx.as<void>(), sizeof(double) * k * k, st)).ok()) return s;
    if (!(s = d2h(xty, g->out_xty.as<void>(), sizeof(double) * k * m, st)).ok()) return s;
    if (cfg & 15u) {  // fast.hpp:25-30
      if (!(s = d2h(sum_x, vec, sizeof(double) * k, st)).ok()) return s;
      if (!(s = d2h(sum_y, vec + k, sizeof(double) * m, st)).ok()) return s;
      if (!(s = d2h(mean_x, vec + 2 * w, sizeof(double) * k, st)).ok()) return s;
      if (!(s = d2h(mean_y, vec + 2 * w + k, sizeof(double) * m, st)).ok()) return s;
    }
    if (cfg & (CVG_SCALE_X | CVG_SCALE_Y)) {  // fast.hpp:31-34
      if (!(s = d2h(sum_sq_x, vec + w, sizeof(double) * k, st)).ok()) return s;
      if (!(s = d2h(sum_sq_y, vec + w + k, sizeof(double) * m, st)).ok()) return s;
    }
    return cvg::cuda_status(cudaStreamSynchronize(st), "stream synchronize");
  });
}

int cvg_global_fold_products(cvg_global* g, const int64_t* v_rows, int64_t n_val, uint32_t cfg, double* xtx_t,
                             double* xty_t, double* mean_x_t, double* mean_y_t, double* std_x_t, double* std_y_t,
                             int64_t* n_train, char* err, size_t errlen) {
  return guarded(err, errlen, [&]() -> Status {
    if (!g) return Status::Err(CVG_E_INVALID_ARG, "null global");
    if (cudaSetDevice(g->ctx->device) != cudaSuccess) return Status::Err(CVG_E_CUDA, "cudaSetDevice failed");
    if (cfg > 15u) return Status::Err(CVG_E_INVALID_ARG, "configuration mask outside 0..15");
    const int64_t n = g->n, k = g->k, m = g->m;
    // fast.hpp:78-82
    if (n_val == 0) return Status::Err(CVG_E_INVALID_ARG, "fold_products: empty validation partition");
    if (n_val >= n) return Status::Err(CVG_E_INVALID_ARG, "fold_products: degenerate fold covers all rows");
    if ((cfg & (CVG_SCALE_X | CVG_SCALE_Y)) && n - n_val < 2)
      return Status::Err(CVG_E_SCALABILITY, "fold_products: scaling needs at least 2 training rows");
    for (int64_t i = 0; i < n_val; ++i)
      if (v_rows[i] < 0 || v_rows[i] >= n || (i && v_rows[i] <= v_rows[i - 1]))
        return Status::Err(CVG_E_INVALID_ARG, "fold_products: v_rows must be ascending row indices in [0, n)");
    Status s;
    cudaStream_t st = g->ctx->stream;
    if (!(s = g->fold.create(g->ctx, g->dtype, n, k, m, 1, 0, 1, false)).ok()) return s;
    if (!(s = g->fold.bind_rows(v_rows, n_val)).ok()) return s;
    if (!(s = g->fold.gram(g->x.as<void>(), k, g->y.as<void>(), m, nullptr, g->all.shift())).ok()) return s;
    if (!(s = g->out_xtx.ensure(sizeof(double) * k * k)).ok()) return s;
    if (!(s = g->out_xty.ensure(sizeof(double) * k * m)).ok()) return s;
    if (!(s = g->out_vec.ensure(sizeof(double) * 3 * (k + m))).ok()) return s;
    double* vec = g->out_vec.as<double>();
    const int64_t w = k + m;
    if (!(s = g->fold.finish(nullptr, 1, g->all.local(), &cfg, 1, g->out_xtx.as<double>(), g->out_xty.as<double>(),
                             vec, vec + k, vec + w, vec + w + k))
             .ok())
      return s;
    if (!(s = d2h(xtx_t, g->out_xtx.as<void>(), sizeof(double) * k * k, st)).ok()) return s;
    if (!(s = d2h(xty_t, g->out_xty.as<void>(), sizeof(double) * k * m, st)).ok()) return s;
    if (cfg & 15u) {
      if (!(s = d2h(mean_x_t, vec, sizeof(double) * k, st)).ok()) return s;
      if (!(s = d2h(mean_y_t, vec + k, sizeof(double) * m, st)).ok()) return s;
    }
    if (cfg & CVG_SCALE_X)
      if (!(s = d2h(std_x_t, vec + w, sizeof(double) * k, st)).ok()) return s;
    if (cfg & CVG_SCALE_Y)
      if (!(s = d2h(std_y_t, vec + w + k, sizeof(double) * m, st)).ok()) return s;
    if (n_train) *n_train = n - n_val;
    return cvg::cuda_status(cudaStreamSynchronize(st), "stream synchronize");
  });
}

namespace {
// Pooled pinned host blocks (cvg_host_alloc): freed blocks are kept for reuse, so output arrays handed to a caller
// and dropped again cost neither cudaHostAlloc nor first-touch page faults on the next call.
struct HostPool {
  std::mutex mu;
  std::multimap<size_t, void*> free_blocks;
  std::map<void*, size_t> size_of;
  size_t cached = 0;
  static constexpr size_t kMaxCached = size_t(8) << 30;
};
HostPool& host_pool() {
  static HostPool* pool = new HostPool();  // never destroyed: finalizers may run at interpreter exit
  return *pool;
}
}  // namespace

int cvg_host_alloc(size_t bytes, void** out) {
  if (!out) return CVG_E_INVALID_ARG;
  *out = nullptr;
  const size_t want = std::max<size_t>((bytes + (size_t(1) << 16) - 1) & ~((size_t(1) << 16) - 1), size_t(1) << 16);
  HostPool& hp = host_pool();
  {
    std::lock_guard<std::mutex> lk(hp.mu);
    auto it = hp.free_blocks.lower_bound(want);
    if (it != hp.free_blocks.end() && it->first <= 2 * want) {
      *out = it->second;
      hp.cached -= it->first;
      hp.free_blocks.erase(it);
      return CVG_OK;
    }
  }
  void* p = nullptr;
  if (cudaHostAlloc(&p, want, cudaHostAllocPortable) != cudaSuccess) {
    cudaGetLastError();
    return CVG_E_OOM;
  }
  std::lock_guard<std::mutex> lk(hp.mu);
  hp.size_of[p] = want;
  *out = p;
  return CVG_OK;
}

void cvg_host_free(void* p) {
  if (!p) return;
  HostPool& hp = host_pool();
  std::lock_guard<std::mutex> lk(hp.mu);
  auto it = hp.size_of.find(p);
  if (it == hp.size_of.end()) return;
  if (hp.cached + it->second > HostPool::kMaxCached) {
    cudaFreeHost(p);
    hp.size_of.erase(it);
    return;
  }
  hp.free_blocks.emplace(it->second, p);
  hp.cached += it->second;
}

int cvg_selftest_division(cvg_context* ctx, int64_t n, uint64_t seed, int64_t* mismatches, int64_t* fast) {
  return guarded(nullptr, 0, [&]() -> Status {
    if (!ctx || n < 0) return Status::Err(CVG_E_INVALID_ARG, "bad arguments");
    Status s = cvg::cuda_status(cudaSetDevice(ctx->device), "cudaSetDevice");
    if (!s.ok()) return s;
    cvg::DevBuf counts;
    if (!(s = counts.ensure(2 * sizeof(unsigned long long))).ok()) return s;
    if (!(s = cvg::cuda_status(cudaMemsetAsync(counts.as<void>(), 0, 2 * sizeof(unsigned long long), ctx->stream),
                               "memset")).ok())
      return s;
    cvg::launch_selftest_division(seed, n, counts.as<unsigned long long>(), ctx->stream);
    ctx->launches += 1;
    unsigned long long h[2] = {0, 0};
    if (!(s = d2h(h, counts.as<void>(), sizeof h, ctx->stream)).ok()) return s;
    if (!(s = cvg::cuda_status(cudaStreamSynchronize(ctx->stream), "stream synchronize")).ok()) return s;
    if (mismatches) *mismatches = (int64_t)h[0];
    if (fast) *fast = (int64_t)h[1];
    return Status::Ok();
  });
}


int cvg_training_mean(cvg_context* ctx, const double* global_mean, const double* val_mean, int64_t len, int64_t n,
                      int64_t n_val, double* out, char* err, size_t errlen) {
  return guarded(err, errlen, [&]() -> Status {
    if (!ctx) return Status::Err(CVG_E_INVALID_ARG, "null context");
    if (n_val >= n) return Status::Err(CVG_E_INVALID_ARG, "training_mean: validation rows cover the dataset");
    return small_vector_op(ctx, {{global_mean, len}, {val_mean, len}}, out, len,
                           [&](const std::vector<const double*>& d, double* o) {
                             cvg::launch_training_mean(d[0], d[1], len, n, n_val, o, ctx->stream);
                           });
  });
}

int cvg_training_std(cvg_context* ctx, const double* mean_t, const double* sum_t, const double* sum_sq_t,
                     int64_t len, int64_t n_train, double* out, char* err, size_t errlen) {
  return guarded(err, errlen, [&]() -> Status {
    if (!ctx) return Status::Err(CVG_E_INVALID_ARG, "null context");
    if (n_train < 2) return Status::Err(CVG_E_SCALABILITY, "training_std: need at least 2 training rows");
    return small_vector_op(ctx, {{mean_t, len}, {sum_t, len}, {sum_sq_t, len}}, out, len,
                           [&](const std::vector<const double*>& d, double* o) {
                             cvg::launch_training_std(d[0], d[1], d[2], len, n_train, o, ctx->stream);
                           });
  });
}

int cvg_hadamard_outer_divide(cvg_context* ctx, const double* mat, int64_t rows, int64_t cols, const double* left,
                              int64_t n_left, const double* right, int64_t n_right, double* out, char* err,
                              size_t errlen) {
  return guarded(err, errlen, [&]() -> Status {
    if (!ctx) return Status::Err(CVG_E_INVALID_ARG, "null context");
    if (n_left != rows || n_right != cols)
      return Status::Err(CVG_E_DIMENSION, "divisor vector lengths must match matrix shape");
    for (int64_t i = 0; i < n_left; ++i)
      if (!(left[i] > 0.0))
        return Status::Err(CVG_E_INVALID_ARG, "hadamard_outer_divide: non-positive left divisor");
    for (int64_t j = 0; j < n_right; ++j)
      if (!(right[j] > 0.0))
        return Status::Err(CVG_E_INVALID_ARG, "hadamard_outer_divide: non-positive right divisor");
    return small_vector_op(ctx, {{mat, rows * cols}, {left, rows}, {right, cols}}, out, rows * cols,
                           [&](const std::vector<const double*>& d, double* o) {
                             cvg::launch_hadamard(d[0], rows, cols, d[1], d[2], o, ctx->stream);
                           });
  });
}

}  // extern "C"
