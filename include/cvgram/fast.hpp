#pragma once
// The fast engine (reference fast.hpp:1-152), on the B200: one Gram pass over
// fold-bucketed rows serves the whole-data products and every fold's
// validation products; the per-fold downdate, centering and scaling run in the
// device epilogue.  Same signatures, validation order and exceptions.

#include <type_traits>
#include <vector>

#include "cvgram/core.hpp"
#include "cvgram/engine.hpp"
#include "cvgram/partition.hpp"

namespace cvgram {

/// Whole-dataset products and the statistic vectors cfg needs (fast.hpp:19-36).
inline GlobalCache precompute_global(const DatasetPair& data, const PreprocessConfig& cfg) {
  GlobalCache cache;
  cache.n_rows = data.n_rows();
  cache.device = make_device_global(data);
  const Index k = data.n_features(), m = data.n_responses();
  cache.xtx = Matrix(k, k);
  cache.xty = Matrix(k, m);
  Vector sx(k), sy(m), mx(k), my(m), qx(k), qy(m);
  char err[512] = {0};
  detail::check(cvg_global_export(cache.device->h, cfg.mask(), cache.xtx.data(), cache.xty.data(), sx.data(),
                                  sy.data(), mx.data(), my.data(), qx.data(), qy.data(), err, sizeof err),
                err);
  if (cfg.any()) {
    cache.sum_x = sx;
    cache.sum_y = sy;
    cache.mean_x = mx;
    cache.mean_y = my;
  }
  if (cfg.any_scale()) {
    cache.sum_sq_x = qx;
    cache.sum_sq_y = qy;
  }
  return cache;
}

/// (n/(n-n_val))·global_mean − (n_val/(n-n_val))·val_mean (fast.hpp:40-47), on the device.
inline Vector training_mean(const Vector& global_mean, const Vector& val_mean, Index n, Index n_val) {
  Vector out(global_mean.size());
  char err[512] = {0};
  detail::check(cvg_training_mean(detail::Context::get(), global_mean.data(), val_mean.data(), global_mean.size(), n,
                                  n_val, out.data(), err, sizeof err),
                err);
  return out;
}

/// Bessel-corrected std from training sums, clamp, zero -> 1 (fast.hpp:53-69), on the device.
inline Vector training_std(const Vector& mean_t, const Vector& sum_t, const Vector& sum_sq_t, Index n_train) {
  Vector out(mean_t.size());
  char err[512] = {0};
  detail::check(cvg_training_std(detail::Context::get(), mean_t.data(), sum_t.data(), sum_sq_t.data(), mean_t.size(),
                                 n_train, out.data(), err, sizeof err),
                err);
  return out;
}

/// Training products for one fold from the cache + its validation rows (fast.hpp:73-130).
inline FoldResult fold_products(const GlobalCache& cache, const DatasetPair& data, const std::vector<Index>& v_rows,
                                const PreprocessConfig& cfg, int fold_id = 0) {
  std::shared_ptr<DeviceGlobal> dev = cache.device;
  if (!dev || dev->x_data != data.x().data() || dev->n != data.n_rows()) dev = make_device_global(data);
  const Index k = data.n_features(), m = data.n_responses();
  FoldResult r;
  r.fold_id = fold_id;
  r.xtx_t = Matrix(k, k);
  r.xty_t = Matrix(k, m);
  Vector mx(k), my(m), sx(k), sy(m);
  std::vector<int64_t> rows(v_rows.begin(), v_rows.end());
  int64_t n_train = 0;
  char err[512] = {0};
  detail::check(cvg_global_fold_products(dev->h, rows.data(), static_cast<int64_t>(rows.size()), cfg.mask(),
                                         r.xtx_t.data(), r.xty_t.data(), mx.data(), my.data(), sx.data(), sy.data(),
                                         &n_train, err, sizeof err),
                err);
  r.stats.n_train = n_train;
  r.stats.n_val = static_cast<Index>(v_rows.size());
  if (cfg.any()) {
    r.stats.mean_x_t = mx;
    r.stats.mean_y_t = my;
  }
  if (cfg.scale_x) r.stats.std_x_t = sx;
  if (cfg.scale_y) r.stats.std_y_t = sy;
  return r;
}

/// Several configurations from one Gram pass; result[c][f] is fold f+1 of cfgs[c].
inline std::vector<std::vector<FoldResult>> run_all_folds_configs(const DatasetPair& data, const Partitioning& part,
                                                                  const std::vector<PreprocessConfig>& cfgs) {
  const Index n = data.n_rows(), k = data.n_features(), m = data.n_responses();
  const int p = part.p;
  const size_t nc = cfgs.size();
  std::vector<int32_t> labels(part.labels.begin(), part.labels.end());
  std::vector<uint32_t> masks;
  for (const auto& c : cfgs) masks.push_back(c.mask());
  const size_t pp = p > 0 ? static_cast<size_t>(p) : 0;
  std::vector<double> xtx(nc * pp * k * k), xty(nc * pp * k * m), mx(nc * pp * k), my(nc * pp * m),
      sx(nc * pp * k), sy(nc * pp * m);
  std::vector<int64_t> nt(pp), nv(pp);
  char err[512] = {0};
  detail::check(cvg_run_all_folds(detail::Context::get(), CVG_DTYPE_F64, data.x().data(), data.y().data(), n, k, m,
                                  labels.data(), part.n_rows(), p, masks.data(), static_cast<int32_t>(nc), xtx.data(),
                                  xty.data(), mx.data(), my.data(), sx.data(), sy.data(), nt.data(), nv.data(), err,
                                  sizeof err),
                err);
  std::vector<std::vector<FoldResult>> out(nc);
  auto vec = [](const double* src, Index len) {
    Vector v(len);
    std::copy(src, src + len, v.data());
    return v;
  };
  for (size_t c = 0; c < nc; ++c) {
    out[c].resize(pp);
    for (size_t f = 0; f < pp; ++f) {
      FoldResult& r = out[c][f];
      r.fold_id = static_cast<int>(f) + 1;
      r.xtx_t = Matrix(k, k);
      r.xty_t = Matrix(k, m);
      std::copy_n(xtx.data() + (c * pp + f) * k * k, k * k, r.xtx_t.data());
      std::copy_n(xty.data() + (c * pp + f) * k * m, k * m, r.xty_t.data());
      r.stats.n_train = nt[f];
      r.stats.n_val = nv[f];
      if (cfgs[c].any()) {
        r.stats.mean_x_t = vec(mx.data() + (c * pp + f) * k, k);
        r.stats.mean_y_t = vec(my.data() + (c * pp + f) * m, m);
      }
      if (cfgs[c].scale_x) r.stats.std_x_t = vec(sx.data() + (c * pp + f) * k, k);
      if (cfgs[c].scale_y) r.stats.std_y_t = vec(sy.data() + (c * pp + f) * m, m);
    }
  }
  return out;
}

/// Lazy per-fold generation (cvg_run_all_folds_stream) for leave-one-out-scale P:
/// fn(config_index, FoldResult&&) is called for every configuration and fold, folds
/// ascending, while only `batch` folds of outputs exist at a time.  fn may return
/// bool (true stops the run) or void.  Same values as run_all_folds_configs.
template <class F>
inline void for_each_fold(const DatasetPair& data, const Partitioning& part, const std::vector<PreprocessConfig>& cfgs,
                          F&& fn, int batch = 1024) {
  const Index n = data.n_rows(), k = data.n_features(), m = data.n_responses();
  std::vector<int32_t> labels(part.labels.begin(), part.labels.end());
  std::vector<uint32_t> masks;
  for (const auto& c : cfgs) masks.push_back(c.mask());
  struct State {
    F* fn;
    const std::vector<PreprocessConfig>* cfgs;
    Index k, m;
  } state{&fn, &cfgs, k, m};
  auto tramp = [](int32_t lo, int32_t hi, const double* xtx, const double* xty, const double* mx, const double* my,
                  const double* sx, const double* sy, const int64_t* nt, const int64_t* nv, void* user) -> int {
    State& st = *static_cast<State*>(user);
    const Index nb = hi - lo, kk = st.k, mm = st.m;
    const size_t nc = st.cfgs->size();
    auto vec = [](const double* src, Index len) {
      Vector v(len);
      std::copy(src, src + len, v.data());
      return v;
    };
    for (Index f = 0; f < nb; ++f)
      for (size_t c = 0; c < nc; ++c) {
        const PreprocessConfig& cfg = (*st.cfgs)[c];
        FoldResult r;
        r.fold_id = static_cast<int>(lo + f) + 1;
        r.xtx_t = Matrix(kk, kk);
        r.xty_t = Matrix(kk, mm);
        std::copy_n(xtx + (c * nb + f) * kk * kk, kk * kk, r.xtx_t.data());
        std::copy_n(xty + (c * nb + f) * kk * mm, kk * mm, r.xty_t.data());
        r.stats.n_train = nt[f];
        r.stats.n_val = nv[f];
        if (cfg.any()) {
          r.stats.mean_x_t = vec(mx + f * kk, kk);
          r.stats.mean_y_t = vec(my + f * mm, mm);
        }
        if (cfg.scale_x) r.stats.std_x_t = vec(sx + f * kk, kk);
        if (cfg.scale_y) r.stats.std_y_t = vec(sy + f * mm, mm);
        if constexpr (std::is_same_v<decltype((*st.fn)(0, std::move(r))), bool>) {
          if ((*st.fn)(static_cast<int>(c), std::move(r))) return 1;
        } else {
          (*st.fn)(static_cast<int>(c), std::move(r));
        }
      }
    return 0;
  };
  char err[512] = {0};
  detail::check(cvg_run_all_folds_stream(detail::Context::get(), CVG_DTYPE_F64, data.x().data(), data.y().data(), n, k,
                                         m, labels.data(), part.n_rows(), part.p, masks.data(),
                                         static_cast<int32_t>(masks.size()), batch, +tramp, &state, err, sizeof err),
                err);
}

/// One global pass, then every fold; ascending fold_id (fast.hpp:133-152).
/// n_threads only scheduled folds in the reference; the device grid replaces
/// it and results never depend on it (threading.hpp:8-10).
inline std::vector<FoldResult> run_all_folds(const DatasetPair& data, const Partitioning& part,
                                             const PreprocessConfig& cfg, int n_threads = 1) {
  (void)n_threads;
  if (part.n_rows() != data.n_rows()) throw dimension_error("partitioning length does not match sample count");
  return std::move(run_all_folds_configs(data, part, std::vector<PreprocessConfig>{cfg})[0]);
}

}  // namespace cvgram
