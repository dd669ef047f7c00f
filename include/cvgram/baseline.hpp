#pragma once
// The baseline engine (reference baseline.hpp:1-99) on the B200: every fold's
// training rows are contracted directly in their own mean-centered basis (two
// passes, no downdate) — the independent engine `cvgram verify` checks the
// fast path against.  Same signatures, validation and exceptions.

#include <vector>

#include "cvgram/core.hpp"
#include "cvgram/engine.hpp"
#include "cvgram/partition.hpp"

namespace cvgram {

/// One fold by direct recomputation from its training rows (baseline.hpp:42-76).
inline FoldResult baseline_single_fold(const DatasetPair& data, const std::vector<Index>& v_rows,
                                       const PreprocessConfig& cfg, int fold_id = 0) {
  const Index k = data.n_features(), m = data.n_responses();
  FoldResult r;
  r.fold_id = fold_id;
  r.xtx_t = Matrix(k, k);
  r.xty_t = Matrix(k, m);
  Vector mx(k), my(m), sx(k), sy(m);
  std::vector<int64_t> rows(v_rows.begin(), v_rows.end());
  int64_t n_train = 0;
  char err[512] = {0};
  detail::check(cvg_baseline_single_fold(detail::Context::get(), CVG_DTYPE_F64, data.x().data(), data.y().data(),
                                         data.n_rows(), k, m, rows.data(), static_cast<int64_t>(rows.size()),
                                         cfg.mask(), r.xtx_t.data(), r.xty_t.data(), mx.data(), my.data(), sx.data(),
                                         sy.data(), &n_train, err, sizeof err),
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

/// Per-fold training products by direct recomputation; ascending fold order (baseline.hpp:79-97).
inline std::vector<FoldResult> baseline_fold_products(const DatasetPair& data, const Partitioning& part,
                                                      const PreprocessConfig& cfg, int n_threads = 1) {
  (void)n_threads;
  const Index n = data.n_rows(), k = data.n_features(), m = data.n_responses();
  const int p = part.p;
  const size_t pp = p > 0 ? static_cast<size_t>(p) : 0;
  std::vector<int32_t> labels(part.labels.begin(), part.labels.end());
  const uint32_t mask = cfg.mask();
  std::vector<double> xtx(pp * k * k), xty(pp * k * m), mx(pp * k), my(pp * m), sx(pp * k), sy(pp * m);
  std::vector<int64_t> nt(pp), nv(pp);
  char err[512] = {0};
  detail::check(cvg_baseline_fold_products(detail::Context::get(), CVG_DTYPE_F64, data.x().data(), data.y().data(), n,
                                           k, m, labels.data(), part.n_rows(), p, &mask, 1, xtx.data(), xty.data(),
                                           mx.data(), my.data(), sx.data(), sy.data(), nt.data(), nv.data(), err,
                                           sizeof err),
                err);
  std::vector<FoldResult> out(pp);
  auto vec = [](const double* src, Index len) {
    Vector v(len);
    std::copy(src, src + len, v.data());
    return v;
  };
  for (size_t f = 0; f < pp; ++f) {
    FoldResult& r = out[f];
    r.fold_id = static_cast<int>(f) + 1;
    r.xtx_t = Matrix(k, k);
    r.xty_t = Matrix(k, m);
    std::copy_n(xtx.data() + f * k * k, k * k, r.xtx_t.data());
    std::copy_n(xty.data() + f * k * m, k * m, r.xty_t.data());
    r.stats.n_train = nt[f];
    r.stats.n_val = nv[f];
    if (cfg.any()) {
      r.stats.mean_x_t = vec(mx.data() + f * k, k);
      r.stats.mean_y_t = vec(my.data() + f * m, m);
    }
    if (cfg.scale_x) r.stats.std_x_t = vec(sx.data() + f * k, k);
    if (cfg.scale_y) r.stats.std_y_t = vec(sy.data() + f * m, m);
  }
  return out;
}

}  // namespace cvgram
