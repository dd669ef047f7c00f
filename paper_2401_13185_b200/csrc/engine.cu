// Host orchestration: plans the fold-bucketed layout, launches K1..K5 on the
// context stream and keeps every reduction in a fixed order.
//
// Call stack it replaces: run_all_folds (fast.hpp:133-152) ->
// precompute_global (fast.hpp:19-36) + build_validation_partitions
// (partition.hpp:61-68) + parallel_for over fold_products (fast.hpp:73-130,
// threading.hpp:12-26).  Here: bucket (device) -> K1 reorder/shift -> K2 fold
// Gram -> K4 fold/total sums -> [cross-rank combine] -> K5 stats + products.
#include <algorithm>
#include <climits>
#include <cstring>
#include <string>

#include "engine.cuh"

cudaEvent_t cvg_context::take_event() {
  if (!event_pool.empty()) {
    cudaEvent_t e = event_pool.back();
    event_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

void cvg_context::begin(int cls) {
  Rec r{cls, take_event(), take_event()};
  cudaEventRecord(r.a, stream);
  recs.push_back(r);
}

void cvg_context::end() { cudaEventRecord(recs.back().b, stream); }

void cvg_context::clear_recs() {
  for (auto& r : recs) {
    event_pool.push_back(r.a);
    event_pool.push_back(r.b);
  }
  recs.clear();
}

namespace cvg {

Status cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return Status::Ok();
  const int code = (e == cudaErrorMemoryAllocation) ? 6 : 5;
  return Status::Err(code, std::string(what) + ": " + cudaGetErrorString(e));
}

#define CVG_CK(expr)                                     \
  do {                                                   \
    Status _s = cuda_status((expr), #expr);              \
    if (!_s.ok()) return _s;                             \
  } while (0)
#define CVG_TRY(expr)          \
  do {                         \
    Status _s = (expr);        \
    if (!_s.ok()) return _s;   \
  } while (0)

Status DevBuf::ensure(size_t bytes) {
  if (bytes <= bytes_) return Status::Ok();
  release();
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return Status::Err(6, std::string("device allocation of ") + std::to_string(bytes) + " bytes failed: " +
                              cudaGetErrorString(e));
  }
  p_ = p;
  bytes_ = bytes;
  return Status::Ok();
}

void DevBuf::release() {
  if (p_) cudaFree(p_);
  p_ = nullptr;
  bytes_ = 0;
}

std::vector<int2> gram_tiles(int64_t k, int64_t m, int64_t kp) {
  const int nt = (int)(kp / kTile);
  const int tx = (int)((k - 1) / kTile);  // last tile holding X columns
  const int to = (int)((k + m) / kTile);  // tile holding the ones column
  std::vector<int2> t;
  for (int i = 0; i < nt; ++i)
    for (int j = i; j < nt; ++j)
      if (i <= tx || j == i || j == to) t.push_back(make_int2(i, j));
  return t;
}

Status Plan::count_launch(int n) {
  ctx_->launches += n;
  return cuda_status(cudaGetLastError(), "kernel launch");
}

Status Plan::create(cvg_context* ctx, int dtype, int64_t n, int64_t k, int64_t m, int32_t p, int32_t fb, int32_t fe,
                    bool validate) {
  ctx_ = ctx;
  dtype_ = dtype;
  n_ = n;
  k_ = k;
  m_ = m;
  w_ = k + m;
  p_ = p;
  fb_ = fb;
  fe_ = fe;
  bound_ = grammed_ = false;
  if (dtype != 0 && dtype != 1) return Status::Err(4, "unsupported dtype");
  if (n < 2) return Status::Err(1, "need at least 2 samples");
  if (k < 1 || m < 1) return Status::Err(1, "x and y must each have at least one column");
  if (validate) {
    if (p < 2) return Status::Err(2, "fold count must be at least 2, got " + std::to_string(p));
    if ((int64_t)p > n)
      return Status::Err(2, "fold count " + std::to_string(p) + " exceeds sample count " + std::to_string(n));
  }
  if (fb < 0 || fe > p || fb > fe) return Status::Err(4, "owned fold range is outside [0, p]");
  kp_ = padded_cols(k, m);
  tiles_ = gram_tiles(k, m, kp_);
  out_tiles_.clear();
  for (const int2& t : tiles_)
    if ((int64_t)t.x * kTile < k) out_tiles_.push_back(t);
  CVG_CK(cudaSetDevice(ctx->device));
  CVG_TRY(tiles_d_.ensure(tiles_.size() * sizeof(int2)));
  CVG_TRY(out_tiles_d_.ensure(out_tiles_.size() * sizeof(int2)));
  CVG_CK(cudaMemcpyAsync(tiles_d_.as<int2>(), tiles_.data(), tiles_.size() * sizeof(int2), cudaMemcpyHostToDevice,
                         ctx->stream));
  CVG_CK(cudaMemcpyAsync(out_tiles_d_.as<int2>(), out_tiles_.data(), out_tiles_.size() * sizeof(int2),
                         cudaMemcpyHostToDevice, ctx->stream));
  CVG_TRY(local_.ensure(sizeof(double) * kp_ * kp_));
  CVG_TRY(shift_.ensure(sizeof(double) * kp_));
  CVG_TRY(flag_.ensure(sizeof(int)));
  return Status::Ok();
}

Status Plan::bind_labels(const int32_t* d_labels, bool validate, bool require_scalable) {
  cudaStream_t s = ctx_->stream;
  const int64_t ntiles = (n_ + kTileRowsPerWarp - 1) / kTileRowsPerWarp;
  CVG_TRY(tile_counts_.ensure(sizeof(int32_t) * ntiles * p_));
  CVG_TRY(fold_counts_.ensure(sizeof(int64_t) * p_));
  CVG_TRY(bad_.ensure(sizeof(unsigned long long)));
  CVG_CK(cudaMemsetAsync(tile_counts_.as<void>(), 0, sizeof(int32_t) * ntiles * p_, s));
  CVG_CK(cudaMemsetAsync(bad_.as<void>(), 0xff, sizeof(unsigned long long), s));
  {
    Timed t(ctx_, kBucket);
    launch_tile_histogram(d_labels, n_, p_, tile_counts_.as<int32_t>(), bad_.as<unsigned long long>(), s);
  }
  CVG_TRY(count_launch());
  {
    Timed t(ctx_, kBucket);
    launch_tile_scan(tile_counts_.as<int32_t>(), ntiles, p_, fold_counts_.as<int64_t>(), s);
  }
  CVG_TRY(count_launch());
  counts_.assign(p_, 0);
  unsigned long long bad = 0;
  CVG_CK(cudaMemcpyAsync(counts_.data(), fold_counts_.as<int64_t>(), sizeof(int64_t) * p_, cudaMemcpyDeviceToHost,
                         s));
  CVG_CK(cudaMemcpyAsync(&bad, bad_.as<unsigned long long>(), sizeof bad, cudaMemcpyDeviceToHost, s));
  CVG_CK(cudaStreamSynchronize(s));
  if (bad != ~0ull) {  // partition.hpp:34-38, first offending sample
    int32_t label = 0;
    CVG_CK(cudaMemcpy(&label, d_labels + bad, sizeof label, cudaMemcpyDeviceToHost));
    return Status::Err(2, "label " + std::to_string(label) + " at sample " + std::to_string(bad + 1) +
                              " is outside {1.." + std::to_string(p_) + "}");
  }
  if (validate) {
    for (int32_t f = 0; f < p_; ++f)
      if (counts_[f] == 0) return Status::Err(2, "fold " + std::to_string(f + 1) + " is empty");
    if (require_scalable)
      for (int32_t f = 0; f < p_; ++f)
        if (n_ - counts_[f] < 2)
          return Status::Err(3, "fold " + std::to_string(f + 1) + " leaves a training partition of " +
                                    std::to_string(n_ - counts_[f]) + " rows; scaling needs at least 2");
  }
  CVG_TRY(plan_segments());
  CVG_CK(cudaMemsetAsync(src_row_.as<void>(), 0xff, sizeof(int64_t) * std::max<int64_t>(zrows_, 1), s));
  {
    Timed t(ctx_, kBucket);
    launch_scatter(d_labels, n_, p_, fb_, fe_, tile_counts_.as<int32_t>(), zbase_d_.as<int64_t>(),
                   src_row_.as<int64_t>(), s);
  }
  CVG_TRY(count_launch());
  bound_ = true;
  return Status::Ok();
}

Status Plan::bind_rows(const int64_t* rows, int64_t nrows) {
  if (p_ != 1 || fb_ != 0 || fe_ != 1) return Status::Err(4, "bind_rows needs a single-fold plan");
  counts_.assign(1, nrows);
  CVG_TRY(plan_segments());
  std::vector<int64_t> src(std::max<int64_t>(zrows_, 1), -1);
  std::copy(rows, rows + nrows, src.begin());
  CVG_CK(cudaMemcpyAsync(src_row_.as<int64_t>(), src.data(), sizeof(int64_t) * src.size(), cudaMemcpyHostToDevice,
                         ctx_->stream));
  CVG_CK(cudaStreamSynchronize(ctx_->stream));  // `src` is a pageable temporary
  bound_ = true;
  return Status::Ok();
}

Status Plan::plan_segments() {
  segs_.clear();
  fold_seg_begin_.assign(1, 0);
  fold_zbase_.clear();
  zrows_ = 0;
  for (int32_t f = fb_; f < fe_; ++f) {
    const int64_t padded = round_up(counts_[f], kRowStep);
    fold_zbase_.push_back(zrows_);
    for (int64_t off = 0; off < padded; off += kChunkRows)
      segs_.push_back(GramTask{zrows_ + off, std::min<int64_t>(kChunkRows, padded - off)});
    zrows_ += padded;
    fold_seg_begin_.push_back((int32_t)segs_.size());
  }
  const int nown = fe_ - fb_;
  cudaStream_t s = ctx_->stream;
  CVG_TRY(zbase_d_.ensure(sizeof(int64_t) * std::max(nown, 1)));
  CVG_TRY(src_row_.ensure(sizeof(int64_t) * std::max<int64_t>(zrows_, 1)));
  CVG_TRY(z_.ensure(sizeof(double) * std::max<int64_t>(zrows_, 1) * kp_));
  CVG_TRY(part_.ensure(sizeof(double) * std::max<size_t>(segs_.size(), 1) * kp_ * kp_));
  CVG_TRY(segs_d_.ensure(sizeof(GramTask) * std::max<size_t>(segs_.size(), 1)));
  CVG_TRY(nval_d_.ensure(sizeof(int64_t) * std::max(nown, 1)));
  if (nown > 0) {
    CVG_CK(cudaMemcpyAsync(zbase_d_.as<int64_t>(), fold_zbase_.data(), sizeof(int64_t) * nown,
                           cudaMemcpyHostToDevice, s));
    CVG_CK(cudaMemcpyAsync(nval_d_.as<int64_t>(), counts_.data() + fb_, sizeof(int64_t) * nown,
                           cudaMemcpyHostToDevice, s));
  }
  if (!segs_.empty())
    CVG_CK(cudaMemcpyAsync(segs_d_.as<GramTask>(), segs_.data(), sizeof(GramTask) * segs_.size(),
                           cudaMemcpyHostToDevice, s));
  // Fold Gram pointers: the segment partial itself for single-segment folds,
  // otherwise a fixed-order sum into foldbuf (K4).
  int nmulti = 0;
  for (int f = 0; f < nown; ++f)
    if (fold_seg_begin_[f + 1] - fold_seg_begin_[f] != 1) ++nmulti;
  CVG_TRY(foldbuf_.ensure(sizeof(double) * std::max(nmulti, 1) * kp_ * kp_));
  fold_ptrs_.assign(nown, nullptr);
  std::vector<const double*> gsrc;
  std::vector<int32_t> gbeg{0};
  std::vector<double*> gdst;
  int slot = 0;
  for (int f = 0; f < nown; ++f) {
    const int a = fold_seg_begin_[f], b = fold_seg_begin_[f + 1];
    if (b - a == 1) {
      fold_ptrs_[f] = part_.as<double>() + (int64_t)a * kp_ * kp_;
    } else {
      double* dst = foldbuf_.as<double>() + (int64_t)slot++ * kp_ * kp_;
      fold_ptrs_[f] = dst;
      for (int sgi = a; sgi < b; ++sgi) gsrc.push_back(part_.as<double>() + (int64_t)sgi * kp_ * kp_);
      gbeg.push_back((int32_t)gsrc.size());
      gdst.push_back(dst);
    }
  }
  // group list: [multi-segment folds...] then the local fold-tree node in a
  // second launch (it depends on the first).
  std::vector<const double*> all_src = gsrc;
  all_src.insert(all_src.end(), fold_ptrs_.begin(), fold_ptrs_.end());
  std::vector<int32_t> all_beg = gbeg;
  all_beg.push_back((int32_t)all_src.size());
  std::vector<double*> all_dst = gdst;
  all_dst.push_back(local_.as<double>());
  CVG_TRY(grp_src_.ensure(sizeof(void*) * std::max<size_t>(all_src.size(), 1)));
  CVG_TRY(grp_begin_.ensure(sizeof(int32_t) * all_beg.size()));
  CVG_TRY(grp_dst_.ensure(sizeof(void*) * all_dst.size()));
  CVG_TRY(foldptr_d_.ensure(sizeof(void*) * std::max(nown, 1)));
  if (!all_src.empty())
    CVG_CK(cudaMemcpyAsync(grp_src_.as<void>(), all_src.data(), sizeof(void*) * all_src.size(),
                           cudaMemcpyHostToDevice, s));
  CVG_CK(cudaMemcpyAsync(grp_begin_.as<void>(), all_beg.data(), sizeof(int32_t) * all_beg.size(),
                         cudaMemcpyHostToDevice, s));
  CVG_CK(cudaMemcpyAsync(grp_dst_.as<void>(), all_dst.data(), sizeof(void*) * all_dst.size(), cudaMemcpyHostToDevice,
                         s));
  if (nown > 0)
    CVG_CK(cudaMemcpyAsync(foldptr_d_.as<void>(), fold_ptrs_.data(), sizeof(void*) * nown, cudaMemcpyHostToDevice,
                           s));
  // Host vectors above are pageable temporaries: make the copies complete.
  CVG_CK(cudaStreamSynchronize(s));
  return Status::Ok();
}

Status Plan::gram(const void* d_x, int64_t ldx, const void* d_y, int64_t ldy, const double* host_shift,
                  const double* dev_shift) {
  if (!bound_) return Status::Err(4, "plan has no bound partitioning");
  cudaStream_t s = ctx_->stream;
  double* shift = shift_.as<double>();
  if (dev_shift) {
    CVG_CK(cudaMemcpyAsync(shift, dev_shift, sizeof(double) * w_, cudaMemcpyDeviceToDevice, s));
  } else if (host_shift) {
    CVG_CK(cudaMemcpyAsync(shift, host_shift, sizeof(double) * w_, cudaMemcpyHostToDevice, s));
    CVG_CK(cudaStreamSynchronize(s));
  } else {
    Timed t(ctx_, kReorder);
    launch_shift_from_row0(dtype_, d_x, d_y, k_, m_, shift, s);
    CVG_TRY(count_launch());
  }
  CVG_CK(cudaMemsetAsync(flag_.as<void>(), 0, sizeof(int), s));
  if (zrows_ > 0) {
    {
      Timed t(ctx_, kReorder);
      launch_reorder(dtype_, d_x, ldx, d_y, ldy, k_, m_, src_row_.as<int64_t>(), zrows_, kp_, shift,
                     z_.as<double>(), flag_.as<int>(), s);
    }
    CVG_TRY(count_launch());
  }
  if (!segs_.empty()) {
    {
      Timed t(ctx_, kGram);
      launch_gram_f64(z_.as<double>(), kp_, segs_d_.as<GramTask>(), (int64_t)segs_.size(), tiles_d_.as<int2>(),
                      (int)tiles_.size(), part_.as<double>(), s);
    }
    CVG_TRY(count_launch());
  }
  const int nown = fe_ - fb_;
  int nmulti = 0;
  for (int f = 0; f < nown; ++f)
    if (fold_seg_begin_[f + 1] - fold_seg_begin_[f] != 1) ++nmulti;
  const double* const* srcs = grp_src_.as<const double*>();
  double* const* dsts = grp_dst_.as<double*>();
  const int32_t* beg = grp_begin_.as<int32_t>();
  if (nmulti > 0) {
    Timed t(ctx_, kTree);
    launch_tree_sum(srcs, beg, nmulti, dsts, kp_, tiles_d_.as<int2>(), (int)tiles_.size(), s);
    CVG_TRY(count_launch());
  }
  {
    Timed t(ctx_, kTree);
    launch_tree_sum(srcs, beg + nmulti, 1, dsts + nmulti, kp_, tiles_d_.as<int2>(), (int)tiles_.size(), s);
  }
  CVG_TRY(count_launch());
  grammed_ = true;
  return Status::Ok();
}

Status Plan::finish(const double* d_rank_partials, int32_t n_ranks, const double* total_override,
                    const uint32_t* cfgs, int32_t ncfg, double* d_xtx, double* d_xty, double* d_mean_x,
                    double* d_mean_y, double* d_std_x, double* d_std_y) {
  if (!grammed_) return Status::Err(4, "finish called before gram");
  cudaStream_t s = ctx_->stream;
  const double* total = nullptr;
  if (total_override) {
    total = total_override;
  } else if (d_rank_partials && n_ranks > 1) {
    CVG_TRY(total_.ensure(sizeof(double) * kp_ * kp_));
    std::vector<const double*> src(n_ranks);
    for (int r = 0; r < n_ranks; ++r) src[r] = d_rank_partials + (int64_t)r * kp_ * kp_;
    std::vector<int32_t> beg{0, n_ranks};
    double* dst = total_.as<double>();
    CVG_TRY(rankptr_d_.ensure(sizeof(void*) * n_ranks));
    CVG_TRY(rankbeg_d_.ensure(sizeof(int32_t) * 2));
    CVG_TRY(rankdst_d_.ensure(sizeof(void*)));
    CVG_CK(cudaMemcpyAsync(rankptr_d_.as<void>(), src.data(), sizeof(void*) * n_ranks, cudaMemcpyHostToDevice, s));
    CVG_CK(cudaMemcpyAsync(rankbeg_d_.as<void>(), beg.data(), sizeof(int32_t) * 2, cudaMemcpyHostToDevice, s));
    CVG_CK(cudaMemcpyAsync(rankdst_d_.as<void>(), &dst, sizeof(void*), cudaMemcpyHostToDevice, s));
    {
      Timed t(ctx_, kTree);
      launch_tree_sum(rankptr_d_.as<const double*>(), rankbeg_d_.as<int32_t>(), 1, rankdst_d_.as<double*>(), kp_,
                      tiles_d_.as<int2>(), (int)tiles_.size(), s);
    }
    CVG_TRY(count_launch());
    CVG_CK(cudaStreamSynchronize(s));  // host pointer vectors above are temporaries
    total = dst;
  } else if (d_rank_partials && n_ranks == 1) {
    total = d_rank_partials;
  } else {
    if (!owns_all()) return Status::Err(4, "plan owns a subset of folds: pass every rank's partial");
    total = local_.as<double>();
  }
  const int nown = fe_ - fb_;
  if (nown == 0) return Status::Ok();
  CVG_TRY(st_mz_.ensure(sizeof(double) * nown * w_));
  CVG_TRY(st_sT_.ensure(sizeof(double) * nown * w_));
  CVG_TRY(st_sd_.ensure(sizeof(double) * nown * w_));
  FoldStatsDev st{st_mz_.as<double>(), st_sT_.as<double>(), st_sd_.as<double>()};
  {
    Timed t(ctx_, kStats);
    launch_fold_stats(total, foldptr_d_.as<const double*>(), nval_d_.as<int64_t>(), nown, n_, k_, m_, kp_,
                      shift_.as<double>(), st, d_mean_x, d_mean_y, d_std_x, d_std_y, s);
  }
  CVG_TRY(count_launch());
  if (ncfg > 0) {
    CVG_TRY(cfg_d_.ensure(sizeof(uint32_t) * ncfg));
    CVG_CK(cudaMemcpyAsync(cfg_d_.as<void>(), cfgs, sizeof(uint32_t) * ncfg, cudaMemcpyHostToDevice, s));
    {
      Timed t(ctx_, kProducts);
      launch_products(total, foldptr_d_.as<const double*>(), nval_d_.as<int64_t>(), nown, n_, k_, m_, kp_,
                      shift_.as<double>(), st, out_tiles_d_.as<int2>(), (int)out_tiles_.size(),
                      cfg_d_.as<uint32_t>(), ncfg, d_xtx, d_xty, s);
    }
    CVG_TRY(count_launch());
  }
  int flag = 0;
  CVG_CK(cudaMemcpyAsync(&flag, flag_.as<int>(), sizeof flag, cudaMemcpyDeviceToHost, s));
  CVG_CK(cudaStreamSynchronize(s));
  if (flag) return Status::Err(1, "x and y entries must be finite");
  return Status::Ok();
}

}  // namespace cvg
