// Host orchestration: plans the fold-bucketed layout, launches K1..K5 on the
// context stream and keeps every reduction in a fixed order.
//
// Call stack it replaces: run_all_folds (fast.hpp:133-152) ->
// precompute_global (fast.hpp:19-36) + build_validation_partitions
// (partition.hpp:61-68) + parallel_for over fold_products (fast.hpp:73-130,
// threading.hpp:12-26).  Here: bucket (device) -> K1 reorder/shift -> K2 fold
// Gram -> K4 fold/total sums -> [cross-rank combine] -> K5 stats + products.
// Variants: host inputs streamed by column slabs on a copy stream (gram_host),
// compacted rows through a row map (multi-GPU all-to-all ingest), small-fold
// mode (every fold <= 32 rows: no per-fold partials, fold Grams formed in K5),
// and K5 over an emitted-fold subrange (streaming leave-one-out-scale P).
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <string>

#include <cstdio>

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

cvg::Status cvg_context::ensure_copy_stream() {
  if (copy_stream) return cvg::Status::Ok();
  return cvg::cuda_status(cudaStreamCreateWithFlags(&copy_stream, cudaStreamNonBlocking), "copy stream");
}

cvg::Status cvg_context::ensure_aux_stream() {
  if (aux_stream) return cvg::Status::Ok();
  return cvg::cuda_status(cudaStreamCreateWithFlags(&aux_stream, cudaStreamNonBlocking), "aux stream");
}

cudaEvent_t cvg_context::stream_event(size_t i) {
  while (sync_events.size() <= i) {
    cudaEvent_t e = nullptr;
    cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    sync_events.push_back(e);
  }
  return sync_events[i];
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

PinnedStage::~PinnedStage() {
  if (pending_) cudaEventSynchronize(ev_);
  if (ev_) cudaEventDestroy(ev_);
  if (p_) cudaFreeHost(p_);
}

Status PinnedStage::upload(std::initializer_list<Part> parts, cudaStream_t s) {
  size_t need = 0;
  for (const Part& q : parts) need += (q.bytes + 15) & ~size_t(15);
  if (pending_) {  // the previous upload must have left the buffer
    CVG_CK(cudaEventSynchronize(ev_));
    pending_ = false;
  }
  if (need > bytes_) {
    if (p_) cudaFreeHost(p_);
    p_ = nullptr;
    bytes_ = 0;
    CVG_CK(cudaHostAlloc(&p_, std::max<size_t>(need, 4096), cudaHostAllocDefault));
    bytes_ = std::max<size_t>(need, 4096);
  }
  if (!ev_) CVG_CK(cudaEventCreateWithFlags(&ev_, cudaEventDisableTiming));
  char* h = static_cast<char*>(p_);
  for (const Part& q : parts) {
    if (!q.bytes) continue;
    std::memcpy(h, q.src, q.bytes);
    CVG_CK(cudaMemcpyAsync(q.dst, h, q.bytes, cudaMemcpyHostToDevice, s));
    h += (q.bytes + 15) & ~size_t(15);
  }
  CVG_CK(cudaEventRecord(ev_, s));
  pending_ = true;
  return Status::Ok();
}

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

// int8 Gram items (k_gram_i8.cu): one 64-column block c as B, two 64-row blocks as the A halves, each half
// direct (the upper tile (a, c), a <= c) or transposed (the upper tile (c, a), a > c, computed as its
// transpose).  Column c starts with its needed tiles (a, c); a column with an odd count would leave a half
// unused, so odd columns are paired (c1 < c2) by moving the tile (c1, c2) into column c1 as a transposed half.
// Each column is then cut into halves: 128-aligned pairs (2i, 2i + 1) first (one TMA box), the rest in order.
// Every needed tile is produced exactly once; at most one half of the whole cover is unused when the tile
// count is odd (configs[1]: 36 tiles in 18 items; the 128-aligned tiling needed 20, four of them half below
// the diagonal).
std::vector<int2> i8_items(const std::vector<int2>& tiles, int nb) {
  std::vector<std::vector<std::pair<int, int>>> col(nb);  // (row block, mode 1 direct | 2 transposed)
  std::vector<std::vector<bool>> need(nb, std::vector<bool>(nb, false));
  for (const int2& t : tiles) {
    col[t.y].push_back({t.x, 1});
    need[t.x][t.y] = true;
  }
  std::vector<int> odd;
  for (int c = 0; c < nb; ++c)
    if (col[c].size() % 2) odd.push_back(c);
  std::vector<bool> done(odd.size(), false);
  for (size_t p = 0; p < odd.size(); ++p) {
    if (done[p]) continue;
    for (size_t q = p + 1; q < odd.size(); ++q) {
      const int c1 = odd[p], c2 = odd[q];
      if (done[q] || !need[c1][c2]) continue;
      auto& v = col[c2];
      for (size_t i = 0; i < v.size(); ++i)
        if (v[i].first == c1 && v[i].second == 1) {
          v.erase(v.begin() + (long)i);
          break;
        }
      col[c1].push_back({c2, 2});
      done[p] = done[q] = true;
      break;
    }
  }
  std::vector<int2> items;
  for (int c = 0; c < nb; ++c) {
    auto v = col[c];
    std::sort(v.begin(), v.end());
    std::vector<bool> taken(v.size(), false);
    auto emit = [&](size_t i, long j) {  // j < 0: half 1 unused
      const auto& h0 = v[i];
      const int a1 = j >= 0 ? v[(size_t)j].first : h0.first;
      const int m1 = j >= 0 ? v[(size_t)j].second : 0;
      items.push_back(make_int2(h0.first | (a1 << 16), c | (h0.second << 16) | (m1 << 18)));
      taken[i] = true;
      if (j >= 0) taken[(size_t)j] = true;
    };
    for (size_t i = 0; i + 1 < v.size(); ++i)
      if (!taken[i] && !taken[i + 1] && v[i].first % 2 == 0 && v[i + 1].first == v[i].first + 1) emit(i, (long)i + 1);
    long pend = -1;
    for (size_t i = 0; i < v.size(); ++i) {
      if (taken[i]) continue;
      if (pend < 0) {
        pend = (long)i;
      } else {
        emit((size_t)pend, (long)i);
        pend = -1;
      }
    }
    if (pend >= 0) emit((size_t)pend, -1);
  }
  return items;
}

std::vector<int2> gram_tiles(int64_t k, int64_t m, int64_t kp, int edge) {
  const int nt = (int)(kp / edge);
  const int tx = (int)((k - 1) / edge);  // last tile holding X columns
  const int to = (int)((k + m) / edge);  // tile holding the ones column
  std::vector<int2> t;
  for (int i = 0; i < nt; ++i)
    for (int j = i; j < nt; ++j)
      if (i <= tx || j == i || j == to) t.push_back(make_int2(i, j));
  return t;
}



const double* TreeProgram::emit(const std::vector<const double*>& leaves, int a, int b, int depth, double* root_dst,
                                std::vector<std::vector<TreeOp>>& by_depth, int64_t kp) {
  if ((int)by_depth.size() <= depth) by_depth.resize(depth + 1);
  if (b - a <= 1 && !root_dst) return leaves[a];  // interior leaf: read in place
  double* out = root_dst ? root_dst : scratch_.as<double>() + (next_slot_++) * kp * kp;
  TreeOp op{};
  op.d = out;
  op.size = b - a;
  int cnt = 0;
  // the node's frontier kTreeFanDepth levels down (S(a,b) = S(a,mid) + S(mid,b)), left to right: leaves, or
  // nodes evaluated by ops one level deeper
  std::function<void(int, int, int)> frontier = [&](int lo, int hi, int d) {
    if (hi - lo == 1) {
      op.in[cnt++] = leaves[lo];
    } else if (d == kTreeFanDepth) {
      op.in[cnt++] = emit(leaves, lo, hi, depth + 1, nullptr, by_depth, kp);
    } else {
      const int mid = lo + (hi - lo) / 2;
      frontier(lo, mid, d + 1);
      frontier(mid, hi, d + 1);
    }
  };
  if (b > a) frontier(a, b, 0);
  by_depth[depth].push_back(op);
  return out;
}

Status TreeProgram::build(const std::vector<TreeGroup>& groups, int64_t kp, cudaStream_t s) {
  int64_t slots = 0;  // internal nodes other than each group's root
  for (const auto& g : groups) slots += std::max<int64_t>((int64_t)g.leaves.size() - 2, 0);
  CVG_TRY(scratch_.ensure(sizeof(double) * std::max<int64_t>(slots, 1) * kp * kp));
  next_slot_ = 0;
  std::vector<std::vector<TreeOp>> by_depth;
  for (const auto& g : groups) emit(g.leaves, 0, (int)g.leaves.size(), 0, g.dst, by_depth, kp);
  flat_.clear();
  level_off_.assign(1, 0);
  for (int d = (int)by_depth.size() - 1; d >= 0; --d) {  // deepest level first
    if (by_depth[d].empty()) continue;
    flat_.insert(flat_.end(), by_depth[d].begin(), by_depth[d].end());
    level_off_.push_back((int)flat_.size());
  }
  CVG_TRY(ops_d_.ensure(sizeof(TreeOp) * std::max<size_t>(flat_.size(), 1)));
  if (!flat_.empty())
    CVG_TRY(stage_.upload({{flat_.data(), sizeof(TreeOp) * flat_.size(), ops_d_.as<void>()}}, s));
  return Status::Ok();
}

Status TreeProgram::run(cvg_context* ctx, const int2* tiles, int ntiles, int64_t kp) const {
  for (int l = 0; l + 1 < (int)level_off_.size(); ++l) {
    {
      Timed t(ctx, kTree);
      launch_tree_ops(ops_d_.as<TreeOp>() + level_off_[l], level_off_[l + 1] - level_off_[l], kp, tiles, ntiles,
                       ctx->stream);
    }
    ctx->launches += 1;
    CVG_CK(cudaGetLastError());
  }
  return Status::Ok();
}

// Rows per segment: a fixed constant per dtype (never a function of the GPU
// count, so sums stay bit-identical across world sizes).  CVG_CHUNK_ROWS
// overrides it for tuning experiments (rounded to the plan's row step).

// fp32 operand kind: the scaled fp16 split on kind::f16 (default) or, with
// CVG_FP32_KIND=tf32, the 3xTF32 split on kind::tf32 (k_gram_tf32.cu; A/B tests).
bool Plan::fp32_tf32() {
  static const bool v = [] {
    const char* e = std::getenv("CVG_FP32_KIND");
    return e && std::string(e) == "tf32";
  }();
  return v;
}

// fp64 operand kind: exact int8 digit slices on tcgen05 kind::i8 (default; k_gram_i8.cu) or,
// with CVG_FP64_KIND=dmma, the fp64 DMMA Gram (k_gram_f64.cu).  Read at plan creation, so one
// process can A/B both.
static bool fp64_i8_env() {
  const char* e = std::getenv("CVG_FP64_KIND");
  return !(e && std::string(e) == "dmma");
}
static int i8_slices_env() {  // base-256 digits: 6 (48 bits, default) or 5 (40 bits)
  const char* e = std::getenv("CVG_I8_SLICES");
  return e && std::atoi(e) == 5 ? 5 : 6;
}
// Row-sample stride of the int8 path's segment maxima (CVG_I8_SAMPLE; 1 = every row, one exact pass).
static int i8_sample_env() {
  const char* e = std::getenv("CVG_I8_SAMPLE");
  const int v = e ? std::atoi(e) : 16;
  return v >= 1 ? v : 16;
}

// The fp16 path's row group G (one exponent per group and column, one fp32 TMEM
// chunk) is also the fold padding and segment alignment.  Largest of 256 / 128 /
// 64 whose padding stays within 1/8 of the 64-row minimum; a function of the
// global fold sizes only, so every rank plan picks the same G.
void Plan::choose_row_step() {
  row_step_ = kRowStep;
  if (i8_) row_step_ = 64;  // one int8 Gram stage
  if (!f16_path()) return;
  auto padded = [&](int64_t g) {
    int64_t t = 0;
    for (int64_t c : counts_) t += round_up(std::max<int64_t>(c, 1), g);
    return t;
  };
  const int64_t base = padded(64);
  row_step_ = 64;
  for (int64_t g : {256, 128})
    if (padded(g) * 8 <= base * 9) {
      row_step_ = g;
      break;
    }
}

int64_t Plan::chunk_rows() const {
  static const int64_t env = [] {
    const char* v = std::getenv("CVG_CHUNK_ROWS");
    const long long r = v ? std::atoll(v) : 0;
    return (int64_t)(r > 0 ? r : 0);
  }();
  if (env > 0) {
    int64_t r = round_up(env, row_step_);
    // int8 digits: exact int32 TMEM sums need slices * 2^14 * rows < 2^31 (21,845 rows at 6 digits)
    if (i8_path()) r = std::min(r, ((INT32_MAX / ((int64_t)slices_ << 14)) / row_step_) * row_step_);
    return r;
  }
  return round_up(i8_path() ? kChunkRowsI8 : dtype_ == 0 ? kChunkRows : f16_path() ? kChunkRowsF32 : kChunkRowsTf32,
                  row_step_);
}

// Rows per segment of a fold of `count` rows: the fold is cut into
// ceil(padded / chunk_rows()) segments of equal size (rounded up to the row step), so
// no fold ends in a sliver segment and the Gram's CTAs carry even work.
int64_t Plan::seg_rows(int64_t count) const {
  const int64_t padded = round_up(count, row_step_), chunk = chunk_rows();
  const int64_t nseg = std::max<int64_t>(1, (padded + chunk - 1) / chunk);
  return std::max<int64_t>(row_step_, round_up((padded + nseg - 1) / nseg, row_step_));
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
  if (n > INT32_MAX) return Status::Err(4, "more than 2^31 - 1 samples per plan is unsupported (int32 row indices)");
  if (k < 1 || m < 1) return Status::Err(1, "x and y must each have at least one column");
  if (validate) {
    if (p < 2) return Status::Err(2, "fold count must be at least 2, got " + std::to_string(p));
    if ((int64_t)p > n)
      return Status::Err(2, "fold count " + std::to_string(p) + " exceeds sample count " + std::to_string(n));
  }
  if (fb < 0 || fe > p || fb > fe) return Status::Err(4, "owned fold range is outside [0, p]");
  rank_mode_ = false;
  emits_ = true;
  seg_lo_ = seg_hi_ = -1;
  kp_ = padded_cols(k, m, dtype);
  tiles_ = gram_tiles(k, m, kp_);
  tiles128_ = dtype == 1 ? gram_tiles(k, m, kp_, kTileF32) : std::vector<int2>{};
  i8_ = dtype == 0 && fp64_i8_env();  // fp32 inputs: the scaled fp16 split (or 3xTF32), never int8 digits
  slices_ = i8_slices_env();
  sample_ = i8_sample_env();
  tilesq_.clear();
  if (i8_) {  // 128 x 64 int8-Gram items covering the needed upper 64-tiles exactly once
    tilesq_ = i8_items(tiles_, (int)(kp_ / kTile));
    CVG_TRY(tilesq_d_.ensure(tilesq_.size() * sizeof(int2)));
    CVG_CK(cudaMemcpyAsync(tilesq_d_.as<int2>(), tilesq_.data(), tilesq_.size() * sizeof(int2), cudaMemcpyHostToDevice,
                           ctx->stream));
  }
  // output tiles, the diagonal ones first (launch_products sends the rest to the warp-owned kernel)
  out_tiles_.clear();
  for (const int2& t : tiles_)
    if ((int64_t)t.x * kTile < k && t.x == t.y) out_tiles_.push_back(t);
  out_ndiag_ = (int)out_tiles_.size();
  for (const int2& t : tiles_)
    if ((int64_t)t.x * kTile < k && t.x != t.y) out_tiles_.push_back(t);
  CVG_CK(cudaSetDevice(ctx->device));
  CVG_TRY(tiles_d_.ensure(tiles_.size() * sizeof(int2)));
  CVG_TRY(out_tiles_d_.ensure(out_tiles_.size() * sizeof(int2)));
  CVG_CK(cudaMemcpyAsync(tiles_d_.as<int2>(), tiles_.data(), tiles_.size() * sizeof(int2), cudaMemcpyHostToDevice,
                         ctx->stream));
  CVG_CK(cudaMemcpyAsync(out_tiles_d_.as<int2>(), out_tiles_.data(), out_tiles_.size() * sizeof(int2),
                         cudaMemcpyHostToDevice, ctx->stream));
  if (!tiles128_.empty()) {
    CVG_TRY(tiles128_d_.ensure(tiles128_.size() * sizeof(int2)));
    CVG_CK(cudaMemcpyAsync(tiles128_d_.as<int2>(), tiles128_.data(), tiles128_.size() * sizeof(int2),
                           cudaMemcpyHostToDevice, ctx->stream));
  }
  CVG_TRY(local_.ensure(sizeof(double) * kp_ * kp_));
  CVG_TRY(shift_.ensure(sizeof(double) * kp_));
  CVG_CK(cudaMemsetAsync(shift_.as<void>(), 0, sizeof(double) * kp_, ctx->stream));  // ones/padding columns
  CVG_TRY(flag_.ensure(sizeof(int)));
  return Status::Ok();
}

Status Plan::create_rank(cvg_context* ctx, int dtype, int64_t n, int64_t k, int64_t m, int32_t p, int32_t rank,
                         int32_t world) {
  if (world < 1 || rank < 0 || rank >= world) return Status::Err(4, "rank outside [0, world)");
  CVG_TRY(create(ctx, dtype, n, k, m, p, 0, p, true));
  rank_mode_ = true;
  rank_ = rank;
  world_ = world;
  return Status::Ok();
}

void Plan::assign_rank() {
  int32_t lo = 0, hi = world_, a = 0, b = p_;
  int64_t s0 = -1, s1 = -1;
  int32_t glo = 0, ghi = 0;
  while (hi - lo > 1) {
    const int32_t rmid = lo + (hi - lo) / 2;
    if (b - a == 1) {  // one fold, several ranks: split its segments
      if (s0 < 0) {
        s0 = 0;
        const int64_t sr = seg_rows(counts_[a]);
        s1 = (round_up(counts_[a], row_step_) + sr - 1) / sr;
        glo = lo;
        ghi = hi;
      }
      const int64_t smid = s0 + (s1 - s0) / 2;
      if (rank_ < rmid) {
        hi = rmid;
        s1 = smid;
      } else {
        lo = rmid;
        s0 = smid;
      }
    } else {
      const int32_t fmid = a + (b - a) / 2;
      if (rank_ < rmid) {
        hi = rmid;
        b = fmid;
      } else {
        lo = rmid;
        a = fmid;
      }
    }
  }
  fb_ = a;
  fe_ = b;
  seg_lo_ = s0;
  seg_hi_ = s1;
  group_lo_ = glo;
  group_hi_ = ghi;
  emits_ = s0 < 0 || rank_ == glo;
}

Status Plan::bind_labels(const int32_t* d_labels, bool validate, bool require_scalable) {
  src_n_ = n_;
  cudaStream_t s = ctx_->stream;
  const int64_t tile_rows = bucket_tile_rows(n_, p_);
  const int64_t ntiles = (n_ + tile_rows - 1) / tile_rows;
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
  small_ = false;
  if (validate) {
    for (int32_t f = 0; f < p_; ++f)
      if (counts_[f] == 0) return Status::Err(2, "fold " + std::to_string(f + 1) + " is empty");
    if (require_scalable)
      for (int32_t f = 0; f < p_; ++f)
        if (n_ - counts_[f] < 2)
          return Status::Err(3, "fold " + std::to_string(f + 1) + " leaves a training partition of " +
                                    std::to_string(n_ - counts_[f]) + " rows; scaling needs at least 2");
  }
  choose_row_step();
  if (rank_mode_) assign_rank();
  small_ = false;
  if (dtype_ == 0 && !rank_mode_ && fb_ == 0 && fe_ == p_ && small_folds_enabled()) {
    int64_t mx = 0;
    for (int32_t f = 0; f < p_; ++f) mx = std::max(mx, counts_[f]);
    small_ = mx <= kSmallFoldRows;
  }
  {
    // The segment plan (Z layout, segment list, block -> segment table, tree ops, fold pointers and their
    // device copies) is a function of the fold sizes and this plan's window only: binding another
    // partitioning with the same sizes (repeated CV over equal-sized folds) reuses it, which takes the host
    // planning and its uploads out of the gap between the fold counts' read-back and the scatter.
    PlanKey key{counts_, fb_, fe_, seg_lo_, seg_hi_, row_step_, small_, i8_path()};
    if (!(planned_ && key == plan_key_)) {
      planned_ = false;
      CVG_TRY(plan_segments());
      plan_key_ = std::move(key);
      planned_ = true;
    }
  }
  CVG_CK(cudaMemsetAsync(src_row_.as<void>(), 0xff, sizeof(int64_t) * std::max<int64_t>(zrows_, 1), s));
  {
    Timed t(ctx_, kBucket);
    const int64_t win_lo = seg_lo_ >= 0 ? seg_lo_ * seg_rows(counts_[fb_]) : 0;
    const int64_t win_hi = seg_lo_ >= 0 ? win_lo + zrows_ : INT64_MAX;
    launch_scatter(d_labels, n_, p_, fb_, fe_, tile_counts_.as<int32_t>(), zbase_d_.as<int64_t>(), win_lo, win_hi,
                   src_row_.as<int64_t>(), zrows_, s);
  }
  CVG_TRY(count_launch());
  bound_ = true;
  return Status::Ok();
}

// CVG_SMALL_FOLDS=0 keeps per-fold Gram partials even when every fold is tiny (A/B tests).
bool Plan::small_fold_mode(int dtype, const std::vector<int64_t>& counts) {
  if (dtype != 0 || !small_folds_enabled()) return false;
  int64_t mx = 0;
  for (int64_t c : counts) mx = std::max(mx, c);
  return mx <= kSmallFoldRows;
}

bool Plan::small_folds_enabled() {
  static const bool on = [] {
    const char* v = std::getenv("CVG_SMALL_FOLDS");
    return !(v && v[0] == '0');
  }();
  return on;
}

Status Plan::bind_rows(const int64_t* rows, int64_t nrows, int64_t n_src) {
  if (p_ != 1 || fb_ != 0 || fe_ != 1) return Status::Err(4, "bind_rows needs a single-fold plan");
  small_ = false;
  src_n_ = n_src < 0 ? n_ : n_src;
  if (src_n_ > INT32_MAX) return Status::Err(4, "bind_rows: source matrices beyond 2^31 - 1 rows are unsupported");
  for (int64_t i = 0; i < nrows; ++i)
    if (rows[i] < 0 || rows[i] >= src_n_) return Status::Err(4, "bind_rows: row index outside the source matrix");
  counts_.assign(1, nrows);
  choose_row_step();
  planned_ = false;
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
  if (small_) {
    // Small-fold mode: folds packed back to back (no per-fold padding); segments are
    // equal fixed-size row chunks of Z regardless of fold boundaries (they only feed
    // the whole-data Gram); each fold's own Gram is formed in the epilogue.
    int64_t rows = 0;
    for (int32_t f = fb_; f < fe_; ++f) {
      fold_zbase_.push_back(rows);
      rows += counts_[f];
      fold_seg_begin_.push_back(0);
    }
    zrows_ = round_up(std::max<int64_t>(rows, 1), kRowStep);
    const int64_t chunk = seg_rows(zrows_);
    for (int64_t off = 0; off < zrows_; off += chunk)
      segs_.push_back(GramTask{off, std::min<int64_t>(chunk, zrows_ - off)});
  }
  for (int32_t f = fb_; f < fe_ && !small_; ++f) {
    const int64_t padded = round_up(counts_[f], row_step_);
    const int64_t chunk = seg_rows(counts_[f]);
    // Owned window of the fold's bucketed rows: all of it, or (shared fold) segments [seg_lo_, seg_hi_).
    const int64_t w0 = seg_lo_ >= 0 ? std::min(padded, seg_lo_ * chunk) : 0;
    const int64_t w1 = seg_lo_ >= 0 ? std::min(padded, seg_hi_ * chunk) : padded;
    fold_zbase_.push_back(zrows_);
    for (int64_t off = w0; off < w1; off += chunk)
      segs_.push_back(GramTask{zrows_ + (off - w0), std::min<int64_t>(chunk, w1 - off)});
    zrows_ += w1 - w0;
    fold_seg_begin_.push_back((int32_t)segs_.size());
  }
  const int nown = fe_ - fb_;
  cudaStream_t s = ctx_->stream;
  CVG_TRY(zbase_d_.ensure(sizeof(int64_t) * std::max(nown, 1)));
  CVG_TRY(src_row_.ensure(sizeof(int64_t) * std::max<int64_t>(zrows_, 1)));
  if (dtype_ == 1 && !i8_path()) {  // blocked-transposed hi / lo operands for the tcgen05 Gram (fp16 or TF32)
    const size_t e = f16_path() ? 2 : 4;
    CVG_TRY(zt_hi_.ensure(e * std::max<int64_t>(zrows_, row_step_) * kp_));
    CVG_TRY(zt_lo_.ensure(e * std::max<int64_t>(zrows_, row_step_) * kp_));
    if (f16_path()) CVG_TRY(unscale_.ensure(sizeof(float) * std::max<int64_t>(zrows_ / row_step_, 1) * kp_));
  } else if (i8_path()) {  // int8 digit slices, per-(segment, column) exponents, 64-row block -> segment
    CVG_TRY(zq_.ensure((size_t)slices_ * std::max<int64_t>(zrows_, 64) * kp_));
    CVG_TRY(segmax_.ensure(sizeof(unsigned long long) * std::max<size_t>(segs_.size(), 1) * kp_));
    CVG_TRY(ovf_.ensure(sizeof(int) * std::max<size_t>(segs_.size(), 1)));
    std::vector<int> bs(std::max<int64_t>(zrows_ / 64, 1), 0);
    for (size_t sgi = 0; sgi < segs_.size(); ++sgi)
      for (int64_t r = segs_[sgi].zrow; r < segs_[sgi].zrow + segs_[sgi].rows; r += 64) bs[r / 64] = (int)sgi;
    CVG_TRY(blkseg_.ensure(sizeof(int) * bs.size()));
    CVG_TRY(blkseg_stage_.upload({{bs.data(), sizeof(int) * bs.size(), blkseg_.as<void>()}}, s));
  } else {
    CVG_TRY(z_.ensure(sizeof(double) * std::max<int64_t>(zrows_, 1) * kp_));
  }
  CVG_TRY(part_.ensure(sizeof(double) * std::max<size_t>(segs_.size(), 1) * kp_ * kp_));
  CVG_TRY(segs_d_.ensure(sizeof(GramTask) * std::max<size_t>(segs_.size(), 1)));
  CVG_TRY(nval_d_.ensure(sizeof(int64_t) * std::max(nown, 1)));
  CVG_TRY(seg_stage_.upload({{fold_zbase_.data(), sizeof(int64_t) * nown, zbase_d_.as<void>()},
                             {counts_.data() + fb_, sizeof(int64_t) * nown, nval_d_.as<void>()},
                             {segs_.data(), sizeof(GramTask) * segs_.size(), segs_d_.as<void>()}},
                            s));
  if (small_) {  // no per-fold Grams: the plan's node is the tree over all chunks
    TreeGroup g{{}, local_.as<double>()};
    for (size_t sgi = 0; sgi < segs_.size(); ++sgi) g.leaves.push_back(part_.as<double>() + (int64_t)sgi * kp_ * kp_);
    CVG_TRY(fold_tree_.build({}, kp_, s));
    CVG_TRY(local_tree_.build({g}, kp_, s));
    fold_ptrs_.assign(nown, nullptr);
    CVG_TRY(foldptr_d_.ensure(sizeof(void*) * std::max(nown, 1)));
    CVG_TRY(ptr_stage_.upload({{fold_ptrs_.data(), sizeof(void*) * nown, foldptr_d_.as<void>()}}, s));
    return Status::Ok();
  }
  // Fold Gram pointers: the segment partial itself for single-segment folds,
  // otherwise a fixed-order sum of its segments into foldbuf (K4, phase 1).
  int nmulti = 0;
  for (int f = 0; f < nown; ++f)
    if (fold_seg_begin_[f + 1] - fold_seg_begin_[f] != 1) ++nmulti;
  CVG_TRY(foldbuf_.ensure(sizeof(double) * std::max(nmulti, 1) * kp_ * kp_));
  fold_ptrs_.assign(nown, nullptr);
  std::vector<TreeGroup> phase1;
  if (seg_lo_ >= 0) {
    // Shared fold: this plan's node is the sum over its segment range; the
    // fold's full Gram is rebuilt from the group's partials in finish().
    TreeGroup g{{}, local_.as<double>()};
    for (size_t sgi = 0; sgi < segs_.size(); ++sgi) g.leaves.push_back(part_.as<double>() + (int64_t)sgi * kp_ * kp_);
    phase1.push_back(std::move(g));
    fold_ptrs_[0] = foldbuf_.as<double>();
    CVG_TRY(fold_tree_.build(phase1, kp_, s));
    CVG_TRY(local_tree_.build({}, kp_, s));
    CVG_TRY(foldptr_d_.ensure(sizeof(void*)));
    CVG_TRY(ptr_stage_.upload({{fold_ptrs_.data(), sizeof(void*), foldptr_d_.as<void>()}}, s));
    return Status::Ok();
  }
  int slot = 0;
  for (int f = 0; f < nown; ++f) {
    const int a = fold_seg_begin_[f], b = fold_seg_begin_[f + 1];
    if (b - a == 1) {
      fold_ptrs_[f] = part_.as<double>() + (int64_t)a * kp_ * kp_;
    } else {
      double* dst = foldbuf_.as<double>() + (int64_t)slot++ * kp_ * kp_;
      fold_ptrs_[f] = dst;
      TreeGroup g{{}, dst};
      for (int sgi = a; sgi < b; ++sgi) g.leaves.push_back(part_.as<double>() + (int64_t)sgi * kp_ * kp_);
      phase1.push_back(std::move(g));
    }
  }
  CVG_TRY(fold_tree_.build(phase1, kp_, s));
  // Phase 2: this plan's node of the fold tree, over the owned folds in order.
  std::vector<TreeGroup> phase2{TreeGroup{std::vector<const double*>(fold_ptrs_.begin(), fold_ptrs_.end()),
                                          local_.as<double>()}};
  CVG_TRY(local_tree_.build(phase2, kp_, s));
  CVG_TRY(foldptr_d_.ensure(sizeof(void*) * std::max(nown, 1)));
  CVG_TRY(ptr_stage_.upload({{fold_ptrs_.data(), sizeof(void*) * nown, foldptr_d_.as<void>()}}, s));
  return Status::Ok();
}

Status Plan::gram(const void* d_x, int64_t ldx, const void* d_y, int64_t ldy, const double* host_shift,
                  const double* dev_shift, const int64_t* d_row_map, int64_t n_compact) {
  if (!bound_) return Status::Err(4, "plan has no bound partitioning");
  cudaStream_t s = ctx_->stream;
  const int64_t* rows = src_row_.as<int64_t>();
  int64_t nsrc = src_n_;
  if (d_row_map) {
    // compacted inputs: K1 reads compact row map[src_row[r]]; row 0 may be absent, so the shift is explicit
    if (!host_shift && !dev_shift) return Status::Err(4, "a row-mapped gram needs an explicit shift");
    CVG_TRY(src_map_.ensure(sizeof(int64_t) * std::max<int64_t>(zrows_, 1)));
    CVG_CK(cudaMemsetAsync(flag_.as<void>(), 0, sizeof(int), s));
    launch_remap_rows(src_row_.as<int64_t>(), zrows_, d_row_map, n_, n_compact, src_map_.as<int64_t>(),
                      flag_.as<int>(), s);
    CVG_TRY(count_launch());
    int bad = 0;
    CVG_CK(cudaMemcpyAsync(&bad, flag_.as<int>(), sizeof bad, cudaMemcpyDeviceToHost, s));
    CVG_CK(cudaStreamSynchronize(s));
    if (bad) return Status::Err(4, "row map does not cover every row of the owned folds");
    rows = src_map_.as<int64_t>();
    nsrc = n_compact;
  }
  double* shift = shift_.as<double>();
  if (dev_shift) {
    CVG_CK(cudaMemcpyAsync(shift, dev_shift, sizeof(double) * w_, cudaMemcpyDeviceToDevice, s));
  } else if (host_shift) {
    CVG_TRY(shift_stage_.upload({{host_shift, sizeof(double) * w_, shift}}, s));
  } else {
    Timed t(ctx_, kReorder);
    launch_shift_from_row0(dtype_, d_x, d_y, k_, m_, shift, s);
    CVG_TRY(count_launch());
  }
  CVG_CK(cudaMemsetAsync(flag_.as<void>(), 0, sizeof(int), s));
  if (dtype_ == 1 && !i8_path()) {
    // fp32: K1H / K1T (bucket, shift, split, blocked transpose) then the tcgen05 Gram.
    if (zrows_ > 0) {
      {
        Timed t(ctx_, kReorder);
        if (f16_path()) {
          if (!launch_reorder_split_h(dtype_, d_x, ldx, d_y, ldy, k_, m_, rows, zrows_, kp_, 0, kp_, nsrc, shift,
                                      (int)row_step_, zt_hi_.as<void>(), zt_lo_.as<void>(), unscale_.as<float>(),
                                      flag_.as<int>(), s))
            return Status::Err(5, "cuTensorMapEncodeTiled unavailable or rejected the operand layout");
        } else
          launch_reorder_split_t(dtype_, d_x, ldx, d_y, ldy, k_, m_, rows, zrows_, kp_, 0, kp_, shift,
                                 zt_hi_.as<float>(), zt_lo_.as<float>(), flag_.as<int>(), s);
      }
      CVG_TRY(count_launch());
    }
    if (!segs_.empty()) {
      bool ok;
      {
        Timed t(ctx_, kGram);
        ok = f16_path()
                 ? launch_gram_f16s(zt_hi_.as<void>(), zt_lo_.as<void>(), unscale_.as<float>(), (int)row_step_,
                                    zrows_, kp_, segs_d_.as<GramTask>(), (int64_t)segs_.size(),
                                    tiles128_d_.as<int2>(), (int)tiles128_.size(), part_.as<double>(), s)
                 : launch_gram_tf32(zt_hi_.as<float>(), zt_lo_.as<float>(), zrows_, kp_, segs_d_.as<GramTask>(),
                                    (int64_t)segs_.size(), tiles128_d_.as<int2>(), (int)tiles128_.size(),
                                    part_.as<double>(), 3, s);
      }
      if (!ok) return Status::Err(5, "cuTensorMapEncodeTiled unavailable or rejected the operand layout");
      CVG_TRY(count_launch());
    }
  } else if (i8_path()) {
    // fp64 on int8 digit slices: segment exponents, K1Q, tcgen05 kind::i8 Gram.
    if (zrows_ > 0) {
      CVG_CK(cudaMemsetAsync(segmax_.as<void>(), 0, sizeof(unsigned long long) * segs_.size() * kp_, s));
      if (sample_ > 1) CVG_CK(cudaMemsetAsync(ovf_.as<void>(), 0, sizeof(int) * segs_.size(), s));
    }
    overlapped_ = false;
    if (zrows_ > 0 && !segs_.empty() && !tilesq_.empty() && i8_overlap_enabled() && !ctx_->overlap_failed) {
      CVG_TRY(i8_overlapped(d_x, ldx, d_y, ldy, rows, nsrc));
    } else {
      if (zrows_ > 0) CVG_TRY(i8_prep(d_x, ldx, d_y, ldy, rows, nsrc, 0, kp_, false));
      CVG_TRY(i8_gram(tilesq_d_.as<int2>(), (int)tilesq_.size()));
    }
    CVG_TRY(i8_flags_to_host());
    CVG_TRY(gram_trees());
    CVG_TRY(i8_exact_pass(d_x, ldx, d_y, ldy, rows, nsrc));
    return poison_local();
  } else {
    // fp64: K1 builds the fold-bucketed, shifted copy Z.  (Gathering X rows
    // straight into the Gram's shared-memory stages, or overlapping K1 with K2
    // inside one persistent launch, were both measured slower — DESIGN.md §8.)
    if (zrows_ > 0) {
      {
        Timed t(ctx_, kReorder);
        launch_reorder(dtype_, d_x, ldx, d_y, ldy, k_, m_, rows, zrows_, kp_, 0, kp_, nsrc, shift,
                       z_.as<double>(), flag_.as<int>(), s);
      }
      CVG_TRY(count_launch());
    }
    if (!segs_.empty()) {
      {
        Timed t(ctx_, kGram);
        launch_gram_f64(z_.as<double>(), kp_, zrows_, segs_d_.as<GramTask>(), (int64_t)segs_.size(), tiles_d_.as<int2>(),
                        (int)tiles_.size(), part_.as<double>(), s);
      }
      CVG_TRY(count_launch());
    }
  }
  CVG_TRY(gram_trees());
  return poison_local();
}

Status Plan::poison_local() {
  launch_poison_if_flag(flag_.as<int>(), local_.as<double>(), ctx_->stream);
  return count_launch();
}

// One int8-path preparation pass over Z columns [c0, c1): segment maxima (a row sample of stride
// sample_, or -- exact pass -- every row of the segments flagged in ovf_, on top of the sampled max),
// then K1Q (sampled pass: out-of-range values flag their segment; exact pass: the non-finite flag).
Status Plan::i8_prep(const void* d_x, int64_t ldx, const void* d_y, int64_t ldy, const int64_t* rows, int64_t nsrc,
                     int64_t c0, int64_t c1, bool exact) {
  cudaStream_t s = ctx_->stream;
  const bool sampled = sample_ > 1;
  {
    Timed t(ctx_, kReorder);
    launch_segmax(dtype_, d_x, ldx, d_y, ldy, k_, m_, rows, segs_d_.as<GramTask>(), (int64_t)segs_.size(),
                  max_seg_rows(), kp_, c0, c1, nsrc, shift_.as<double>(), exact ? 1 : sample_,
                  exact ? ovf_.as<int>() : nullptr, segmax_.as<unsigned long long>(), s);
  }
  CVG_TRY(count_launch());
  {
    Timed t(ctx_, kReorder);
    if (!launch_reorder_q(dtype_, slices_, d_x, ldx, d_y, ldy, k_, m_, rows, zrows_, kp_, c0, c1, nsrc,
                          shift_.as<double>(), blkseg_.as<int>(), segmax_.as<unsigned long long>(), sampled ? 1 : 0,
                          sampled && !exact ? ovf_.as<int>() : nullptr, zq_.as<int8_t>(), flag_.as<int>(), s))
      return Status::Err(5, "cuTensorMapEncodeTiled unavailable or rejected the operand layout");
  }
  return count_launch();
}

// The int8 Gram's tail-split workspace (k_gram_i8.cu): sized for one part per SM.  CVG_I8_SPLIT=0 disables it.
Status Plan::ensure_split_ws() {
  const char* v = std::getenv("CVG_I8_SPLIT");
  if (v && v[0] == '0') {
    split_ws_.release();
    split_cnt_.release();
    return Status::Ok();
  }
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx_->device);
  CVG_TRY(split_ws_.ensure(gram_i8_split_ws_bytes(sms)));
  return split_cnt_.ensure(sizeof(unsigned) * (size_t)sms);
}

Status Plan::i8_gram(const int2* tiles, int ntiles) {
  if (segs_.empty() || ntiles == 0) return Status::Ok();
  bool ok;
  {
    Timed t(ctx_, kGram);
    CVG_TRY(ensure_split_ws());
    ok = launch_gram_i8(slices_, zq_.as<int8_t>(), segmax_.as<unsigned long long>(), sample_ > 1 ? 1 : 0, zrows_, kp_,
                        segs_d_.as<GramTask>(), (int64_t)segs_.size(), tiles, ntiles, part_.as<double>(),
                        ctx_->stream, 0, 0, 0, nullptr, nullptr, split_ws_.as<int32_t>(), split_cnt_.as<unsigned>(),
                        min_seg_rows());
  }
  if (!ok) return Status::Err(5, "cuTensorMapEncodeTiled unavailable or rejected the operand layout");
  return count_launch();
}

// K1Q's HBM-bound cut runs beside the tensor-bound Gram instead of before it when the segments are long
// enough (>= 1024 rows on average: short segments pay the per-item acquire and keep the 16-column drain)
// CVG_I8_OVERLAP=0 keeps the serial schedule, =1 forces the overlap.  Read per call (tests A/B both).
bool Plan::i8_overlap_enabled() const {
  const char* v = std::getenv("CVG_I8_OVERLAP");
  if (v && (v[0] == '0' || v[0] == '1')) return v[0] == '1';
  if (segs_.empty() || zrows_ / (int64_t)segs_.size() < 1024) return false;
  // ... and with at least ~2.5 waves of Gram items: below that (c1 on 8 GPUs: 12 folds = 216 items) the Gram's
  // first wave only waits for the cut (measured per rank: 0.78-0.82 ms together, 0.75-0.77 ms back to back)
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx_->device);
  return (int64_t)segs_.size() * (int64_t)tilesq_.size() * 2 >= 5 * (int64_t)sms;
}

// The cut beside the Gram.  The aux stream runs the direct-store cut on one persistent CTA per SM (Z order);
// the main stream runs the lean Gram, whose items (segment-major, the same order) each wait for their
// segment's published block count.  Same digits, same MMAs, same drain: bit-identical to the serial path.
Status Plan::i8_overlapped(const void* d_x, int64_t ldx, const void* d_y, int64_t ldy, const int64_t* rows,
                           int64_t nsrc) {
  cudaStream_t s = ctx_->stream;
  CVG_TRY(ctx_->ensure_aux_stream());
  CVG_TRY(ensure_split_ws());
  const bool sampled = sample_ > 1;
  const size_t nseg = segs_.size();
  CVG_TRY(seg_ready_.ensure(sizeof(unsigned) * (nseg + 1)));
  CVG_CK(cudaMemsetAsync(seg_ready_.as<void>(), 0, sizeof(unsigned) * (nseg + 1), s));
  {
    Timed t(ctx_, kReorder);
    launch_segmax(dtype_, d_x, ldx, d_y, ldy, k_, m_, rows, segs_d_.as<GramTask>(), (int64_t)nseg, max_seg_rows(), kp_,
                  0, kp_, nsrc, shift_.as<double>(), sample_, nullptr, segmax_.as<unsigned long long>(), s);
  }
  CVG_TRY(count_launch());
  cudaEvent_t ev0 = ctx_->stream_event(0), ev1 = ctx_->stream_event(1);
  CVG_CK(cudaEventRecord(ev0, s));
  CVG_CK(cudaStreamWaitEvent(ctx_->aux_stream, ev0, 0));
  // CVG_I8_OVERLAP_FAULT=1 (tests): the cut publishes nothing, so the Gram's wait must time out and the
  // serial redo below must produce the same bits
  const char* fv = std::getenv("CVG_I8_OVERLAP_FAULT");
  const bool fault = fv && fv[0] == '1';
  bool ok;
  {
    Timed t(ctx_, kGram);  // the overlapped region: cut and Gram
    ok = launch_reorder_q(dtype_, slices_, d_x, ldx, d_y, ldy, k_, m_, rows, zrows_, kp_, 0, kp_, nsrc,
                          shift_.as<double>(), blkseg_.as<int>(), segmax_.as<unsigned long long>(), sampled ? 1 : 0,
                          sampled ? ovf_.as<int>() : nullptr, zq_.as<int8_t>(), flag_.as<int>(), ctx_->aux_stream, 0,
                          -1, 0, 1, fault ? nullptr : seg_ready_.as<unsigned>());
    CVG_CK(cudaEventRecord(ev1, ctx_->aux_stream));
    ok = ok && launch_gram_i8(slices_, zq_.as<int8_t>(), segmax_.as<unsigned long long>(), sampled ? 1 : 0, zrows_, kp_,
                              segs_d_.as<GramTask>(), (int64_t)nseg, tilesq_d_.as<int2>(), (int)tilesq_.size(),
                              part_.as<double>(), s, 0, 0, 1, seg_ready_.as<unsigned>(),
                              reinterpret_cast<int*>(seg_ready_.as<unsigned>() + nseg), split_ws_.as<int32_t>(),
                              split_cnt_.as<unsigned>(), min_seg_rows());
    CVG_CK(cudaStreamWaitEvent(s, ev1, 0));
  }
  if (!ok) return Status::Err(5, "cuTensorMapEncodeTiled unavailable or rejected the operand layout");
  overlapped_ = true;
  return count_launch(2);
}

// Sampled exponents only: if any segment held a value beyond 2x its sampled max (or a nonzero value
// in a column whose sample was all zero), redo those segments' maxima over every row, then K1Q and the
// Gram for all columns (unflagged segments reproduce the same bits) and the trees.  The decision is per
// segment and depends on the segment's rows only, so results stay bit-identical across GPU counts.
Status Plan::i8_exact_pass(const void* d_x, int64_t ldx, const void* d_y, int64_t ldy, const int64_t* rows,
                           int64_t nsrc) {
  if (!flags_pending_) return Status::Ok();
  flags_pending_ = false;
  // wait for the flags' copy only (i8_flags_to_host): the trees queued behind it keep the GPU busy meanwhile
  CVG_CK(cudaEventSynchronize(flags_ev_.get()));
  const size_t nseg = segs_.size();
  ovf_host_.assign(nseg, 0);
  if (sample_ > 1) std::copy(flags_host_.get(), flags_host_.get() + nseg, ovf_host_.begin());
  const int aborted = overlapped_ ? flags_host_.get()[nseg] : 0;
  overlapped_ = false;
  if (aborted) {
    // A Gram item gave up waiting for the cut (the two kernels did not share the SMs): the digits are complete
    // by now (the cut never waits), so redo the Gram alone, and keep this context on the serial path.
    ctx_->overlap_failed = true;
    std::fprintf(stderr, "cvgram: the cut did not run beside the Gram (a Gram item waited %d ms); serial schedule from here on\n", 1000);
    CVG_TRY(i8_gram(tilesq_d_.as<int2>(), (int)tilesq_.size()));
    CVG_TRY(gram_trees());
  }
  int64_t flagged = 0;
  for (int v : ovf_host_) flagged += v != 0;
  exact_segments_ = flagged;
  if (!flagged) return Status::Ok();
  CVG_TRY(i8_prep(d_x, ldx, d_y, ldy, rows, nsrc, 0, kp_, true));
  CVG_TRY(i8_gram(tilesq_d_.as<int2>(), (int)tilesq_.size()));
  return gram_trees();
}

// The int8 path's host decisions (segments to redo from exact maxima; the overlapped Gram's abort flag) are
// final once the cut and the Gram are done: copy them into pinned memory right there and record an event, so
// that the host waits for that copy while the fold trees run, not for the whole stream.
Status Plan::i8_flags_to_host() {
  flags_pending_ = false;
  if ((sample_ <= 1 && !overlapped_) || segs_.empty()) return Status::Ok();
  cudaStream_t s = ctx_->stream;
  const size_t nseg = segs_.size();
  CVG_TRY(flags_host_.ensure(nseg + 1));
  CVG_TRY(flags_ev_.ensure());
  if (sample_ > 1)
    CVG_CK(cudaMemcpyAsync(flags_host_.get(), ovf_.as<int>(), sizeof(int) * nseg, cudaMemcpyDeviceToHost, s));
  if (overlapped_)
    CVG_CK(cudaMemcpyAsync(flags_host_.get() + nseg, seg_ready_.as<unsigned>() + nseg, sizeof(int),
                           cudaMemcpyDeviceToHost, s));
  CVG_CK(cudaEventRecord(flags_ev_.get(), s));
  flags_pending_ = true;
  return Status::Ok();
}

Status Plan::gram_trees() {
  CVG_TRY(fold_tree_.run(ctx_, tiles_d_.as<int2>(), (int)tiles_.size(), kp_));
  CVG_TRY(local_tree_.run(ctx_, tiles_d_.as<int2>(), (int)tiles_.size(), kp_));
  grammed_ = true;
  return Status::Ok();
}

// Host-resident x | y streamed by column slabs (cvg_run_all_folds).  The Gram
// tile (i, j), i <= j, needs only Z columns of tile columns i and j, so X's
// columns are copied in slabs of tile columns on a copy stream, and each
// slab's K1 and the tiles it completes run on the compute stream while the
// next slab is in flight.  Every tile is the same kernel over the same segments as gram(), so
// the result is bit-identical; only the schedule changes.
Status Plan::gram_host(const void* h_x, const void* h_y, void* d_x, void* d_y, const double* host_shift) {
  if (!bound_) return Status::Err(4, "plan has no bound partitioning");
  cudaStream_t s = ctx_->stream;
  CVG_TRY(ctx_->ensure_copy_stream());
  const size_t e = dtype_ == 1 ? 4 : 8;
  const int E = dtype_ == 1 && !i8_path() ? kTileF32 : kTile;
  const int nt = (int)(kp_ / E);
  const std::vector<int2>& tl = i8_path() ? tilesq_ : dtype_ == 1 ? tiles128_ : tiles_;
  // the last 64-column block a tile reads (int8 tiles: the A rows they write, and J)
  auto last_col = [&](const int2& t) {
    if (!i8_path()) return t.y;
    const int c = t.y & 0xffff, a0 = t.x & 0xffff, a1 = t.x >> 16;
    return std::max(c, std::max(a0, ((t.y >> 18) & 3) ? a1 : a0));
  };
  // Slabs (in tile columns): [0, nt/2), [nt/2, nt-1), [nt-1, nt).  Tiles touching
  // the last-arriving column are the only Gram work exposed after the final copy
  // (nt of the nt(nt+1)/2 upper tiles); wide early slabs keep the 2-D copies at
  // >= 53 GB/s (measured: 2 KB rows 54, 512 B rows 50, 256 B rows 46 GB/s).
  std::vector<int> bounds{0};
  if (nt >= 3) bounds.push_back((nt + 1) / 2);
  if (nt >= 2 && bounds.back() < nt - 1) bounds.push_back(nt - 1);
  bounds.push_back(nt);
  // each slab's tiles (column tile in the slab)
  std::vector<int2> byslab;
  std::vector<int> off{0};
  for (size_t sl = 0; sl + 1 < bounds.size(); ++sl) {
    for (const int2& t : tl)
      if (last_col(t) >= bounds[sl] && last_col(t) < bounds[sl + 1]) byslab.push_back(t);
    off.push_back((int)byslab.size());
  }
  CVG_TRY(tiles_bycol_d_.ensure(sizeof(int2) * std::max<size_t>(byslab.size(), 1)));
  CVG_TRY(col_stage_.upload({{byslab.data(), sizeof(int2) * byslab.size(), tiles_bycol_d_.as<void>()}}, s));
  double* shift = shift_.as<double>();
  CVG_TRY(shift_stage_.upload({{host_shift, sizeof(double) * w_, shift}}, s));
  CVG_CK(cudaMemsetAsync(flag_.as<void>(), 0, sizeof(int), s));
  if (i8_path() && !segs_.empty()) {
    CVG_CK(cudaMemsetAsync(segmax_.as<void>(), 0, sizeof(unsigned long long) * segs_.size() * kp_, s));
    if (sample_ > 1) CVG_CK(cudaMemsetAsync(ovf_.as<void>(), 0, sizeof(int) * segs_.size(), s));
  }
  // the copy stream may overwrite d_x / d_y only after earlier work on s is done
  cudaEvent_t ev0 = ctx_->stream_event(0);
  CVG_CK(cudaEventRecord(ev0, s));
  CVG_CK(cudaStreamWaitEvent(ctx_->copy_stream, ev0, 0));
  for (size_t slab = 0; slab + 1 < bounds.size(); ++slab) {
    const int a = bounds[slab], b = bounds[slab + 1];
    const int64_t z0 = (int64_t)a * E, z1 = (int64_t)b * E;
    const int64_t x0 = std::min(z0, k_), x1 = std::min(z1, k_);
    if (x1 - x0 == k_)  // the whole row: one contiguous copy
      CVG_CK(cudaMemcpyAsync(d_x, h_x, n_ * k_ * e, cudaMemcpyHostToDevice, ctx_->copy_stream));
    else if (x1 > x0)
      CVG_CK(cudaMemcpy2DAsync(static_cast<char*>(d_x) + x0 * e, k_ * e, static_cast<const char*>(h_x) + x0 * e,
                               k_ * e, (x1 - x0) * e, n_, cudaMemcpyHostToDevice, ctx_->copy_stream));
    // Y (narrow rows: a 2-D copy would be DMA-descriptor bound) goes whole, contiguously,
    // with the first slab that holds any of its columns.
    if (z0 <= k_ && k_ < z1)
      CVG_CK(cudaMemcpyAsync(d_y, h_y, n_ * m_ * e, cudaMemcpyHostToDevice, ctx_->copy_stream));
    cudaEvent_t ev = ctx_->stream_event(1 + slab);
    CVG_CK(cudaEventRecord(ev, ctx_->copy_stream));
    CVG_CK(cudaStreamWaitEvent(s, ev, 0));
    const int t0 = off[slab], t1 = off[slab + 1];
    if (zrows_ > 0 && i8_path()) {
      CVG_TRY(i8_prep(d_x, k_, d_y, m_, src_row_.as<int64_t>(), src_n_, z0, z1, false));
    } else if (zrows_ > 0) {
      {
        Timed t(ctx_, kReorder);
        if (f16_path()) {
          if (!launch_reorder_split_h(dtype_, d_x, k_, d_y, m_, k_, m_, src_row_.as<int64_t>(), zrows_, kp_, z0, z1,
                                      src_n_, shift, (int)row_step_, zt_hi_.as<void>(), zt_lo_.as<void>(),
                                      unscale_.as<float>(), flag_.as<int>(), s))
            return Status::Err(5, "cuTensorMapEncodeTiled unavailable or rejected the operand layout");
        }
        else if (dtype_ == 1)
          launch_reorder_split_t(dtype_, d_x, k_, d_y, m_, k_, m_, src_row_.as<int64_t>(), zrows_, kp_, z0, z1, shift,
                                 zt_hi_.as<float>(), zt_lo_.as<float>(), flag_.as<int>(), s);
        else
          launch_reorder(dtype_, d_x, k_, d_y, m_, k_, m_, src_row_.as<int64_t>(), zrows_, kp_, z0, z1, src_n_, shift,
                         z_.as<double>(), flag_.as<int>(), s);
      }
      CVG_TRY(count_launch());
    }
    if (!segs_.empty() && t1 > t0) {
      bool ok = true;
      {
        Timed t(ctx_, kGram);
        if (f16_path())
          ok = launch_gram_f16s(zt_hi_.as<void>(), zt_lo_.as<void>(), unscale_.as<float>(), (int)row_step_, zrows_,
                                kp_, segs_d_.as<GramTask>(), (int64_t)segs_.size(), tiles_bycol_d_.as<int2>() + t0,
                                t1 - t0, part_.as<double>(), s);
        else if (i8_path())
          ok = launch_gram_i8(slices_, zq_.as<int8_t>(), segmax_.as<unsigned long long>(), sample_ > 1 ? 1 : 0, zrows_,
                              kp_, segs_d_.as<GramTask>(), (int64_t)segs_.size(), tiles_bycol_d_.as<int2>() + t0,
                              t1 - t0, part_.as<double>(), s);
        else if (dtype_ == 1)
          ok = launch_gram_tf32(zt_hi_.as<float>(), zt_lo_.as<float>(), zrows_, kp_, segs_d_.as<GramTask>(),
                                (int64_t)segs_.size(), tiles_bycol_d_.as<int2>() + t0, t1 - t0, part_.as<double>(), 3,
                                s);
        else
          launch_gram_f64(z_.as<double>(), kp_, zrows_, segs_d_.as<GramTask>(), (int64_t)segs_.size(),
                          tiles_bycol_d_.as<int2>() + t0, t1 - t0, part_.as<double>(), s);
      }
      if (!ok) return Status::Err(5, "cuTensorMapEncodeTiled unavailable or rejected the operand layout");
      CVG_TRY(count_launch());
    }
  }
  if (i8_path()) CVG_TRY(i8_flags_to_host());
  CVG_TRY(gram_trees());
  if (i8_path()) CVG_TRY(i8_exact_pass(d_x, k_, d_y, m_, src_row_.as<int64_t>(), src_n_));
  return poison_local();
}

Status Plan::finish(const double* d_rank_partials, int32_t n_ranks, const double* total_override,
                    const uint32_t* cfgs, int32_t ncfg, double* d_xtx, double* d_xty, double* d_mean_x,
                    double* d_mean_y, double* d_std_x, double* d_std_y, int32_t range_lo, int32_t range_hi) {
  if (!grammed_) return Status::Err(4, "finish called before gram");
  cudaStream_t s = ctx_->stream;
  const double* total = nullptr;
  if (total_override) {
    total = total_override;
  } else if (d_rank_partials && n_ranks > 1) {
    CVG_TRY(total_.ensure(sizeof(double) * kp_ * kp_));
    TreeGroup g{{}, total_.as<double>()};
    for (int r = 0; r < n_ranks; ++r) g.leaves.push_back(d_rank_partials + (int64_t)r * kp_ * kp_);
    CVG_TRY(rank_tree_.build({g}, kp_, s));
    CVG_TRY(rank_tree_.run(ctx_, tiles_d_.as<int2>(), (int)tiles_.size(), kp_));
    total = total_.as<double>();
  } else if (d_rank_partials && n_ranks == 1) {
    total = d_rank_partials;
  } else {
    if (!owns_all()) return Status::Err(4, "plan owns a subset of folds: pass every rank's partial");
    total = local_.as<double>();
  }
  if (seg_lo_ >= 0) {
    // Shared fold: its Gram is the group's node of the canonical tree.
    if (!d_rank_partials || n_ranks != world_) return Status::Err(4, "shared fold: pass every rank's partial");
    TreeGroup g{{}, foldbuf_.as<double>()};
    for (int r = group_lo_; r < group_hi_; ++r) g.leaves.push_back(d_rank_partials + (int64_t)r * kp_ * kp_);
    CVG_TRY(group_tree_.build({g}, kp_, s));
    CVG_TRY(group_tree_.run(ctx_, tiles_d_.as<int2>(), (int)tiles_.size(), kp_));
  }
  // Emitted folds [lo, hi) of the owned ones (default: all); outputs are packed for that range, so a
  // caller can stream huge P (e.g. leave-one-out) through bounded buffers.
  const int32_t lo = range_lo < 0 ? 0 : range_lo;
  const int32_t hi = range_hi < 0 ? this->nown() : range_hi;
  if (lo > hi || hi > this->nown()) return Status::Err(4, "fold range outside the plan's emitted folds");
  const int nown = hi - lo;
  if (nown == 0) {
    CVG_CK(cudaStreamSynchronize(s));
    return Status::Ok();
  }
  CVG_TRY(st_mz_.ensure(sizeof(double) * nown * kp_));
  CVG_TRY(st_sT_.ensure(sizeof(double) * nown * kp_));
  CVG_TRY(st_sd_.ensure(sizeof(double) * nown * kp_));
  FoldStatsDev st{st_mz_.as<double>(), st_sT_.as<double>(), st_sd_.as<double>()};
  const double* const* fptr = foldptr_d_.as<const double*>() + lo;
  const int64_t* nval = nval_d_.as<int64_t>() + lo;
  SmallFolds sf = small_folds();
  if (sf.zbase) sf.zbase += lo;
  {
    Timed t(ctx_, kStats);
    launch_fold_stats(total, fptr, nval, nown, n_, k_, m_, kp_, shift_.as<double>(), st, d_mean_x, d_mean_y, d_std_x,
                      d_std_y, flag_.as<int>(), s, sf);
  }
  CVG_TRY(count_launch());
  if (ncfg > 0) {
    CVG_TRY(cfg_d_.ensure(sizeof(uint32_t) * ncfg));
    CVG_TRY(cfg_stage_.upload({{cfgs, sizeof(uint32_t) * ncfg, cfg_d_.as<void>()}}, s));
    int nl = 0;
    {
      Timed t(ctx_, kProducts);
      nl = launch_products(total, fptr, nval, nown, n_, k_, m_, kp_, shift_.as<double>(), st, out_tiles_d_.as<int2>(),
                           (int)out_tiles_.size(), out_ndiag_, cfg_d_.as<uint32_t>(), ncfg, d_xtx, d_xty, s, sf);
    }
    CVG_TRY(count_launch(nl));
  }
  int flag = 0;
  CVG_CK(cudaMemcpyAsync(&flag, flag_.as<int>(), sizeof flag, cudaMemcpyDeviceToHost, s));
  CVG_CK(cudaStreamSynchronize(s));
  if (flag & 2)  // K1H range bit (an out-of-range value also surfaces as non-finite Gram entries: bit 0)
    return Status::Err(1, "fp32 inputs: |x - x[0]| >= 2^79 exceeds the fp32 tensor-core accumulation range");
  if (flag) return Status::Err(1, "x and y entries must be finite");
  return Status::Ok();
}

Status Plan::finish_direct(const uint32_t* cfgs, int32_t ncfg, double* d_xtx, double* d_xty, double* d_mean_x,
                           double* d_mean_y, double* d_std_x, double* d_std_y) {
  if (!grammed_ || p_ != 1) return Status::Err(4, "finish_direct needs a grammed single-fold plan");
  cudaStream_t s = ctx_->stream;
  CVG_TRY(zero_g_.ensure(sizeof(double) * kp_ * kp_));
  CVG_TRY(zero_nval_.ensure(sizeof(int64_t)));
  CVG_TRY(zero_ptr_.ensure(sizeof(void*)));
  CVG_CK(cudaMemsetAsync(zero_g_.as<void>(), 0, sizeof(double) * kp_ * kp_, s));
  CVG_CK(cudaMemsetAsync(zero_nval_.as<void>(), 0, sizeof(int64_t), s));
  const double* zp = zero_g_.as<double>();
  CVG_CK(cudaMemcpyAsync(zero_ptr_.as<void>(), &zp, sizeof(void*), cudaMemcpyHostToDevice, s));
  const int64_t n_saved = n_;
  n_ = counts_[0];  // the training set is exactly the bound rows
  CVG_TRY(st_mz_.ensure(sizeof(double) * kp_));
  CVG_TRY(st_sT_.ensure(sizeof(double) * kp_));
  CVG_TRY(st_sd_.ensure(sizeof(double) * kp_));
  FoldStatsDev st{st_mz_.as<double>(), st_sT_.as<double>(), st_sd_.as<double>()};
  {
    Timed t(ctx_, kStats);
    launch_fold_stats(local_.as<double>(), zero_ptr_.as<const double*>(), zero_nval_.as<int64_t>(), 1, n_, k_, m_,
                      kp_, shift_.as<double>(), st, d_mean_x, d_mean_y, d_std_x, d_std_y, flag_.as<int>(), s);
  }
  Status rc = count_launch();
  if (rc.ok() && ncfg > 0) {
    rc = cfg_d_.ensure(sizeof(uint32_t) * ncfg);
    if (rc.ok()) rc = cuda_status(cudaMemcpyAsync(cfg_d_.as<void>(), cfgs, sizeof(uint32_t) * ncfg,
                                                  cudaMemcpyHostToDevice, s), "H2D cfgs");
    if (rc.ok()) {
      int nl = 0;
      {
        Timed t(ctx_, kProducts);
        nl = launch_products(local_.as<double>(), zero_ptr_.as<const double*>(), zero_nval_.as<int64_t>(), 1, n_, k_,
                             m_, kp_, shift_.as<double>(), st, out_tiles_d_.as<int2>(), (int)out_tiles_.size(),
                             out_ndiag_, cfg_d_.as<uint32_t>(), ncfg, d_xtx, d_xty, s);
      }
      rc = count_launch(nl);
    }
  }
  n_ = n_saved;
  CVG_TRY(rc);
  return cuda_status(cudaStreamSynchronize(s), "stream synchronize");
}

Status Plan::direct_means(double* d_mean) {
  // mean = shift + column sums / count (the stats kernel's mean outputs, [x | y]).
  return finish_direct(nullptr, 0, nullptr, nullptr, d_mean, d_mean + k_, nullptr, nullptr);
}

}  // namespace cvg
