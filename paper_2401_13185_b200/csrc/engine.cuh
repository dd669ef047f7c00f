// Host orchestration of the cvgram B200 engine: context, plan, global cache.
#pragma once

#include <initializer_list>
#include <memory>
#include <string>
#include <vector>

#include "cvg_internal.cuh"

struct cvg_context;

namespace cvg {

// Grow-only device buffer.
class DevBuf {
 public:
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  Status ensure(size_t bytes);
  void release();
  template <typename T>
  T* as() const { return static_cast<T*>(p_); }
  size_t bytes() const { return bytes_; }

 private:
  void* p_ = nullptr;
  size_t bytes_ = 0;
};

Status cuda_status(cudaError_t e, const char* what);

// Pinned staging for small host->device uploads on the hot path (segment
// tables, tree programs, the shift, configuration masks): copies from pinned
// memory are truly asynchronous, where a pageable cudaMemcpyAsync synchronises
// the stream.  Before the buffer is rewritten, the previous upload from it is
// waited for (an event), so back-to-back calls stay correct.
class PinnedStage {
 public:
  PinnedStage() = default;
  PinnedStage(const PinnedStage&) = delete;
  PinnedStage& operator=(const PinnedStage&) = delete;
  ~PinnedStage();
  // Uploads `parts` (host pointer, bytes, device destination) through the buffer on stream s.
  struct Part {
    const void* src;
    size_t bytes;
    void* dst;
  };
  Status upload(std::initializer_list<Part> parts, cudaStream_t s);

 private:
  void* p_ = nullptr;
  size_t bytes_ = 0;
  cudaEvent_t ev_ = nullptr;
  bool pending_ = false;
};

// A set of midpoint-tree sums flattened into levels of independent pairwise
// adds (K4).  Group g: dst = S(leaves[0..n)); n == 1 copies, n == 0 zeroes.
struct TreeGroup {
  std::vector<const double*> leaves;
  double* dst;
};
class TreeProgram {
 public:
  Status build(const std::vector<TreeGroup>& groups, int64_t kp, cudaStream_t s);
  Status run(cvg_context* ctx, const int2* tiles, int ntiles, int64_t kp) const;
  int levels() const { return (int)level_off_.size() - 1; }

 private:
  const double* emit(const std::vector<const double*>& leaves, int a, int b, int depth, double* root_dst,
                     std::vector<std::vector<TreeOp>>& by_depth, int64_t kp);
  std::vector<int> level_off_;
  std::vector<TreeOp> flat_;
  DevBuf scratch_, ops_d_;
  PinnedStage stage_;
  int64_t next_slot_ = 0;
};

// One partitioning of n rows into p folds, of which folds [fb, fe) are owned.
class Plan {
 public:
  Status create(cvg_context* ctx, int dtype, int64_t n, int64_t k, int64_t m, int32_t p, int32_t fb, int32_t fe,
                bool validate);
  // Rank mode: the owned part of the canonical fold tree is decided at bind time
  // (cvg_fold_range's descent, continued into one fold's segment range when
  // more ranks than folds remain — SURVEY.md §8e's P < G case).
  Status create_rank(cvg_context* ctx, int dtype, int64_t n, int64_t k, int64_t m, int32_t p, int32_t rank,
                     int32_t world);
  // Device labels -> fold-bucketed row order (validates like partition.hpp:21-58 when `validate`).
  Status bind_labels(const int32_t* d_labels, bool validate, bool require_scalable);
  // Explicit ascending rows of the single owned fold (fold_products / precompute_global).
  // rows index a source X of n_src rows (< 0: the plan's n); checked on the host.
  Status bind_rows(const int64_t* rows, int64_t nrows, int64_t n_src = -1);
  // K1 + K2 + K4.  Exactly one of host_shift / dev_shift may be non-null; both null => row 0.
  // d_row_map (optional, n int64): x / y hold only the rows the map covers,
  // original row i at compact row d_row_map[i] (< n_compact); -1 = absent.
  Status gram(const void* d_x, int64_t ldx, const void* d_y, int64_t ldy, const double* host_shift,
              const double* dev_shift, const int64_t* d_row_map = nullptr, int64_t n_compact = 0);
  // Same as gram() for HOST x | y (row-major, ldx = k, ldy = m): column slabs
  // are copied into d_x / d_y (n x k, n x m) on the context's copy stream while
  // earlier slabs' K1 + Gram tiles run; bit-identical to gram().
  Status gram_host(const void* h_x, const void* h_y, void* d_x, void* d_y, const double* host_shift);
  // Cross-rank combine (optional) + K5 for the owned folds into device outputs.
  // [range_lo, range_hi): emitted-fold subrange (default all), outputs packed for it.
  Status finish(const double* d_rank_partials, int32_t n_ranks, const double* total_override,
                const uint32_t* cfgs, int32_t ncfg, double* d_xtx, double* d_xty, double* d_mean_x,
                double* d_mean_y, double* d_std_x, double* d_std_y, int32_t range_lo = -1, int32_t range_hi = -1);

  // Baseline (direct) epilogue for a bind_rows plan: the bound rows ARE the
  // training set (no downdate): total = their Gram, fold Gram = 0, n_val = 0.
  Status finish_direct(const uint32_t* cfgs, int32_t ncfg, double* d_xtx, double* d_xty, double* d_mean_x,
                       double* d_mean_y, double* d_std_x, double* d_std_y);
  // Training means of the bound rows (shift + column sums / count), on the device.
  Status direct_means(double* d_mean);
  const double* local() const { return local_.as<double>(); }
  const double* shift() const { return shift_.as<double>(); }
  int64_t kp() const { return kp_; }
  int64_t partial_count() const { return kp_ * kp_; }
  int nown() const { return emits_ ? fe_ - fb_ : 0; }  // folds this plan emits
  int32_t fold_begin() const { return fb_; }
  int32_t fold_end() const { return emits_ ? fe_ : fb_; }
  const std::vector<int64_t>& counts() const { return counts_; }
  bool owns_all() const { return fb_ == 0 && fe_ == p_; }
  int64_t n() const { return n_; }
  int64_t k() const { return k_; }
  int64_t m() const { return m_; }
  int32_t p() const { return p_; }
  int dtype() const { return dtype_; }
  cvg_context* ctx() const { return ctx_; }
  int64_t zrows() const { return zrows_; }
  int64_t nseg() const { return (int64_t)segs_.size(); }
  int ntiles() const { return (int)tiles_.size(); }

 private:
  Status plan_segments();
  Status gram_trees();
  Status poison_local();  // non-finite flag -> NaN in the exchanged partial (launch_poison_if_flag)
  Status i8_prep(const void* d_x, int64_t ldx, const void* d_y, int64_t ldy, const int64_t* rows, int64_t nsrc,
                 int64_t c0, int64_t c1, bool exact);
  Status i8_gram(const int2* tiles, int ntiles);
  Status i8_flags_to_host();
  Status ensure_split_ws();
  Status i8_exact_pass(const void* d_x, int64_t ldx, const void* d_y, int64_t ldy, const int64_t* rows, int64_t nsrc);
  // the cut beside the Gram (engine.cu; CVG_I8_OVERLAP=0|1 overrides the segment-length rule): one direct-store cut CTA and one lean Gram CTA per SM
  Status i8_overlapped(const void* d_x, int64_t ldx, const void* d_y, int64_t ldy, const int64_t* rows, int64_t nsrc);
  bool i8_overlap_enabled() const;
  static bool small_folds_enabled();

 public:
  // A single full-range plan over these fold sizes runs small-fold mode (a different fixed summation order than
  // rank-mode plans, which keep per-fold partials).
  static bool small_fold_mode(int dtype, const std::vector<int64_t>& counts);

 private:
  SmallFolds small_folds() const {
    SmallFolds sf;
    if (small_) {
      sf.z = z_.as<double>();
      sf.zbase = zbase_d_.as<int64_t>();
    }
    return sf;
  }
  Status count_launch(int n = 1);
  void assign_rank();  // rank mode: fb_/fe_, segment window, fold group
  int64_t chunk_rows() const;
  int64_t seg_rows(int64_t count) const;
  int64_t min_seg_rows() const {
    int64_t r = INT64_MAX;
    for (const GramTask& g : segs_) r = std::min(r, g.rows);
    return segs_.empty() ? 0 : r;
  }
  int64_t max_seg_rows() const {
    int64_t r = 0;
    for (const GramTask& g : segs_) r = std::max(r, g.rows);
    return r;
  }
  bool f16_path() const { return dtype_ == 1 && !fp32_tf32() && !i8_; }
  static bool fp32_tf32();
  // fp64 Gram on tcgen05 kind::i8 (int8 digit slices, k_gram_i8.cu); small-fold mode keeps
  // the DMMA path (its epilogue reads fp64 Z rows).
  bool i8_path() const { return i8_ && !small_; }
  void choose_row_step();  // fold padding / segment alignment (fp16 path: its row group G)

  cvg_context* ctx_ = nullptr;
  int dtype_ = 0;
  int64_t n_ = 0, k_ = 0, m_ = 0, w_ = 0, kp_ = 0;
  int32_t p_ = 0, fb_ = 0, fe_ = 0;
  std::vector<int2> tiles_, out_tiles_, tiles128_;
  int out_ndiag_ = 0;  // out_tiles_[0, out_ndiag_) are diagonal tiles
  std::vector<int2> tilesq_;    // int8 Gram items {a0 | a1 << 16, c | mode0 << 16 | mode1 << 18} (i8_items)
  bool i8_ = false;             // int8 digit slices: fp64 default (CVG_FP64_KIND=dmma: DMMA); fp32 with CVG_FP32_KIND=i8
  int sample_ = 16;             // int8 path: segment maxima over every sample_-th row (CVG_I8_SAMPLE; 1 = exact)
  int64_t exact_segments_ = 0;  // segments the last gram redid from their exact max
  std::vector<int> ovf_host_;
  struct PlanKey {  // what plan_segments() depends on
    std::vector<int64_t> counts;
    int32_t fb = 0, fe = 0;
    int64_t seg_lo = 0, seg_hi = 0, row_step = 0;
    bool small = false, i8 = false;
    bool operator==(const PlanKey& o) const {
      return fb == o.fb && fe == o.fe && seg_lo == o.seg_lo && seg_hi == o.seg_hi && row_step == o.row_step &&
             small == o.small && i8 == o.i8 && counts == o.counts;
    }
  };
  PlanKey plan_key_;
  bool planned_ = false;        // plan_key_ describes the segment plan the device buffers hold
  struct PinnedInts {  // pinned host words for small device -> host flag copies
    int* p = nullptr;
    size_t cap = 0;
    ~PinnedInts() {
      if (p) cudaFreeHost(p);
    }
    Status ensure(size_t n) {
      if (n <= cap) return Status::Ok();
      if (p) cudaFreeHost(p);
      p = nullptr;
      cap = 0;
      Status st = cuda_status(cudaHostAlloc(reinterpret_cast<void**>(&p), sizeof(int) * n, cudaHostAllocDefault),
                              "cudaHostAlloc (flags)");
      if (st.ok()) cap = n;
      return st;
    }
    int* get() const { return p; }
  };
  struct OwnedEvent {
    cudaEvent_t e = nullptr;
    ~OwnedEvent() {
      if (e) cudaEventDestroy(e);
    }
    Status ensure() {
      return e ? Status::Ok() : cuda_status(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
    }
    cudaEvent_t get() const { return e; }
  };
  PinnedInts flags_host_;       // int8 path: ovf[nseg] + the overlapped Gram's abort flag
  OwnedEvent flags_ev_;
  bool flags_pending_ = false;
  DevBuf split_ws_, split_cnt_;  // int8 Gram tail split: int32 dumps and per-item arrival counters
  DevBuf seg_ready_;            // overlapped cut: per-segment finished-block counts + the abort flag (last word)
  bool overlapped_ = false;     // the last gram ran the cut beside the Gram (its abort flag is pending)
  int slices_ = 6;              // base-256 int8 digits per value (fp64: CVG_I8_SLICES = 5 | 6; fp32: CVG_I8_SLICES_F32 = 3 | 4)
  std::vector<int64_t> counts_;  // per fold (all p) validation sizes
  std::vector<GramTask> segs_;
  std::vector<int32_t> fold_seg_begin_;
  std::vector<int64_t> fold_zbase_;
  int64_t zrows_ = 0;
  int64_t src_n_ = 0;  // rows of the x / y the row map indexes (K1 bounds)
  int64_t row_step_ = kRowStep;  // folds pad to, and segments align on, this many rows
  bool small_ = false;  // small-fold mode (every fold <= kSmallFoldRows rows; see plan_segments)
  bool bound_ = false, grammed_ = false;
  bool rank_mode_ = false, emits_ = true;
  int32_t rank_ = 0, world_ = 1;
  int64_t seg_lo_ = -1, seg_hi_ = -1;   // shared fold: owned segment range (else -1)
  int32_t group_lo_ = 0, group_hi_ = 0; // ranks sharing the fold
  TreeProgram group_tree_;
  DevBuf zero_g_, zero_nval_, zero_ptr_;

  DevBuf zq_, segmax_, ovf_, blkseg_, tilesq_d_, tiles_d_, out_tiles_d_, tiles128_d_, zt_hi_, zt_lo_, unscale_, tile_counts_, fold_counts_, bad_, zbase_d_, src_row_, z_, part_, foldbuf_, local_,
      total_, shift_, flag_, tiles_bycol_d_, src_map_, segs_d_, foldptr_d_, nval_d_, st_mz_, st_sT_, st_sd_, cfg_d_;
  TreeProgram fold_tree_, local_tree_, rank_tree_;
  PinnedStage blkseg_stage_, seg_stage_, ptr_stage_, shift_stage_, cfg_stage_, col_stage_;
  std::vector<const double*> fold_ptrs_;
};

// Device scratch of the host-buffer entry point (cvg_run_all_folds), reused across calls.
struct HostScratch {
  DevBuf x, y, labels, xtx, xty, mx, my, sx, sy;
  Plan plan;
  void* stage = nullptr;  // 2 x 32 MB pinned staging for large D2H into pageable memory (capi.cu d2h_large)
  cudaEvent_t stage_ev[2] = {nullptr, nullptr};
  ~HostScratch() {
    if (stage) cudaFreeHost(stage);
    for (cudaEvent_t e : stage_ev)
      if (e) cudaEventDestroy(e);
  }
};

}  // namespace cvg

struct cvg_context {
  int device = 0;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  int64_t launches = 0;
  std::unique_ptr<cvg::HostScratch> scratch;
  // cvg_context_create_multi: one sub-context per rank (device) and, for distinct devices, one NCCL
  // communicator per rank (multi.cu); empty for a single-device context
  std::vector<cvg_context*> ranks;
  std::vector<void*> comms;  // ncclComm_t
  bool nccl = false;
  // optional per-class kernel timing (cvg_context_enable_timing)
  bool timing = false;
  struct Rec {
    int cls;
    cudaEvent_t a, b;
  };
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> event_pool;
  cudaEvent_t take_event();
  // host-input streaming (Plan::gram_host): a copy stream and reusable events
  cudaStream_t copy_stream = nullptr;
  cudaStream_t aux_stream = nullptr;  // the cut that runs beside the int8 Gram
  bool overlap_failed = false;        // a Gram waited out its timeout once: stay on the serial path
  std::vector<cudaEvent_t> sync_events;
  cvg::Status ensure_copy_stream();
  cvg::Status ensure_aux_stream();
  cudaEvent_t stream_event(size_t i);
  void begin(int cls);
  void end();
  void clear_recs();
};

namespace cvg {
enum KernelClass { kBucket = 0, kReorder = 1, kGram = 2, kTree = 3, kStats = 4, kProducts = 5, kClasses = 6 };
// Records CUDA events around one launch when the context is timing.
class Timed {
 public:
  Timed(cvg_context* c, int cls) : c_(c) {
    if (c_->timing) c_->begin(cls);
  }
  ~Timed() {
    if (c_->timing) c_->end();
  }

 private:
  cvg_context* c_;
};
}  // namespace cvg

struct cvg_plan {
  cvg::Plan plan;
};

struct cvg_global {
  cvg_context* ctx = nullptr;
  int dtype = 0;
  int64_t n = 0, k = 0, m = 0;
  cvg::DevBuf x, y;
  cvg::Plan all;   // one fold = every row: the whole-data Gram
  cvg::Plan fold;  // scratch plan for fold_products
  cvg::DevBuf out_xtx, out_xty, out_vec, cfg_d;
};
