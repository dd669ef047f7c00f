// Several B200s behind one C-ABI context (cvg_context_create_multi): the reference's only parallelism knob is
// run_all_folds(..., n_threads) (fast.hpp:133-152, threading.hpp:12-26); here a C or C++ caller of
// cvgram::run_all_folds gets every GPU of the node with no torch and no launcher.
//
// One host thread per device drives that device's rank plan; the exchanges are issued from the calling thread
// as NCCL groups over the ranks' communicators (ncclCommInitAll; NVLink / NVSwitch), or -- when the device list
// repeats a device (one-GPU emulation of a multi-GPU context) or CVG_EXCHANGE=peer -- as device-to-device copies.
// No kernel ever waits on another rank's kernel: every exchange is a host-ordered phase between launches.
//
// cvg_run_all_folds on a multi-device context (host buffers in and out):
//   every rank owns a node of the canonical fold tree (cvg_fold_range; when ranks outnumber folds, a node of one
//   fold's segment tree) -- the same ownership as the torch.distributed driver (plan.py), so outputs are
//   bit-identical to one GPU for power-of-two rank counts;
//   P >= G: rank r copies only its contiguous row shard over its own PCIe link; rows are gathered by owning rank
//     on the device and sent over NVLink (one grouped send/recv per matrix: each owner receives its folds' rows in
//     original order); the owner's plan reads the compacted rows through a row map (Plan::gram with a row map);
//   P < G: every rank streams the whole X | Y in by column slabs (Plan::gram_host) -- the fold is shared;
//   then the run's single collective: all-gather of every rank's partial Gram (kp^2 doubles), the fixed-order
//   tree sum into the whole-data Gram, and each rank's epilogue for the folds it emits, copied back into the
//   caller's [n_cfg][P][...] arrays at those folds' offsets.
#include <dlfcn.h>
#include <nccl.h>  // types only: the library is opened at run time (the engine loads without NCCL)

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/cvgram_b200.h"
#include "engine.cuh"
#include "multi.cuh"

namespace cvg {

namespace {

struct NcclApi {
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  std::string why;  // empty when loaded
};

const NcclApi& nccl() {
  static const NcclApi api = [] {
    NcclApi a;
    void* h = nullptr;
    for (const char* name : {"libnccl.so.2", "libnccl.so"})
      if ((h = dlopen(name, RTLD_NOW | RTLD_GLOBAL))) break;
    if (!h) {
      a.why = std::string("libnccl not loadable: ") + dlerror();
      return a;
    }
    auto sym = [&](const char* s) { return dlsym(h, s); };
    a.CommInitAll = reinterpret_cast<decltype(a.CommInitAll)>(sym("ncclCommInitAll"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
    a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(sym("ncclGroupStart"));
    a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(sym("ncclGroupEnd"));
    a.Send = reinterpret_cast<decltype(a.Send)>(sym("ncclSend"));
    a.Recv = reinterpret_cast<decltype(a.Recv)>(sym("ncclRecv"));
    a.AllGather = reinterpret_cast<decltype(a.AllGather)>(sym("ncclAllGather"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("ncclGetErrorString"));
    if (!a.CommInitAll || !a.CommDestroy || !a.GroupStart || !a.GroupEnd || !a.Send || !a.Recv || !a.AllGather ||
        !a.GetErrorString)
      a.why = "libnccl lacks a required symbol";
    return a;
  }();
  return api;
}

Status nccl_status(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return Status::Ok();
  return Status::Err(CVG_E_NCCL, std::string(what) + ": " + nccl().GetErrorString(r));
}

// dst[i][:] = src[idx[i]][:] (rows of `cols` elements, contiguous): one warp per row.
template <typename T>
__global__ void gather_rows_kernel(const T* __restrict__ src, const int64_t* __restrict__ idx, int64_t nrows,
                                   int64_t cols, T* __restrict__ dst) {
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
  for (int64_t i = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; i < nrows; i += warps) {
    const T* s = src + idx[i] * cols;
    T* d = dst + i * cols;
    for (int64_t c = threadIdx.x & 31; c < cols; c += 32) d[c] = s[c];
  }
}

void launch_gather_rows(int dtype, const void* src, const int64_t* idx, int64_t nrows, int64_t cols, void* dst,
                        cudaStream_t s) {
  if (nrows <= 0 || cols <= 0) return;
  const unsigned blocks = (unsigned)std::min<int64_t>((nrows + 7) / 8, 148 * 16);
  if (dtype == CVG_DTYPE_F32)
    gather_rows_kernel<float><<<blocks, 256, 0, s>>>((const float*)src, idx, nrows, cols, (float*)dst);
  else
    gather_rows_kernel<double><<<blocks, 256, 0, s>>>((const double*)src, idx, nrows, cols, (double*)dst);
}

// Per-rank device state of one multi-device run.
struct RankRun {
  Plan plan;
  DevBuf labels, xs, ys, perm, sx, sy, rx, ry, rowmap, gathered, xtx, xty, mx, my, sdx, sdy;
  int64_t nrecv = 0;
  int32_t ob = 0, oe = 0;  // folds this rank emits
  Status st;
};

}  // namespace

Status multi_init(cvg_context* ctx, const int* dev_ids, int n) {
  std::vector<int> devs(dev_ids, dev_ids + n);
  std::vector<int> sorted = devs;
  std::sort(sorted.begin(), sorted.end());
  const bool distinct = std::adjacent_find(sorted.begin(), sorted.end()) == sorted.end();
  const char* ex = std::getenv("CVG_EXCHANGE");
  const bool want_peer = ex && std::strcmp(ex, "peer") == 0;
  for (int r = 0; r < n; ++r) {
    cvg_context* sub = nullptr;
    char err[256] = {0};
    const int rc = cvg_context_create(devs[r], &sub, err, sizeof err);
    if (rc != CVG_OK) return Status::Err(rc, std::string("rank ") + std::to_string(r) + ": " + err);
    ctx->ranks.push_back(sub);
  }
  if (distinct && !want_peer) {
    const NcclApi& api = nccl();
    if (!api.why.empty()) return Status::Err(CVG_E_NCCL, api.why);
    ctx->comms.resize(n);
    Status s = nccl_status(api.CommInitAll(reinterpret_cast<ncclComm_t*>(ctx->comms.data()), n, devs.data()),
                           "ncclCommInitAll");
    if (!s.ok()) {
      ctx->comms.clear();
      return s;
    }
    ctx->nccl = true;
  } else if (distinct) {
    // peer copies between distinct devices: enable direct access where the topology offers it
    for (int a = 0; a < n; ++a)
      for (int b = 0; b < n; ++b) {
        int ok = 0;
        if (a != b && cudaDeviceCanAccessPeer(&ok, devs[a], devs[b]) == cudaSuccess && ok) {
          cudaSetDevice(devs[a]);
          cudaDeviceEnablePeerAccess(devs[b], 0);
          cudaGetLastError();  // already enabled is fine
        }
      }
  }
  return Status::Ok();
}

void multi_destroy(cvg_context* ctx) {
  if (ctx->nccl)
    for (void* c : ctx->comms) nccl().CommDestroy(reinterpret_cast<ncclComm_t>(c));
  ctx->comms.clear();
  for (cvg_context* sub : ctx->ranks) cvg_context_destroy(sub);
  ctx->ranks.clear();
}

Status run_all_folds_multi(cvg_context* ctx, int dtype, const void* x, const void* y, int64_t n, int64_t k, int64_t m,
                           const int32_t* labels, int32_t p, const uint32_t* cfgs, int32_t ncfg,
                           const std::vector<int64_t>& counts, bool scal, double* xtx, double* xty, double* mean_x,
                           double* mean_y, double* std_x, double* std_y) {
  const int G = (int)ctx->ranks.size();
  const size_t e = dtype == CVG_DTYPE_F32 ? 4 : 8;
  const ncclDataType_t nt = dtype == CVG_DTYPE_F32 ? ncclFloat : ncclDouble;
  std::vector<std::unique_ptr<RankRun>> R(G);
  for (auto& rr : R) rr.reset(new RankRun());
  // shift: row 0 of (x | y), the same on every rank
  std::vector<double> shift(k + m);
  for (int64_t c = 0; c < k + m; ++c) {
    const void* src = c < k ? x : y;
    const int64_t i = c < k ? c : c - k;
    shift[c] = dtype == CVG_DTYPE_F32 ? (double)static_cast<const float*>(src)[i] : static_cast<const double*>(src)[i];
  }
  // run fn(r) for every rank on its own host thread (device set), first failure in rank order wins
  auto par = [&](auto&& fn) -> Status {
    std::vector<std::thread> th;
    for (int r = 0; r < G; ++r)
      th.emplace_back([&, r] {
        Status s = cuda_status(cudaSetDevice(ctx->ranks[r]->device), "cudaSetDevice");
        R[r]->st = s.ok() ? fn(r) : s;
      });
    for (auto& t : th) t.join();
    for (int r = 0; r < G; ++r)
      if (!R[r]->st.ok()) return R[r]->st;
    return Status::Ok();
  };
  auto sync_all = [&]() -> Status {
    for (int r = 0; r < G; ++r) {
      Status s = cuda_status(cudaSetDevice(ctx->ranks[r]->device), "cudaSetDevice");
      if (s.ok()) s = cuda_status(cudaStreamSynchronize(ctx->ranks[r]->stream), "stream synchronize");
      if (!s.ok()) return s;
    }
    return Status::Ok();
  };
#define TRY(expr)              \
  do {                         \
    Status s_ = (expr);        \
    if (!s_.ok()) return s_;   \
  } while (0)

  // ---- host routing (whole folds per rank): row owner, each shard's rows in owner order, the owners' row maps
  const bool whole = p >= G;
  const int64_t shard = (n + G - 1) / G;
  std::vector<std::vector<int64_t>> sc(G, std::vector<int64_t>(G, 0));  // sc[r][o]: rows shard r sends to o
  std::vector<std::vector<int64_t>> perm(G), rowmap(G);
  if (whole) {
    std::vector<int32_t> owner_of_fold(p);
    for (int r = 0; r < G; ++r) {
      int32_t b = 0, en = 0;
      cvg_fold_range(p, r, G, &b, &en);
      for (int32_t f = b; f < en; ++f) owner_of_fold[f] = r;
    }
    std::vector<int64_t> cnt(G, 0);
    for (int r = 0; r < G; ++r) rowmap[r].assign(n, -1);
    for (int64_t i = 0; i < n; ++i) {
      const int o = owner_of_fold[labels[i] - 1];
      rowmap[o][i] = cnt[o]++;  // compact row: the owner receives shard 0's rows, then shard 1's, ... in order
    }
    for (int r = 0; r < G; ++r) {
      const int64_t lo = std::min(n, r * shard), hi = std::min(n, (r + 1) * shard);
      perm[r].reserve(hi - lo);
      for (int o = 0; o < G; ++o)
        for (int64_t i = lo; i < hi; ++i)
          if (owner_of_fold[labels[i] - 1] == o) perm[r].push_back(i - lo);
      for (int64_t i = lo; i < hi; ++i) ++sc[r][owner_of_fold[labels[i] - 1]];
    }
    for (int o = 0; o < G; ++o) R[o]->nrecv = cnt[o];
  }

  // ---- phase A (per rank): plan, labels, own shard in, rows gathered by owner
  TRY(par([&](int r) -> Status {
    RankRun& rr = *R[r];
    cvg_context* sub = ctx->ranks[r];
    cudaStream_t st = sub->stream;
    TRY(rr.labels.ensure(sizeof(int32_t) * n));
    TRY(cuda_status(cudaMemcpyAsync(rr.labels.as<void>(), labels, sizeof(int32_t) * n, cudaMemcpyHostToDevice, st),
                    "H2D labels"));
    TRY(rr.plan.create_rank(sub, dtype, n, k, m, p, r, G));
    TRY(rr.plan.bind_labels(rr.labels.as<int32_t>(), true, scal));
    rr.ob = rr.plan.fold_begin();
    rr.oe = rr.plan.fold_end();
    if (!whole) {  // shared folds: the whole X | Y streams in by column slabs
      TRY(rr.xs.ensure(e * n * k));
      TRY(rr.ys.ensure(e * n * m));
      return rr.plan.gram_host(x, y, rr.xs.as<void>(), rr.ys.as<void>(), shift.data());
    }
    const int64_t lo = std::min(n, r * shard), hi = std::min(n, (r + 1) * shard), rows = hi - lo;
    TRY(rr.xs.ensure(e * std::max<int64_t>(rows, 1) * k));
    TRY(rr.ys.ensure(e * std::max<int64_t>(rows, 1) * m));
    TRY(rr.sx.ensure(e * std::max<int64_t>(rows, 1) * k));
    TRY(rr.sy.ensure(e * std::max<int64_t>(rows, 1) * m));
    TRY(rr.perm.ensure(sizeof(int64_t) * std::max<int64_t>(rows, 1)));
    TRY(rr.rx.ensure(e * std::max<int64_t>(rr.nrecv, 1) * k));
    TRY(rr.ry.ensure(e * std::max<int64_t>(rr.nrecv, 1) * m));
    TRY(rr.rowmap.ensure(sizeof(int64_t) * n));
    const char* hx = static_cast<const char*>(x) + e * lo * k;
    const char* hy = static_cast<const char*>(y) + e * lo * m;
    TRY(cuda_status(cudaMemcpyAsync(rr.xs.as<void>(), hx, e * rows * k, cudaMemcpyHostToDevice, st), "H2D x shard"));
    TRY(cuda_status(cudaMemcpyAsync(rr.ys.as<void>(), hy, e * rows * m, cudaMemcpyHostToDevice, st), "H2D y shard"));
    TRY(cuda_status(cudaMemcpyAsync(rr.perm.as<void>(), perm[r].data(), sizeof(int64_t) * rows,
                                    cudaMemcpyHostToDevice, st), "H2D row order"));
    TRY(cuda_status(cudaMemcpyAsync(rr.rowmap.as<void>(), rowmap[r].data(), sizeof(int64_t) * n,
                                    cudaMemcpyHostToDevice, st), "H2D row map"));
    launch_gather_rows(dtype, rr.xs.as<void>(), rr.perm.as<int64_t>(), rows, k, rr.sx.as<void>(), st);
    launch_gather_rows(dtype, rr.ys.as<void>(), rr.perm.as<int64_t>(), rows, m, rr.sy.as<void>(), st);
    sub->launches += 2;
    TRY(cuda_status(cudaGetLastError(), "gather rows"));
    // the host routing tables must outlive the async copies above
    return cuda_status(cudaStreamSynchronize(st), "stream synchronize");
  }));

  // ---- phase B: rows to their fold's owner (whole folds)
  if (whole && G > 1) {
    // send offsets within each shard's gathered rows, receive offsets within each owner's compact rows
    std::vector<std::vector<int64_t>> soff(G, std::vector<int64_t>(G + 1, 0)), roff(G, std::vector<int64_t>(G + 1, 0));
    for (int r = 0; r < G; ++r)
      for (int o = 0; o < G; ++o) soff[r][o + 1] = soff[r][o] + sc[r][o];
    for (int o = 0; o < G; ++o)
      for (int r = 0; r < G; ++r) roff[o][r + 1] = roff[o][r] + sc[r][o];
    for (int mat = 0; mat < 2; ++mat) {
      const int64_t w = mat ? m : k;
      auto sendp = [&](int r, int o) { return (mat ? R[r]->sy : R[r]->sx).as<char>() + e * soff[r][o] * w; };
      auto recvp = [&](int o, int r) { return (mat ? R[o]->ry : R[o]->rx).as<char>() + e * roff[o][r] * w; };
      if (ctx->nccl) {
        const NcclApi& api = nccl();
        TRY(nccl_status(api.GroupStart(), "ncclGroupStart"));
        for (int r = 0; r < G; ++r)
          for (int o = 0; o < G; ++o) {
            if (sc[r][o])
              api.Send(sendp(r, o), (size_t)(sc[r][o] * w), nt, o, (ncclComm_t)ctx->comms[r], ctx->ranks[r]->stream);
            if (sc[o][r])
              api.Recv(recvp(r, o), (size_t)(sc[o][r] * w), nt, o, (ncclComm_t)ctx->comms[r], ctx->ranks[r]->stream);
          }
        TRY(nccl_status(api.GroupEnd(), "ncclGroupEnd (row exchange)"));
      } else {
        for (int r = 0; r < G; ++r)
          for (int o = 0; o < G; ++o)
            if (sc[r][o]) {
              TRY(cuda_status(cudaSetDevice(ctx->ranks[r]->device), "cudaSetDevice"));
              TRY(cuda_status(cudaMemcpyPeerAsync(recvp(o, r), ctx->ranks[o]->device, sendp(r, o), ctx->ranks[r]->device,
                                                  e * sc[r][o] * w, ctx->ranks[r]->stream),
                              "peer copy (row exchange)"));
            }
        TRY(sync_all());
      }
    }
  } else if (whole) {  // one rank: its gathered shard is the whole data in owner (= original) order
    RankRun& rr = *R[0];
    TRY(cuda_status(cudaSetDevice(ctx->ranks[0]->device), "cudaSetDevice"));
    TRY(cuda_status(cudaMemcpyAsync(rr.rx.as<void>(), rr.sx.as<void>(), e * n * k, cudaMemcpyDeviceToDevice,
                                    ctx->ranks[0]->stream), "D2D"));
    TRY(cuda_status(cudaMemcpyAsync(rr.ry.as<void>(), rr.sy.as<void>(), e * n * m, cudaMemcpyDeviceToDevice,
                                    ctx->ranks[0]->stream), "D2D"));
  }

  // ---- phase C (per rank): the owned folds' Gram over the compacted rows
  if (whole)
    TRY(par([&](int r) -> Status {
      RankRun& rr = *R[r];
      return rr.plan.gram(rr.rx.as<void>(), k, rr.ry.as<void>(), m, shift.data(), nullptr, rr.rowmap.as<int64_t>(),
                          rr.nrecv);
    }));

  // ---- phase D: the run's single collective -- every rank's partial Gram, in rank order, on every rank
  const int64_t kp2 = R[0]->plan.partial_count();
  for (int r = 0; r < G; ++r) {
    TRY(cuda_status(cudaSetDevice(ctx->ranks[r]->device), "cudaSetDevice"));
    TRY(R[r]->gathered.ensure(sizeof(double) * G * kp2));
  }
  if (ctx->nccl) {
    const NcclApi& api = nccl();
    TRY(nccl_status(api.GroupStart(), "ncclGroupStart"));
    for (int r = 0; r < G; ++r)
      api.AllGather(R[r]->plan.local(), R[r]->gathered.as<void>(), (size_t)kp2, ncclDouble, (ncclComm_t)ctx->comms[r],
                    ctx->ranks[r]->stream);
    TRY(nccl_status(api.GroupEnd(), "ncclGroupEnd (partial all-gather)"));
  } else {
    TRY(sync_all());
    for (int r = 0; r < G; ++r)
      for (int s2 = 0; s2 < G; ++s2) {
        TRY(cuda_status(cudaSetDevice(ctx->ranks[r]->device), "cudaSetDevice"));
        TRY(cuda_status(cudaMemcpyPeerAsync(R[r]->gathered.as<double>() + (int64_t)s2 * kp2, ctx->ranks[r]->device,
                                            R[s2]->plan.local(), ctx->ranks[s2]->device, sizeof(double) * kp2,
                                            ctx->ranks[r]->stream),
                        "peer copy (partial all-gather)"));
      }
    TRY(sync_all());
  }

  // ---- phase E (per rank): tree sum + the emitted folds' epilogue, copied into the caller's arrays
  TRY(par([&](int r) -> Status {
    RankRun& rr = *R[r];
    cudaStream_t st = ctx->ranks[r]->stream;
    const int64_t no = rr.oe - rr.ob;
    const size_t nxx = (size_t)ncfg * std::max<int64_t>(no, 1) * k * k, nxy = (size_t)ncfg * std::max<int64_t>(no, 1) * k * m;
    TRY(rr.xtx.ensure(sizeof(double) * nxx));
    TRY(rr.xty.ensure(sizeof(double) * nxy));
    TRY(rr.mx.ensure(sizeof(double) * std::max<int64_t>(no, 1) * k));
    TRY(rr.my.ensure(sizeof(double) * std::max<int64_t>(no, 1) * m));
    TRY(rr.sdx.ensure(sizeof(double) * std::max<int64_t>(no, 1) * k));
    TRY(rr.sdy.ensure(sizeof(double) * std::max<int64_t>(no, 1) * m));
    TRY(rr.plan.finish(rr.gathered.as<double>(), G, nullptr, cfgs, ncfg, rr.xtx.as<double>(), rr.xty.as<double>(),
                       rr.mx.as<double>(), rr.my.as<double>(), rr.sdx.as<double>(), rr.sdy.as<double>()));
    if (no == 0) return Status::Ok();
    auto d2h = [&](double* dst, const double* src, int64_t count, const char* what) -> Status {
      if (!dst) return Status::Ok();
      return cuda_status(cudaMemcpyAsync(dst, src, sizeof(double) * count, cudaMemcpyDeviceToHost, st), what);
    };
    for (int32_t c = 0; c < ncfg; ++c) {
      TRY(d2h(xtx + ((size_t)c * p + rr.ob) * k * k, rr.xtx.as<double>() + (size_t)c * no * k * k, no * k * k, "D2H xtx"));
      TRY(d2h(xty + ((size_t)c * p + rr.ob) * k * m, rr.xty.as<double>() + (size_t)c * no * k * m, no * k * m, "D2H xty"));
      // FoldStats fill rules, core.hpp:95-105: means iff any flag, stds iff that side is scaled
      const uint32_t cf = cfgs[c];
      if (cf) {
        TRY(d2h(mean_x ? mean_x + ((size_t)c * p + rr.ob) * k : nullptr, rr.mx.as<double>(), no * k, "D2H mean_x"));
        TRY(d2h(mean_y ? mean_y + ((size_t)c * p + rr.ob) * m : nullptr, rr.my.as<double>(), no * m, "D2H mean_y"));
      }
      if (cf & CVG_SCALE_X)
        TRY(d2h(std_x ? std_x + ((size_t)c * p + rr.ob) * k : nullptr, rr.sdx.as<double>(), no * k, "D2H std_x"));
      if (cf & CVG_SCALE_Y)
        TRY(d2h(std_y ? std_y + ((size_t)c * p + rr.ob) * m : nullptr, rr.sdy.as<double>(), no * m, "D2H std_y"));
    }
    return cuda_status(cudaStreamSynchronize(st), "stream synchronize");
  }));
  // every fold emitted exactly once
  std::vector<int> emitted(p, 0);
  for (int r = 0; r < G; ++r)
    for (int32_t f = R[r]->ob; f < R[r]->oe; ++f) ++emitted[f];
  for (int32_t f = 0; f < p; ++f)
    if (emitted[f] != 1) return Status::Err(CVG_E_CUDA, "internal: fold " + std::to_string(f + 1) + " emitted " +
                                                            std::to_string(emitted[f]) + " times");
  (void)counts;
#undef TRY
  return Status::Ok();
}

}  // namespace cvg
