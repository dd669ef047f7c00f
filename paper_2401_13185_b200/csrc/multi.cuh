// Multi-device contexts (multi.cu): several B200s behind one cvg_context.
#pragma once

#include <cstdint>
#include <vector>

#include "cvg_internal.cuh"

struct cvg_context;

namespace cvg {

// Per-rank sub-contexts on dev_ids[0 .. n) and, for distinct devices, one NCCL communicator each
// (else -- repeated devices, or CVG_EXCHANGE=peer -- the exchanges run as device-to-device copies).
Status multi_init(cvg_context* ctx, const int* dev_ids, int n);
void multi_destroy(cvg_context* ctx);
// run_all_folds across the context's ranks (host buffers); validation already done by the caller.
Status run_all_folds_multi(cvg_context* ctx, int dtype, const void* x, const void* y, int64_t n, int64_t k, int64_t m,
                           const int32_t* labels, int32_t p, const uint32_t* cfgs, int32_t ncfg,
                           const std::vector<int64_t>& counts, bool scal, double* xtx, double* xty, double* mean_x,
                           double* mean_y, double* std_x, double* std_y);

}  // namespace cvg
