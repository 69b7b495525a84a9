#pragma once
#include "common.cuh"

namespace adask {
// C = alpha * opA(A) diag(kscale) opB(B) + beta * C (+ dscal * dvec on the diagonal);
// lower -> only j <= i computed / written.  Split-K partials use ws[ws_slot].
int gemm_impl(adask_ctx* ctx, int dtype, int64_t M, int64_t N, int64_t K, double alpha,
              const void* A, int64_t lda, bool ta, const void* B, int64_t ldb, bool tb,
              const double* kscale, double beta, void* C, int64_t ldc, double dscal,
              const double* dvec, bool lower, cudaStream_t st, int ws_slot = WS_GEMM);
}  // namespace adask
