#pragma once
#include "common.cuh"

namespace adask {
// C = alpha * opA(A) diag(kscale) opB(B) + beta * C (+ dscal * dvec on the diagonal);
// lower -> only j <= i computed / written.  Split-K partials use ws[ws_slot].
int gemm_impl(adask_ctx* ctx, int dtype, int64_t M, int64_t N, int64_t K, double alpha,
              const void* A, int64_t lda, bool ta, const void* B, int64_t ldb, bool tb,
              const double* kscale, double beta, void* C, int64_t ldc, double dscal,
              const double* dvec, bool lower, cudaStream_t st, int ws_slot = WS_GEMM);

// Preconditioner Grams through cuBLAS (plain library SYRK / GEMM, FP64 and
// FP32 pipes, no TF32), written into a row-major buffer (lower triangle):
//   dense:    M = SA^T SA + nu2 diag(lam)            (d x d)
//   woodbury: M = (SA diag(1/lam)) SA^T + nu2 I      (m x m)
int gram_dense(adask_ctx* ctx, int dtype, const void* SA, int64_t m, int64_t d, int64_t ldsa, double nu2,
               const double* lam, void* M, int64_t ldm, cudaStream_t st);
int gram_woodbury(adask_ctx* ctx, int dtype, const void* SA, int64_t m, int64_t d, int64_t ldsa, double nu2,
                  const double* lam, void* M, int64_t ldm, cudaStream_t st);
void blas_release(adask_ctx* ctx);
}  // namespace adask
