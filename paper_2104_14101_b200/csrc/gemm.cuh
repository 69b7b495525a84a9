#pragma once
#include "common.cuh"

namespace adask {
// C = alpha * opA(A) diag(kscale) opB(B) + beta * C (+ dscal * dvec on the diagonal);
// lower -> only j <= i computed / written.  Split-K partials use ws[ws_slot].
int gemm_impl(adask_ctx* ctx, int dtype, int64_t M, int64_t N, int64_t K, double alpha,
              const void* A, int64_t lda, bool ta, const void* B, int64_t ldb, bool tb,
              const double* kscale, double beta, void* C, int64_t ldc, double dscal,
              const double* dvec, bool lower, cudaStream_t st, int ws_slot = WS_GEMM);

// Preconditioner Grams on the FP64 tensor cores (gram.cu, DMMA SYRK), written
// into a row-major buffer (lower triangle):
//   dense:    M = SA^T SA + nu2 diag(lam)            (d x d)
//   woodbury: M = (SA diag(1/lam)) SA^T + nu2 I      (m x m)
int gram_dense(adask_ctx* ctx, int dtype, const void* SA, int64_t m, int64_t d, int64_t ldsa, double nu2,
               const double* lam, void* M, int64_t ldm, cudaStream_t st);
int gram_woodbury(adask_ctx* ctx, int dtype, const void* SA, int64_t m, int64_t d, int64_t ldsa, double nu2,
                  const double* lam, void* M, int64_t ldm, cudaStream_t st);
namespace gram {
// Lower triangle of X^T X (K-outer, X K x N) or (X diag(rl)) X^T (kc, X N x K)
// plus nu2 * (lam or 1) on the diagonal, DMMA tensor cores (gram.cu).
int gram_tc(adask_ctx* ctx, int dtype, const void* X, int64_t ld, int64_t K, int64_t N, bool kc,
            const double* rl, double nu2, const double* lam, void* M, int64_t ldm, bool out_f64, cudaStream_t st);
// C (M x N) = X^T Y (+ C when accumulate): X K x M, Y K x N row-major with
// 16-byte aligned rows, DMMA tensor cores with fp64 accumulation (gram.cu).
int gemm_tn_tc(adask_ctx* ctx, int dtype, const void* X, int64_t ldx, const void* Y, int64_t ldy, int64_t K,
               int64_t M, int64_t N, void* C, int64_t ldc, bool accumulate, cudaStream_t st);
}  // namespace gram
}  // namespace adask
