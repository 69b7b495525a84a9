#pragma once
#include "common.cuh"

namespace adask {
int hess_mult_impl(adask_ctx* ctx, int dtype, const void* A, int64_t n, int64_t d, int64_t lda,
                   const double* X, int64_t c, int64_t ldx, double nu2, const double* lam,
                   const double* B, int64_t ldb, double* out, int64_t ldo, uint32_t flags,
                   cudaStream_t st);
int vec_hess_finish_impl(adask_ctx* ctx, const double* part, int64_t d, int64_t c, int64_t ld,
                         const double* X, double nu2, const double* lam, const double* B,
                         double* out, cudaStream_t st);
// H [x0, x1] with one pass over A (see hessmult.cu); *fused = 0 if not eligible.
int hess_mult_pair_impl(adask_ctx* ctx, int dtype, const void* A, int64_t n, int64_t d, int64_t lda,
                        const double* x0, const double* B0, double* out0, const double* x1, const double* B1,
                        double* out1, double nu2, const double* lam, cudaStream_t st, int* fused,
                        int partial = 0);
}  // namespace adask
