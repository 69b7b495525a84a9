#pragma once
#include "common.cuh"

namespace adask {
// out[i] = alpha * sum_j M[i, j] x[j]; mode 0 full, 1 lower (j <= i), 2 upper (j >= i)
int gemv_rows(adask_ctx* ctx, int dtype, const void* M, int64_t rows, int64_t cols, int64_t ld,
              const double* x, double alpha, double* out, int mode, cudaStream_t st);
// out = H_S^-1 z on the Woodbury path (preconditioner.py:49-52)
int woodbury_apply(adask_ctx* ctx, int dtype, const void* SA, int64_t m, int64_t d, int64_t ldsa,
                   const void* Linv, const void* LinvT, int64_t ldl, const double* lam, double nu2,
                   const double* z, double* out, cudaStream_t st);
}  // namespace adask
