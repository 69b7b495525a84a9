#pragma once
#include "common.cuh"

namespace adask {
// Factor the symmetric k x k matrix M (lower triangle read; M is overwritten)
// into lower L and L^-1 (upper triangles zeroed).  Synchronises to read info.
int cholesky_inplace(adask_ctx* ctx, int dtype, void* M, int64_t k, int64_t ldm, void* L,
                     int64_t ldl, void* Li, int64_t ldi, int64_t* info_host, cudaStream_t st);
int transpose_impl(adask_ctx* ctx, int dtype, const void* in, int64_t ldi, int64_t k, void* out,
                   int64_t ldo, cudaStream_t st);
}  // namespace adask
