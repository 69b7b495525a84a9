#pragma once
#include "common.cuh"

namespace adask {
int sketch_srht_impl(adask_ctx* ctx, int dtype, const void* A, int64_t n, int64_t d, int64_t lda,
                     const adask_pcg64* g, int64_t m, void* SA, int64_t ldsa, int64_t* idx_host,
                     uint32_t flags, cudaStream_t st);
}  // namespace adask
