#pragma once
#include "common.cuh"

namespace adask {
int sketch_sjlt_impl(adask_ctx* ctx, int dtype, const void* A, int64_t n_local, int64_t d,
                     int64_t lda, int64_t row0, int64_t n_total, int64_t m, int64_t s,
                     const adask_pcg64* g, const int64_t* rows_host, uint64_t sign_first,
                     void* SA, int64_t ldsa, uint32_t flags, cudaStream_t st);
int bucket_sort(adask_ctx* ctx, const int32_t* keys, int64_t nent, int64_t m, int32_t s,
                const int32_t** order_out, const int32_t** start_out, cudaStream_t st);
// Bulk-copy streamed bucket accumulation (sjlt_pipe.cu); *launched = 0 when
// the shape is not eligible (then the caller uses its own kernel).
int sjlt_accumulate_pipe(adask_ctx* ctx, int dtype, const void* A, int64_t d, int64_t lda, const int32_t* order,
                         const int32_t* start, const int32_t* sgn, int32_t s, int64_t m, void* SA, int64_t ldsa,
                         int accumulate, cudaStream_t st, int* launched);
}  // namespace adask
