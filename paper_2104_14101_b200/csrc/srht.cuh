#pragma once
#include <vector>

#include "common.cuh"

namespace adask {
int sketch_srht_impl(adask_ctx* ctx, int dtype, const void* A, int64_t n, int64_t d, int64_t lda,
                     const adask_pcg64* g, int64_t m, void* SA, int64_t ldsa, int64_t* idx_host,
                     uint32_t flags, cudaStream_t st, const std::vector<int64_t>* idx_pre = nullptr);
// choice(n_pad, m) after the n sign draws of g (the SRHT's host index draw)
int srht_draw_idx(const adask_pcg64* g, int64_t n, int64_t m, std::vector<int64_t>* idx);
// Incremental growth: the full normalized transform Y (n_pad x d, ld d) at
// the generator's signs, and the draw order perm (n_pad entries, host);
// then SA (+)= Y[perm[:m]] sqrt(n_pad / m).
int srht_transform_impl(adask_ctx* ctx, int dtype, const void* A, int64_t n, int64_t d, int64_t lda,
                        const adask_pcg64* g, void* Y, int64_t* perm_host, cudaStream_t st);
int srht_gather_impl(adask_ctx* ctx, int dtype, const void* Y, int64_t n_pad, int64_t d, const int64_t* perm_dev,
                     int64_t m, void* SA, int64_t ldsa, int accumulate, cudaStream_t st);
// Pipelined pruned FWHT (srht_pipe.cu): persistent TMA-fed tile passes.
int fwht_pipe_eligible(int dtype, const void* A, int64_t n, int64_t n_pad, int64_t lda, int64_t m, bool selected);
int fwht_select_pipe(adask_ctx* ctx, int dtype, const void* A, int64_t n, int64_t d, int64_t lda,
                     const uint32_t* sgn, int64_t n_pad, const int64_t* idx, int64_t m, void* out, int64_t ldo,
                     double c1, double c2, int accumulate, cudaStream_t st, int hybrid = 0);
int fwht_tile_pass2(adask_ctx* ctx, int dtype, int L2, const void* Z, int64_t G, int64_t d, int64_t nslots,
                    const int32_t* d_slot_start, const int32_t* d_ent_hi, const int32_t* d_ent_k, void* out,
                    int64_t ldo, double c1, double c2, int accumulate, cudaStream_t st);
int fwht_build_map2(adask_ctx* ctx, const int32_t* pos, int64_t m, int32_t* map2, int64_t rows, cudaStream_t st);
// Fused SRHT (srht_fused.cu): sign draws, both passes and the selection in one
// persistent kernel with Z L2-resident.  sgn: n_pad-bit scratch for the signs.
int srht_fused_eligible(int dtype, const void* A, int64_t n, int64_t n_pad, int64_t lda);
int srht_fused(adask_ctx* ctx, int dtype, const void* A, int64_t n, int64_t d, int64_t lda, const adask_pcg64* g,
               uint32_t* sgn, int64_t n_pad, const int64_t* idx, int64_t m, void* out, int64_t ldo, double c1,
               double c2, int accumulate, cudaStream_t st);
// 2^19 .. 2^22 padded rows: the fused kernel per 2^18-row sub-block + a combine of the partials.
int srht_fused_big_eligible(int dtype, const void* A, int64_t n, int64_t n_pad, int64_t lda, int64_t m);
int srht_fused_big(adask_ctx* ctx, int dtype, const void* A, int64_t n, int64_t d, int64_t lda,
                   const adask_pcg64* g, uint32_t* sgn, int64_t n_pad, const int64_t* idx, int64_t m, void* out,
                   int64_t ldo, double c1, double c2, int accumulate, cudaStream_t st);
}  // namespace adask
