#pragma once
#include "common.cuh"

namespace adask {
// Factor the symmetric kp x kp matrix M (lower triangle read, ld = kp, padded
// with an identity tail beyond k; M is overwritten) into L, L^-1 and L^-T
// (kp x kp, ld = kp).  One cooperative launch; synchronises to read info.
int chol_factor_inverse(adask_ctx* ctx, int dtype, void* M, int64_t k, int64_t kp, void* L, void* Li,
                        void* LiT, int64_t* info_host, cudaStream_t st);
// Set rows / columns >= k of a kp x kp matrix to the identity.
int pad_identity(adask_ctx* ctx, int dtype, void* M, int64_t k, int64_t kp, cudaStream_t st);
}  // namespace adask
