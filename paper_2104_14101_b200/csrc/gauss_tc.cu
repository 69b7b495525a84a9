// TF32 tensor-core Gaussian sketch (tcgen05) -- see gauss.cu.
#include "common.cuh"

namespace adask {
int gauss_tc_impl(adask_ctx* ctx, const float* A, int64_t n_local, int64_t d, int64_t lda,
                  int64_t row0, int64_t m, uint64_t key, float* SA, int64_t ldsa, bool accumulate,
                  cudaStream_t st) {
  (void)ctx; (void)A; (void)n_local; (void)d; (void)lda; (void)row0; (void)m; (void)key; (void)SA;
  (void)ldsa; (void)accumulate; (void)st;
  return fail(ADASK_E_ARG, "TF32 tensor-core Gaussian sketch not available in this build");
}
}  // namespace adask
