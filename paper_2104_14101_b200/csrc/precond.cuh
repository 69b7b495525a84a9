#pragma once
#include "common.cuh"

struct adask_precond {
  int device;
  int dtype;
  int path;  // 0 cholesky-d, 1 woodbury-m
  int64_t m, d, k;
  int64_t kp;    // k padded to a multiple of 64: leading dimension of L, Linv, LinvT
  cudaStream_t stream;  // build stream (allocations are stream-ordered on it)
  const void* SA;
  int64_t ldsa;
  double nu, nu2;
  double* lam;   // device copy, d
  void* L;       // k x k lower
  void* Linv;    // k x k lower
  void* LinvT;   // k x k upper (transpose of Linv)
};

#include <functional>

namespace adask {
// all-reduce of a partial Gram (M, count elements, dtype) for sharded builds
using GramReduce = std::function<int(void*, int64_t, int)>;
int precond_build_impl(adask_ctx* ctx, int dtype, const void* SA, int64_t m_rows, int64_t m, int64_t d,
                       int64_t ldsa, double nu, const double* lam, const GramReduce* reduce, adask_precond** out,
                       int64_t* info_host, cudaStream_t st);
int precond_apply_impl(adask_ctx* ctx, const adask_precond* P, const double* Z, int64_t c,
                       int64_t ldz, double* out, int64_t ldo, cudaStream_t st);
}  // namespace adask
