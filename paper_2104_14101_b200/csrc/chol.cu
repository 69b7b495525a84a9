// Cholesky factorization with explicit triangular inverse.
// reference: linalg.cholesky (linalg.py:30-44, LAPACK dpotrf via numpy) and
// the two tri_solve calls per preconditioner solve (linalg.py:47-55).
//
// Recursive blocked algorithm on device memory:
//   chol(M) -> (L, L^-1):
//     k <= 64 : one CTA factors the block in SMEM (right-looking) and inverts
//               it by row-parallel forward substitution;
//     else    : L11, L11^-1 = chol(M11)
//               L21  = M21 L11^-T                     (GEMM)
//               M22 -= L21 L21^T (lower)              (GEMM / SYRK)
//               L22, L22^-1 = chol(M22)
//               L^-1_21 = -L22^-1 (L21 L11^-1)        (2 GEMMs)
// All flops of the recursion run in gemm_impl (DFMA for fp64, FFMA fp32).
// A non-positive (or non-finite) pivot records info = pivot index + 1 in
// device memory; the caller checks it once (NotPositiveDefinite).
// Explicit L^-1 turns every per-iteration triangular solve into two
// bandwidth-bound GEMVs over an L2-resident matrix (blas2.cu).
#include "blas2.cuh"
#include "chol.cuh"
#include "common.cuh"
#include "gemm.cuh"

namespace adask {

constexpr int kLeaf = 64;

template <typename T>
__global__ void __launch_bounds__(256) k_chol_leaf(const T* __restrict__ M, int64_t ldm, int k,
                                                   T* __restrict__ L, int64_t ldl,
                                                   T* __restrict__ Li, int64_t ldi, int* info,
                                                   int64_t offset) {
  extern __shared__ double leaf_sm[];
  double(*S)[kLeaf + 1] = reinterpret_cast<double(*)[kLeaf + 1]>(leaf_sm);
  double(*X)[kLeaf + 1] = reinterpret_cast<double(*)[kLeaf + 1]>(leaf_sm + kLeaf * (kLeaf + 1));
  __shared__ int bad;
  const int tid = threadIdx.x;
  if (tid == 0) bad = 0;
  for (int e = tid; e < k * k; e += blockDim.x) {
    int i = e / k, j = e % k;
    S[i][j] = (j <= i) ? (double)M[(int64_t)i * ldm + j] : 0.0;
    X[i][j] = 0.0;
  }
  __syncthreads();
  for (int j = 0; j < k; ++j) {
    double p = S[j][j];
    if (!(p > 0.0) || !isfinite(p)) {
      if (tid == 0 && !bad) {
        bad = 1;
        atomicCAS(info, 0, (int)(offset + j + 1));
      }
    }
    const double djj = sqrt(p);
    __syncthreads();
    for (int i = j + 1 + tid; i < k; i += blockDim.x) S[i][j] = S[i][j] / djj;
    __syncthreads();
    if (tid == 0) S[j][j] = djj;
    const int w = k - j - 1;
    for (int e = tid; e < w * w; e += blockDim.x) {
      int i = j + 1 + e / w, l = j + 1 + e % w;
      if (l <= i) S[i][l] -= S[i][j] * S[l][j];
    }
    __syncthreads();
  }
  // X = L^-1, row by row; 4 threads cooperate on each column's dot product
  const int c = tid >> 2, part = tid & 3;
  for (int i = 0; i < k; ++i) {
    const double rd = 1.0 / S[i][i];
    double s = 0.0;
    if (c < i)
      for (int p = c + part; p < i; p += 4) s = fma(S[i][p], X[p][c], s);
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    if (part == 0) {
      if (c < i) X[i][c] = -s * rd;
      else if (c == i) X[i][c] = rd;
    }
    __syncthreads();
  }
  for (int e = tid; e < k * k; e += blockDim.x) {
    int i = e / k, j = e % k;
    L[(int64_t)i * ldl + j] = (T)(j <= i ? S[i][j] : 0.0);
    if (Li) Li[(int64_t)i * ldi + j] = (T)(j <= i ? X[i][j] : 0.0);
  }
}

template <typename T>
__global__ void k_zero_block(T* P, int64_t ld, int64_t r, int64_t c) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < r * c) P[(e / c) * ld + e % c] = (T)0;
}

template <typename T>
__global__ void k_transpose(const T* __restrict__ in, int64_t ldi, int64_t k, T* __restrict__ out,
                            int64_t ldo) {
  __shared__ T tile[32][33];
  const int64_t bx = (int64_t)blockIdx.x * 32, by = (int64_t)blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    int64_t i = by + r, j = bx + threadIdx.x;
    if (i < k && j < k) tile[r][threadIdx.x] = in[i * ldi + j];
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    int64_t i = bx + r, j = by + threadIdx.x;
    if (i < k && j < k) out[i * ldo + j] = tile[threadIdx.x][r];
  }
}

int transpose_impl(adask_ctx* ctx, int dtype, const void* in, int64_t ldi, int64_t k, void* out,
                   int64_t ldo, cudaStream_t st) {
  dim3 g((unsigned)cdiv(k, 32), (unsigned)cdiv(k, 32)), b(32, 8);
  if (dtype == ADASK_F64)
    k_transpose<double><<<g, b, 0, st>>>((const double*)in, ldi, k, (double*)out, ldo);
  else
    k_transpose<float><<<g, b, 0, st>>>((const float*)in, ldi, k, (float*)out, ldo);
  ADASK_LAUNCHED(ctx);
  return ADASK_OK;
}

struct CholRec {
  adask_ctx* ctx;
  int dtype;
  size_t esz;
  int* info;
  void* tmp;  // >= (k/2 + 64) * (k/2 + 64) elements
  cudaStream_t st;

  char* at(void* base, int64_t ld, int64_t i, int64_t j) const {
    return (char*)base + (size_t)(i * ld + j) * esz;
  }

  int zero(void* P, int64_t ld, int64_t r, int64_t c) {
    if (r <= 0 || c <= 0) return ADASK_OK;
    if (dtype == ADASK_F64)
      k_zero_block<double><<<(unsigned)cdiv(r * c, 256), 256, 0, st>>>((double*)P, ld, r, c);
    else
      k_zero_block<float><<<(unsigned)cdiv(r * c, 256), 256, 0, st>>>((float*)P, ld, r, c);
    ADASK_LAUNCHED(ctx);
    return ADASK_OK;
  }

  // M (destroyed below the diagonal of the trailing blocks), L, Li: k x k
  int run(void* M, int64_t ldm, void* L, int64_t ldl, void* Li, int64_t ldi, int64_t k, int64_t off) {
    if (k <= kLeaf) {
      const int smem = 2 * kLeaf * (kLeaf + 1) * (int)sizeof(double);
      if (dtype == ADASK_F64) {
        ADASK_CUDA(cudaFuncSetAttribute(k_chol_leaf<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        k_chol_leaf<double><<<1, 256, smem, st>>>((const double*)M, ldm, (int)k, (double*)L, ldl,
                                                  (double*)Li, ldi, info, off);
      } else {
        ADASK_CUDA(cudaFuncSetAttribute(k_chol_leaf<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        k_chol_leaf<float><<<1, 256, smem, st>>>((const float*)M, ldm, (int)k, (float*)L, ldl,
                                                 (float*)Li, ldi, info, off);
      }
      ADASK_LAUNCHED(ctx);
      return ADASK_OK;
    }
    int64_t k1 = ((k / 2) + kLeaf - 1) / kLeaf * kLeaf;
    if (k1 >= k) k1 = k - kLeaf;
    const int64_t k2 = k - k1;
    void* M11 = M;
    void* M21 = at(M, ldm, k1, 0);
    void* M22 = at(M, ldm, k1, k1);
    void* L11 = L;
    void* L21 = at(L, ldl, k1, 0);
    void* L22 = at(L, ldl, k1, k1);
    void* I11 = Li;
    void* I21 = at(Li, ldi, k1, 0);
    void* I22 = at(Li, ldi, k1, k1);
    ADASK_TRY(run(M11, ldm, L11, ldl, I11, ldi, k1, off));
    // L21 = M21 * I11^T          [k2 x k1]
    ADASK_TRY(gemm_impl(ctx, dtype, k2, k1, k1, 1.0, M21, ldm, false, I11, ldi, true, nullptr, 0.0,
                        L21, ldl, 0.0, nullptr, false, st));
    // M22 -= L21 L21^T  (lower)
    ADASK_TRY(gemm_impl(ctx, dtype, k2, k2, k1, -1.0, L21, ldl, false, L21, ldl, true, nullptr, 1.0,
                        M22, ldm, 0.0, nullptr, true, st));
    ADASK_TRY(run(M22, ldm, L22, ldl, I22, ldi, k2, off + k1));
    // tmp = L21 I11              [k2 x k1]
    ADASK_TRY(gemm_impl(ctx, dtype, k2, k1, k1, 1.0, L21, ldl, false, I11, ldi, false, nullptr, 0.0,
                        tmp, k1, 0.0, nullptr, false, st));
    // I21 = -I22 tmp             [k2 x k1]
    ADASK_TRY(gemm_impl(ctx, dtype, k2, k1, k2, -1.0, I22, ldi, false, tmp, k1, false, nullptr, 0.0,
                        I21, ldi, 0.0, nullptr, false, st));
    // zero the upper blocks
    ADASK_TRY(zero(at(L, ldl, 0, k1), ldl, k1, k2));
    ADASK_TRY(zero(at(Li, ldi, 0, k1), ldi, k1, k2));
    return ADASK_OK;
  }
};

// M is consumed (its lower triangle is overwritten by Schur complements).
int cholesky_inplace(adask_ctx* ctx, int dtype, void* M, int64_t k, int64_t ldm, void* L,
                     int64_t ldl, void* Li, int64_t ldi, int64_t* info_host, cudaStream_t st) {
  const size_t esz = dtype == ADASK_F64 ? 8 : 4;
  const int64_t half = k / 2 + kLeaf;
  void* wsp = nullptr;
  ADASK_TRY(ctx->ws[WS_CHOL].get(256 + (size_t)half * half * esz, st, &wsp));
  int* info = (int*)wsp;
  ADASK_CUDA(cudaMemsetAsync(info, 0, sizeof(int), st));
  CholRec r{ctx, dtype, esz, info, (char*)wsp + 256, st};
  ADASK_TRY(r.run(M, ldm, L, ldl, Li, ldi, k, 0));
  int h = 0;
  ADASK_CUDA(cudaMemcpyAsync(ctx->pinned_flags, info, sizeof(int), cudaMemcpyDeviceToHost, st));
  ADASK_CUDA(cudaStreamSynchronize(st));
  h = ctx->pinned_flags[0];
  if (info_host) *info_host = h;
  if (h != 0)
    return fail(ADASK_E_NOT_SPD, "Matrix is not positive definite (leading minor %d)", h);
  return ADASK_OK;
}

}  // namespace adask

using namespace adask;

extern "C" int adask_cholesky(adask_ctx* ctx, int dtype, const void* M, int64_t k, int64_t ldm,
                              void* L, void* Linv, int64_t* info_host, void* stream) {
  ADASK_TRY(use_device(ctx));
  if (k < 1 || ldm < k || !M || !L) return fail(ADASK_E_DIM, "cholesky: bad shape");
  if (dtype != ADASK_F64 && dtype != ADASK_F32) return fail(ADASK_E_ARG, "bad dtype");
  cudaStream_t st = S(stream);
  const size_t esz = dtype == ADASK_F64 ? 8 : 4;
  // working copy of M (the recursion overwrites it)
  void* work = nullptr;
  ADASK_CUDA(cudaMallocAsync(&work, (size_t)k * k * esz, st));
  ADASK_CUDA(cudaMemcpy2DAsync(work, (size_t)k * esz, M, (size_t)ldm * esz, (size_t)k * esz, (size_t)k,
                               cudaMemcpyDeviceToDevice, st));
  void* li = Linv;
  void* li_tmp = nullptr;
  if (!li) {
    ADASK_CUDA(cudaMallocAsync(&li_tmp, (size_t)k * k * esz, st));
    li = li_tmp;
  }
  int s = cholesky_inplace(ctx, dtype, work, k, k, L, k, li, k, info_host, st);
  cudaFreeAsync(work, st);
  if (li_tmp) cudaFreeAsync(li_tmp, st);
  return s;
}
