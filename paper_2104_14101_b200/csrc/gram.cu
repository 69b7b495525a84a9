// Preconditioner Grams (preconditioner.py:69-73) on cuBLAS: these are plain
// library GEMMs (SYRK for the dense d x d path, GEMM for the Woodbury m x m
// capacitance), run on the FP64 / FP32 pipes at 85-95% of peak, against ~40%
// for the hand-written register-blocked kernel (gemm.cu) they replace here.
// Row-major buffers are read as their column-major transposes; no TF32.
#include <cublas_v2.h>
#include <cstdlib>

#include "common.cuh"
#include "gemm.cuh"

namespace adask {

static int blas_handle(adask_ctx* ctx, cudaStream_t st, cublasHandle_t* out) {
  if (!ctx->blas) {
    cublasHandle_t h = nullptr;
    if (cublasCreate(&h) != CUBLAS_STATUS_SUCCESS) return fail(ADASK_E_CUDA, "cublasCreate failed");
    cublasSetMathMode(h, CUBLAS_PEDANTIC_MATH);  // no TF32 / reduced-precision shortcuts
    ctx->blas = h;
  }
  cublasHandle_t h = (cublasHandle_t)ctx->blas;
  if (cublasSetStream(h, st) != CUBLAS_STATUS_SUCCESS) return fail(ADASK_E_CUDA, "cublasSetStream failed");
  *out = h;
  return ADASK_OK;
}

void blas_release(adask_ctx* ctx) {
  if (ctx && ctx->blas) {
    cublasDestroy((cublasHandle_t)ctx->blas);
    ctx->blas = nullptr;
  }
}

#define ADASK_BLAS(expr)                                                                    \
  do {                                                                                      \
    cublasStatus_t _s = (expr);                                                             \
    if (_s != CUBLAS_STATUS_SUCCESS) return fail(ADASK_E_CUDA, "%s failed (%d)", #expr, (int)_s); \
  } while (0)

template <typename T>
__global__ void k_add_diag(T* M, int64_t ldm, int64_t k, double nu2, const double* lam) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < k) M[i * ldm + i] = (T)((double)M[i * ldm + i] + nu2 * (lam ? lam[i] : 1.0));
}

// T = SA diag(1/lam), row-major m x d, each entry SA[i][j] / lam[j] (the
// reference's SA / lam, preconditioner.py:72)
template <typename T>
__global__ void k_scale_cols(const T* SA, int64_t m, int64_t d, int64_t ldsa, const double* lam, T* out) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= m * d) return;
  const int64_t i = e / d, j = e - i * d;
  out[i * d + j] = (T)((double)SA[i * ldsa + j] / lam[j]);
}

int gram_dense(adask_ctx* ctx, int dtype, const void* SA, int64_t m, int64_t d, int64_t ldsa, double nu2,
               const double* lam, void* M, int64_t ldm, cudaStream_t st) {
  cublasHandle_t h;
  ADASK_TRY(blas_handle(ctx, st, &h));
  // column-major X = SA^T (d x m, ld = ldsa); C = X X^T, column-major upper =
  // row-major lower.  Up to d = 1024 cuBLAS' GEMM (full square) is faster
  // than its SYRK on this GPU (measured: tools/gemm_probe.py), above it SYRK.
  const bool split = !(getenv("ADASK_GRAM_SPLIT") && atoi(getenv("ADASK_GRAM_SPLIT")) == 0);
  if (d <= 1024 && split && d >= 256 && m >= 2048) {
    // only the lower triangle (row-major) is consumed: C[:, d1:] = X X2^T and
    // C11 = X1 X1^T, 3/4 of the square's flops in two GEMMs (measured at
    // d = 1024: m = 2048 / 4096 fp64 builds 0.69 -> 0.67 / 0.80 -> 0.75 ms,
    // m = 32768 fp32 1.76 -> 1.59 ms; no gain below m = 2048)
    const int d1 = (int)(d / 2 / 16 * 16), d2 = (int)d - d1;
    if (dtype == ADASK_F64) {
      const double one = 1.0, zero = 0.0;
      const double* X = (const double*)SA;
      ADASK_BLAS(cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_T, (int)d, d2, (int)m, &one, X, (int)ldsa, X + d1, (int)ldsa,
                             &zero, (double*)M + (int64_t)d1 * ldm, (int)ldm));
      ADASK_BLAS(cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_T, d1, d1, (int)m, &one, X, (int)ldsa, X, (int)ldsa, &zero,
                             (double*)M, (int)ldm));
    } else {
      const float one = 1.0f, zero = 0.0f;
      const float* X = (const float*)SA;
      ADASK_BLAS(cublasSgemm(h, CUBLAS_OP_N, CUBLAS_OP_T, (int)d, d2, (int)m, &one, X, (int)ldsa, X + d1, (int)ldsa,
                             &zero, (float*)M + (int64_t)d1 * ldm, (int)ldm));
      ADASK_BLAS(cublasSgemm(h, CUBLAS_OP_N, CUBLAS_OP_T, d1, d1, (int)m, &one, X, (int)ldsa, X, (int)ldsa, &zero,
                             (float*)M, (int)ldm));
    }
  } else if (d <= 1024) {
    if (dtype == ADASK_F64) {
      const double one = 1.0, zero = 0.0;
      ADASK_BLAS(cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_T, (int)d, (int)d, (int)m, &one, (const double*)SA,
                             (int)ldsa, (const double*)SA, (int)ldsa, &zero, (double*)M, (int)ldm));
    } else {
      const float one = 1.0f, zero = 0.0f;
      ADASK_BLAS(cublasSgemm(h, CUBLAS_OP_N, CUBLAS_OP_T, (int)d, (int)d, (int)m, &one, (const float*)SA,
                             (int)ldsa, (const float*)SA, (int)ldsa, &zero, (float*)M, (int)ldm));
    }
  } else if (dtype == ADASK_F64) {
    const double one = 1.0, zero = 0.0;
    ADASK_BLAS(cublasDsyrk(h, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N, (int)d, (int)m, &one, (const double*)SA,
                           (int)ldsa, &zero, (double*)M, (int)ldm));
  } else {
    const float one = 1.0f, zero = 0.0f;
    ADASK_BLAS(cublasSsyrk(h, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N, (int)d, (int)m, &one, (const float*)SA,
                           (int)ldsa, &zero, (float*)M, (int)ldm));
  }
  ctx->launches++;
  if (nu2 != 0.0) {
    if (dtype == ADASK_F64)
      k_add_diag<double><<<(unsigned)cdiv(d, 256), 256, 0, st>>>((double*)M, ldm, d, nu2, lam);
    else
      k_add_diag<float><<<(unsigned)cdiv(d, 256), 256, 0, st>>>((float*)M, ldm, d, nu2, lam);
    ADASK_LAUNCHED(ctx);
  }
  return ADASK_OK;
}

int gram_woodbury(adask_ctx* ctx, int dtype, const void* SA, int64_t m, int64_t d, int64_t ldsa, double nu2,
                  const double* lam, void* M, int64_t ldm, cudaStream_t st) {
  cublasHandle_t h;
  ADASK_TRY(blas_handle(ctx, st, &h));
  const size_t esz = dtype == ADASK_F64 ? 8 : 4;
  void* tw = nullptr;
  ADASK_TRY(ctx->ws[WS_GEMM].get((size_t)m * d * esz, st, &tw));
  if (dtype == ADASK_F64)
    k_scale_cols<double><<<(unsigned)cdiv(m * d, 256), 256, 0, st>>>((const double*)SA, m, d, ldsa, lam,
                                                                     (double*)tw);
  else
    k_scale_cols<float><<<(unsigned)cdiv(m * d, 256), 256, 0, st>>>((const float*)SA, m, d, ldsa, lam,
                                                                    (float*)tw);
  ADASK_LAUNCHED(ctx);
  // row-major W[i][j] = sum_k T[i][k] SA[j][k]: column-major C = Y^T P with
  // Y = SA^T, P = T^T (both d x m); C(i, j) = W[j][i], W symmetric
  if (dtype == ADASK_F64) {
    const double one = 1.0, zero = 0.0;
    ADASK_BLAS(cublasDgemm(h, CUBLAS_OP_T, CUBLAS_OP_N, (int)m, (int)m, (int)d, &one, (const double*)SA,
                           (int)ldsa, (const double*)tw, (int)d, &zero, (double*)M, (int)ldm));
  } else {
    const float one = 1.0f, zero = 0.0f;
    ADASK_BLAS(cublasSgemm(h, CUBLAS_OP_T, CUBLAS_OP_N, (int)m, (int)m, (int)d, &one, (const float*)SA,
                           (int)ldsa, (const float*)tw, (int)d, &zero, (float*)M, (int)ldm));
  }
  ctx->launches++;
  if (nu2 != 0.0) {
    if (dtype == ADASK_F64)
      k_add_diag<double><<<(unsigned)cdiv(m, 256), 256, 0, st>>>((double*)M, ldm, m, nu2, nullptr);
    else
      k_add_diag<float><<<(unsigned)cdiv(m, 256), 256, 0, st>>>((float*)M, ldm, m, nu2, nullptr);
    ADASK_LAUNCHED(ctx);
  }
  return ADASK_OK;
}

}  // namespace adask
