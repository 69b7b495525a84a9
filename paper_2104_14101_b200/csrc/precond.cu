// Sketched-Hessian preconditioner H_S = SA^T SA + nu^2 Lam.
// reference: preconditioner.py:26-74 (Preconditioner, build, solve).
//
// build: m >= d (ties dense, :63) -> Gram H_S (d x d) on the lower triangle
//        with nu^2 lam folded into the GEMM epilogue, then Cholesky + L^-1;
//        m <  d -> capacitance W_S = (SA / lam) SA^T + nu^2 I (m x m), same.
// apply: dense    out = L^-T (L^-1 z)              (two triangular row GEMVs)
//        woodbury out = (y - SA^T L^-T L^-1 SA y / lam) / nu^2,  y = z / lam
#include "blas2.cuh"
#include "chol.cuh"
#include <cstdlib>

#include "common.cuh"
#include "gemm.cuh"
#include "precond.cuh"

namespace adask {

int precond_apply_impl(adask_ctx* ctx, const adask_precond* P, const double* Z, int64_t c,
                       int64_t ldz, double* out, int64_t ldo, cudaStream_t st) {
  if (!P) return fail(ADASK_E_ARG, "null preconditioner");
  if (c < 1 || ldz < P->d || ldo < P->d) return fail(ADASK_E_DIM, "precond_apply: bad shape");
  const double esz = P->dtype == ADASK_F64 ? 8.0 : 4.0;
  const double bytes = P->path == 0 ? (double)P->k * P->k * esz
                                    : (2.0 * P->m * P->d + (double)P->m * P->m) * esz;
  ProfScope prof(ctx, PK_APPLY, st, bytes * c);
  for (int64_t j = 0; j < c; ++j) {
    const double* z = Z + j * ldz;
    double* o = out + j * ldo;
    if (P->path == 0) {
      void* wsp = nullptr;
      ADASK_TRY(ctx->ws[WS_APPLY].get((size_t)P->k * sizeof(double), st, &wsp));
      double* t = (double*)wsp;
      ADASK_TRY(gemv_rows(ctx, P->dtype, P->Linv, P->k, P->k, P->kp, z, 1.0, t, 1, st));
      ADASK_TRY(gemv_rows(ctx, P->dtype, P->LinvT, P->k, P->k, P->kp, t, 1.0, o, 2, st));
    } else {
      ADASK_TRY(woodbury_apply(ctx, P->dtype, P->SA, P->m, P->d, P->ldsa, P->Linv, P->LinvT, P->kp,
                               P->lam, P->nu2, z, o, st));
    }
  }
  return ADASK_OK;
}

static void free_precond(adask_precond* P) {
  if (!P) return;
  // one stream-ordered block: lam | L | Linv | LinvT
  if (P->lam) cudaFreeAsync(P->lam, P->stream);
  delete P;
}

}  // namespace adask

using namespace adask;

namespace adask {
template <typename T>
__global__ void k_add_diag(T* M, int64_t ldm, int64_t k, double nu2, const double* lam) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < k) M[i * ldm + i] = (T)((double)M[i * ldm + i] + nu2 * (lam ? lam[i] : 1.0));
}

// build() (preconditioner.py:60-74).  SA holds m_rows rows of the m x d
// sketch; m_rows < m only for a row-sharded dense build, where SA is this
// rank's reduce-scattered slice: the Gram of the slice is all-reduced (sum
// over ranks = SA^T SA) before nu^2 Lam is added and the factor is formed.
int precond_build_impl(adask_ctx* ctx, int dtype, const void* SA, int64_t m_rows, int64_t m, int64_t d,
                       int64_t ldsa, double nu, const double* lam, const GramReduce* reduce, adask_precond** out,
                       int64_t* info_host, cudaStream_t st) {
  if (!out || !lam || (m_rows > 0 && !SA)) return fail(ADASK_E_ARG, "precond_build: null argument");
  if (m < 1 || d < 1 || ldsa < d || m_rows < 0 || m_rows > m)
    return fail(ADASK_E_DIM, "precond_build: bad shape m=%lld d=%lld", (long long)m, (long long)d);
  if (dtype != ADASK_F64 && dtype != ADASK_F32) return fail(ADASK_E_ARG, "bad dtype");
  if (m_rows != m && (m < d || !reduce)) return fail(ADASK_E_ARG, "precond_build: partial rows need the dense path");
  const size_t esz = dtype == ADASK_F64 ? 8 : 4;
  adask_precond* P = new adask_precond();
  P->device = ctx->device;
  P->dtype = dtype;
  P->path = m >= d ? 0 : 1;
  P->m = m;
  P->d = d;
  P->k = m >= d ? d : m;
  P->SA = m_rows == m ? SA : nullptr;  // a sharded dense build keeps no full SA (its apply never reads it)
  P->ldsa = ldsa;
  P->nu = nu;
  P->nu2 = nu * nu;
  const int64_t k = P->k;
  // padded to the dataflow Cholesky's 32-row tiles (64 for the round-1 kernel's NB = 64 variant)
  const int64_t kp = cdiv(k, getenv("ADASK_CHOL_NB") ? 64 : 32) * (getenv("ADASK_CHOL_NB") ? 64 : 32);
  P->kp = kp;
  P->stream = st;
  const size_t lam_bytes = align_up((size_t)d * sizeof(double), 256);
  const size_t mat = align_up((size_t)kp * kp * esz, 256);
  char* blk = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&blk, lam_bytes + 3 * mat, st);
  if (e == cudaSuccess) {
    P->lam = (double*)blk;
    P->L = blk + lam_bytes;
    P->Linv = blk + lam_bytes + mat;
    P->LinvT = blk + lam_bytes + 2 * mat;
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    free_precond(P);
    return fail(ADASK_E_NOMEM, "precond_build: cudaMalloc: %s", cudaGetErrorString(e));
  }
  int s = ADASK_OK;
  const double gram_flops = m >= d ? (double)m_rows * d * (d + 1) : (double)m * (m + 1) * d;
  // the factor (k^3/3) and its triangular inverse (k^3/3); L^-T is a transpose
  const double chol_flops = 2.0 * (double)k * k * k / 3.0;
  ProfScope prof(ctx, PK_BUILD, st, (double)m_rows * d * esz, gram_flops + chol_flops);
  do {
    e = cudaMemcpyAsync(P->lam, lam, (size_t)d * sizeof(double), cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) {
      s = fail(ADASK_E_CUDA, "copy lam: %s", cudaGetErrorString(e));
      break;
    }
    void* wsp = nullptr;
    const size_t gram_bytes = align_up((size_t)kp * kp * esz, 256);
    s = ctx->ws[WS_GRAM].get(gram_bytes + (size_t)d * sizeof(double), st, &wsp);
    if (s) break;
    void* M = wsp;
    {
      ProfScope pg(ctx, PK_GRAM, st, (double)m_rows * d * esz, gram_flops);
      if (P->path == 0 && m_rows != m) {
        // sharded: partial Gram of this rank's rows, all-reduce, then nu^2 Lam
        s = gram_dense(ctx, dtype, SA, m_rows, d, ldsa, 0.0, nullptr, M, kp, st);
        if (!s) s = (*reduce)(M, d * kp, dtype);
        if (!s) {
          if (dtype == ADASK_F64)
            k_add_diag<double><<<(unsigned)cdiv(d, 256), 256, 0, st>>>((double*)M, kp, d, P->nu2, P->lam);
          else
            k_add_diag<float><<<(unsigned)cdiv(d, 256), 256, 0, st>>>((float*)M, kp, d, P->nu2, P->lam);
          cudaError_t le = cudaGetLastError();
          if (le != cudaSuccess) s = fail(ADASK_E_CUDA, "k_add_diag: %s", cudaGetErrorString(le));
          else ctx->launches++;
        }
      } else if (P->path == 0) {
        // H_S = SA^T SA + nu^2 diag(lam)   (preconditioner.py:70)
        s = gram_dense(ctx, dtype, SA, m, d, ldsa, P->nu2, P->lam, M, kp, st);
      } else {
        // W_S = (SA * (1/lam)) SA^T + nu^2 I   (preconditioner.py:72-73)
        s = gram_woodbury(ctx, dtype, SA, m, d, ldsa, P->nu2, P->lam, M, kp, st);
      }
    }
    if (s) break;
    ProfScope pc(ctx, PK_CHOL, st, (double)k * k * esz, chol_flops);
    s = pad_identity(ctx, dtype, M, k, kp, st);
    if (s) break;
    s = chol_factor_inverse(ctx, dtype, M, k, kp, P->L, P->Linv, P->LinvT, info_host, st);
  } while (0);
  if (s != ADASK_OK) {
    cudaStreamSynchronize(st);
    free_precond(P);
    return s;
  }
  *out = P;
  return ADASK_OK;
}
}  // namespace adask

extern "C" int adask_precond_build(adask_ctx* ctx, int dtype, const void* SA, int64_t m, int64_t d,
                                   int64_t ldsa, double nu, const double* lam, adask_precond** out,
                                   int64_t* info_host, void* stream) {
  ADASK_TRY(use_device(ctx));
  return precond_build_impl(ctx, dtype, SA, m, m, d, ldsa, nu, lam, nullptr, out, info_host, S(stream));
}

extern "C" int adask_precond_destroy(adask_precond* P) {
  if (!P) return ADASK_OK;
  int cur = -1;
  const int dev = P->device;
  cudaGetDevice(&cur);
  if (cur != dev) cudaSetDevice(dev);
  free_precond(P);  // stream-ordered free on the build stream
  if (cur >= 0 && cur != dev) cudaSetDevice(cur);
  return ADASK_OK;
}

extern "C" int adask_precond_path(const adask_precond* P) { return P ? P->path : -1; }

extern "C" int adask_precond_factor(const adask_precond* P, const void** L, int64_t* k, int* dtype) {
  if (!P) return fail(ADASK_E_ARG, "null preconditioner");
  if (L) *L = P->L;
  if (k) *k = P->k;
  if (dtype) *dtype = P->dtype;
  return ADASK_OK;
}

extern "C" int adask_precond_apply(adask_ctx* ctx, const adask_precond* P, const double* Z, int64_t c,
                                   int64_t ldz, double* out, int64_t ldo, void* stream) {
  ADASK_TRY(use_device(ctx));
  return precond_apply_impl(ctx, P, Z, c, ldz, out, ldo, S(stream));
}

namespace adask {
template <typename T>
__global__ void k_mirror_lower(T* M, int64_t k, int64_t ld) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= k * k) return;
  int64_t i = e / k, j = e % k;
  if (j > i) M[i * ld + j] = M[j * ld + i];
}
}  // namespace adask

extern "C" int adask_gram(adask_ctx* ctx, int dtype, const void* A, int64_t n, int64_t d, int64_t lda,
                          double nu2, const double* lam, void* out, int64_t ldo, void* stream) {
  return adask_gram_ex(ctx, dtype, A, n, d, lda, nu2, lam, dtype, out, ldo, stream);
}

extern "C" int adask_gram_ex(adask_ctx* ctx, int dtype, const void* A, int64_t n, int64_t d, int64_t lda,
                             double nu2, const double* lam, int out_dtype, void* out, int64_t ldo, void* stream) {
  ADASK_TRY(use_device(ctx));
  if (n < 0 || d < 1 || lda < d || ldo < d) return fail(ADASK_E_DIM, "gram: bad shape");
  if ((dtype != ADASK_F64 && dtype != ADASK_F32) || (out_dtype != ADASK_F64 && out_dtype != ADASK_F32) ||
      (dtype == ADASK_F64 && out_dtype == ADASK_F32))
    return fail(ADASK_E_ARG, "gram: unsupported dtype pair");
  cudaStream_t st = S(stream);
  ADASK_TRY(gram::gram_tc(ctx, dtype, A, lda, n, d, false, nullptr, lam ? nu2 : 0.0, lam, out, ldo,
                          out_dtype == ADASK_F64 && dtype == ADASK_F32, st));
  if (out_dtype == ADASK_F64)
    k_mirror_lower<double><<<(unsigned)cdiv(d * d, 256), 256, 0, st>>>((double*)out, d, ldo);
  else
    k_mirror_lower<float><<<(unsigned)cdiv(d * d, 256), 256, 0, st>>>((float*)out, d, ldo);
  ADASK_LAUNCHED(ctx);
  return ADASK_OK;
}

extern "C" int adask_gram_woodbury(adask_ctx* ctx, int dtype, const void* SA, int64_t m, int64_t d, int64_t ldsa,
                                   double nu2, const double* lam, void* out, int64_t ldo, void* stream) {
  ADASK_TRY(use_device(ctx));
  if (m < 1 || d < 1 || ldsa < d || ldo < m || !lam) return fail(ADASK_E_DIM, "gram_woodbury: bad shape");
  if (dtype != ADASK_F64 && dtype != ADASK_F32) return fail(ADASK_E_ARG, "bad dtype");
  cudaStream_t st = S(stream);
  ADASK_TRY(gram_woodbury(ctx, dtype, SA, m, d, ldsa, nu2, lam, out, ldo, st));
  if (dtype == ADASK_F64)
    k_mirror_lower<double><<<(unsigned)cdiv(m * m, 256), 256, 0, st>>>((double*)out, m, ldo);
  else
    k_mirror_lower<float><<<(unsigned)cdiv(m * m, 256), 256, 0, st>>>((float*)out, m, ldo);
  ADASK_LAUNCHED(ctx);
  return ADASK_OK;
}

extern "C" int adask_precond_copy_factor(adask_ctx* ctx, const adask_precond* P, int which, void* dst,
                                         int64_t ldd, void* stream) {
  ADASK_TRY(use_device(ctx));
  if (!P || !dst || ldd < P->k) return fail(ADASK_E_ARG, "copy_factor: bad arguments");
  const size_t esz = P->dtype == ADASK_F64 ? 8 : 4;
  const void* src = which == 0 ? P->L : which == 1 ? P->Linv : P->LinvT;
  ADASK_CUDA(cudaMemcpy2DAsync(dst, (size_t)ldd * esz, src, (size_t)P->kp * esz, (size_t)P->k * esz,
                               (size_t)P->k, cudaMemcpyDeviceToDevice, S(stream)));
  return ADASK_OK;
}
