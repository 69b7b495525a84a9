// Cholesky factorization with explicit triangular inverse, as ONE cooperative
// persistent kernel.
// reference: linalg.cholesky (linalg.py:30-44, LAPACK dpotrf via numpy) and
// the two tri_solve calls of every preconditioner solve (linalg.py:47-55).
//
// The k x k matrix (padded to kp = 64*nblk with an identity tail) is cut into
// 64 x 64 tiles.  One CTA per SM runs all phases, separated by grid-wide
// barriers (cooperative launch, no host round trips):
//   for each panel j:   diag   CTA 0 factors A_jj in SMEM, inverts L_jj -> Dinv_j
//                       trsm   L_ij = A_ij Dinv_j^T            (tile-parallel)
//                       syrk   A_il -= L_ij L_lj^T, j < l <= i (tile-parallel)
//   inverse by recursive doubling over super-blocks of s = 1, 2, 4, ... tiles:
//                       T  = L21 I11,  I21 = -I22 T             (tile-parallel)
//   finally L^-T is written tile-transposed for the row-GEMV apply.
// Tiles are staged in SMEM as fp64 (fp32 inputs are widened); each 64^3 tile
// product is a 4x4-per-thread register-blocked DFMA loop.  A non-positive or
// non-finite pivot records info = pivot + 1 (NotPositiveDefinite).
// The explicit L^-1 / L^-T turn every per-iteration solve into two
// bandwidth-bound GEMVs over an L2-resident matrix (blas2.cu).
#include <cooperative_groups.h>

#include <type_traits>

#include "chol.cuh"
#include "common.cuh"

namespace cg = cooperative_groups;

namespace adask {

// The kernel body is generic in the tile edge NB; NB = 64 and NB = 32 are
// both compiled (namespaces chol64 / chol32).  NB = 32 halves the length of the
// latency-bound diagonal factorization that sits on the critical path of
// every panel, at the price of twice as many panels.
namespace chol64 {
constexpr int NB = 64;
#include "chol_impl.cuh"
}  // namespace chol64
namespace chol32 {
constexpr int NB = 32;
#include "chol_impl.cuh"
}  // namespace chol32

template <typename T>
__global__ void k_pad_identity(T* M, int k, int kp) {
  // rows/cols >= k of the kp x kp matrix: identity
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)kp * kp) return;
  const int i = (int)(e / kp), j = (int)(e % kp);
  if (i < k && j < k) return;
  M[e] = (T)(i == j ? 1.0 : 0.0);
}

int pad_identity(adask_ctx* ctx, int dtype, void* M, int64_t k, int64_t kp, cudaStream_t st) {
  if (kp == k) return ADASK_OK;
  const unsigned g = (unsigned)cdiv(kp * kp, 256);
  if (dtype == ADASK_F64) k_pad_identity<double><<<g, 256, 0, st>>>((double*)M, (int)k, (int)kp);
  else k_pad_identity<float><<<g, 256, 0, st>>>((float*)M, (int)k, (int)kp);
  ADASK_LAUNCHED(ctx);
  return ADASK_OK;
}

int chol_df_launch(adask_ctx* ctx, int dtype, void* M, int64_t k, int64_t kp, void* L, void* Li, void* LiT,
                   int* info, cudaStream_t st, int* info_mapped);

static int chol_finish(adask_ctx* ctx, int* info, int64_t* info_host, cudaStream_t st) {
  if (ctx->defer_spd) {
    // the driver reads pinned_flags[1] after its next synchronization
    ADASK_CUDA(cudaMemcpyAsync(ctx->pinned_flags + 1, info, sizeof(int), cudaMemcpyDeviceToHost, st));
    if (info_host) *info_host = 0;
    return ADASK_OK;
  }
  ADASK_CUDA(cudaMemcpyAsync(ctx->pinned_flags, info, sizeof(int), cudaMemcpyDeviceToHost, st));
  ADASK_CUDA(cudaStreamSynchronize(st));
  const int h = ctx->pinned_flags[0];
  if (info_host) *info_host = h;
  if (h != 0) return fail(ADASK_E_NOT_SPD, "Matrix is not positive definite (leading minor %d)", h);
  return ADASK_OK;
}

int chol_factor_inverse(adask_ctx* ctx, int dtype, void* M, int64_t k, int64_t kp, void* L, void* Li,
                        void* LiT, int64_t* info_host, cudaStream_t st) {
  const size_t esz = dtype == ADASK_F64 ? 8 : 4;
  if (!getenv("ADASK_CHOL_OLD")) {
    // dataflow kernel (chol_df.cu): writes every tile of L, Li, LiT itself
    if (kp % 32 || kp < k) return fail(ADASK_E_ARG, "chol: bad padding");
    void* wsp = nullptr;
    ADASK_TRY(ctx->ws[WS_CHOL].get(256, st, &wsp));
    int* info = (int*)wsp;  // cleared by the kernel
    if (ctx->defer_spd) {
      // the kernel reports a failure into pinned_flags[1] itself (host-mapped)
      ADASK_TRY(chol_df_launch(ctx, dtype, M, k, kp, L, Li, LiT, info, st, ctx->pinned_flags + 1));
      if (info_host) *info_host = 0;
      return ADASK_OK;
    }
    ADASK_TRY(chol_df_launch(ctx, dtype, M, k, kp, L, Li, LiT, info, st, nullptr));
    return chol_finish(ctx, info, info_host, st);
  }
  // tile edge: 32 unless overridden (ADASK_CHOL_NB=64)
  int nb = 32;
  if (const char* e = getenv("ADASK_CHOL_NB")) nb = atoi(e) == 64 ? 64 : 32;
  if (kp % nb || kp < k) return fail(ADASK_E_ARG, "chol: bad padding");
  void* wsp = nullptr;
  ADASK_TRY(ctx->ws[WS_CHOL].get(256, st, &wsp));
  int* info = (int*)wsp;
  ADASK_CUDA(cudaMemsetAsync(info, 0, sizeof(int), st));
  ADASK_CUDA(cudaMemsetAsync(L, 0, (size_t)kp * kp * esz, st));
  ADASK_CUDA(cudaMemsetAsync(Li, 0, (size_t)kp * kp * esz, st));
  ADASK_CUDA(cudaMemsetAsync(LiT, 0, (size_t)kp * kp * esz, st));
  const int nblk = (int)(kp / nb);
  unsigned long long* tlog = nullptr;
  const bool trace = getenv("ADASK_CHOL_TRACE") != nullptr;
  if (trace) {
    ADASK_CUDA(cudaMallocAsync((void**)&tlog, (3 * nblk + 16) * sizeof(unsigned long long), st));
    ADASK_CUDA(cudaMemsetAsync(tlog, 0, (3 * nblk + 16) * sizeof(unsigned long long), st));
  }
  int grid = 0;
  if (nb == 64)
    ADASK_TRY(chol64::launch(ctx, dtype, M, k, kp, L, Li, LiT, info, tlog, st, &grid));
  else
    ADASK_TRY(chol32::launch(ctx, dtype, M, k, kp, L, Li, LiT, info, tlog, st, &grid));
  if (ctx->defer_spd && !trace) {
    // the driver reads pinned_flags[1] after its next synchronization
    ADASK_CUDA(cudaMemcpyAsync(ctx->pinned_flags + 1, info, sizeof(int), cudaMemcpyDeviceToHost, st));
    if (info_host) *info_host = 0;
    return ADASK_OK;
  }
  ADASK_CUDA(cudaMemcpyAsync(ctx->pinned_flags, info, sizeof(int), cudaMemcpyDeviceToHost, st));
  ADASK_CUDA(cudaStreamSynchronize(st));
  if (trace) {
    std::vector<unsigned long long> tl(3 * nblk + 16);
    cudaMemcpy(tl.data(), tlog, tl.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    cudaFree(tlog);
    double diag = (tl[1] - tl[0]) * 1e-3, trsm = 0, syrk = 0;
    for (int j = 0; j + 1 < nblk; ++j) {
      const unsigned long long t0 = j == 0 ? tl[1] : tl[3 * j];
      trsm += (tl[2 + 3 * j] - t0) * 1e-3;
      syrk += (tl[3 + 3 * j] - tl[2 + 3 * j]) * 1e-3;
    }
    fprintf(stderr, "[chol NB=%d k=%lld kp=%lld grid=%d] diag %.1f us, trsm %.1f us, syrk %.1f us, inverse %.1f us, "
            "transpose %.1f us, total %.1f us\n", nb, (long long)k, (long long)kp, grid, diag, trsm, syrk,
            (tl[3 * nblk + 2] - tl[3 * nblk + 1]) * 1e-3, (tl[3 * nblk + 3] - tl[3 * nblk + 2]) * 1e-3,
            (tl[3 * nblk + 3] - tl[0]) * 1e-3);
    fprintf(stderr, "[chol prologue] tile load %.2f us, diag factor %.2f us (pivots %.2f, inverse %.2f), store %.2f us\n",
            (tl[3 * nblk + 4] - tl[0]) * 1e-3, (tl[3 * nblk + 5] - tl[3 * nblk + 4]) * 1e-3,
            (tl[3 * nblk + 9] - tl[3 * nblk + 8]) * 1e-3, (tl[3 * nblk + 10] - tl[3 * nblk + 9]) * 1e-3,
            (tl[3 * nblk + 6] - tl[3 * nblk + 5]) * 1e-3);
  }
  const int h = ctx->pinned_flags[0];
  if (info_host) *info_host = h;
  if (h != 0) return fail(ADASK_E_NOT_SPD, "Matrix is not positive definite (leading minor %d)", h);
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
  const int64_t kp = cdiv(k, getenv("ADASK_CHOL_NB") ? 64 : 32) * (getenv("ADASK_CHOL_NB") ? 64 : 32);
  const size_t mat = (size_t)kp * kp * esz;
  char* work = nullptr;
  ADASK_CUDA(cudaMallocAsync((void**)&work, 4 * mat, st));
  void *Mp = work, *Lp = work + mat, *Ip = work + 2 * mat, *ITp = work + 3 * mat;
  ADASK_CUDA(cudaMemsetAsync(Mp, 0, mat, st));
  ADASK_CUDA(cudaMemcpy2DAsync(Mp, (size_t)kp * esz, M, (size_t)ldm * esz, (size_t)k * esz, (size_t)k,
                               cudaMemcpyDeviceToDevice, st));
  int s = pad_identity(ctx, dtype, Mp, k, kp, st);
  if (s == ADASK_OK) s = chol_factor_inverse(ctx, dtype, Mp, k, kp, Lp, Ip, ITp, info_host, st);
  if (s == ADASK_OK) {
    cudaMemcpy2DAsync(L, (size_t)k * esz, Lp, (size_t)kp * esz, (size_t)k * esz, (size_t)k,
                      cudaMemcpyDeviceToDevice, st);
    if (Linv)
      cudaMemcpy2DAsync(Linv, (size_t)k * esz, Ip, (size_t)kp * esz, (size_t)k * esz, (size_t)k,
                        cudaMemcpyDeviceToDevice, st);
  }
  cudaFreeAsync(work, st);
  return s;
}
