// Matrix-vector kernels for the preconditioner solves (preconditioner.py:42-53):
// row GEMV with triangular bounds (explicit L^-1 and L^-T applies replace the
// two LAPACK trsv calls of tri_solve, linalg.py:47-55) and the deterministic
// column GEMV (SA^T u) used by the Woodbury path.  Vectors are fp64; matrix
// elements are T.  No atomics.
#include "blas2.cuh"
#include "common.cuh"

namespace adask {

// out[i] = alpha * sum_{j in J(i)} M[i*ld + j] * x[j]   (+ beta_vec? handled by caller)
// mode 0: J = [0, cols), 1: J = [0, i] (lower), 2: J = [i, cols) (upper)
// One warp per row.  The matrix is small and L2-resident (explicit factor
// inverses, SA), so each warp issues up to 8 x 16-byte loads per lane before
// the first FMA: a 1024-wide fp64 row is two load rounds, not eight
// dependent ones (the load latency, not bandwidth, bounds this kernel).
template <typename T>
__global__ void __launch_bounds__(256) k_gemv_rows(const T* __restrict__ M, int64_t rows,
                                                   int64_t cols, int64_t ld,
                                                   const double* __restrict__ x, double alpha,
                                                   double* __restrict__ out, int mode, int vec) {
  pdl_wait();
  constexpr int CE = 16 / (int)sizeof(T);  // elements per 16-byte chunk
  constexpr int U = 8;
  const int lane = threadIdx.x & 31;
  const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (i >= rows) return;
  int64_t j0 = 0, j1 = cols;
  if (mode == 1) j1 = i + 1 < cols ? i + 1 : cols;
  if (mode == 2) j0 = i;
  const T* r = M + i * ld;
  double s[CE];
#pragma unroll
  for (int v = 0; v < CE; ++v) s[v] = 0.0;
  if (vec) {
    // 16-byte chunks [c0, c1) covering [j0, j1); elements outside are masked
    const int64_t c0 = j0 / CE, c1 = (j1 + CE - 1) / CE;
    for (int64_t cb = c0 + lane; cb < c1; cb += 32 * U) {
      T a[U][CE];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t c = cb + 32 * u;
        if (c < c1) {
          if constexpr (sizeof(T) == 8) {
            const double2 q = __ldg(reinterpret_cast<const double2*>(r) + c);
            a[u][0] = q.x;
            a[u][1 % CE] = q.y;
          } else {
            const float4 q = __ldg(reinterpret_cast<const float4*>(r) + c);
            a[u][0] = q.x;
            a[u][1 % CE] = q.y;
            a[u][2 % CE] = q.z;
            a[u][3 % CE] = q.w;
          }
        } else {
#pragma unroll
          for (int v = 0; v < CE; ++v) a[u][v] = (T)0;
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t c = cb + 32 * u;
        if (c < c1) {
#pragma unroll
          for (int v = 0; v < CE; ++v) {
            const int64_t j = c * CE + v;
            if (j >= j0 && j < j1) s[v] = fma((double)a[u][v], x[j], s[v]);
          }
        }
      }
    }
  } else {
    for (int64_t j = j0 + lane; j < j1; j += 32) s[0] = fma((double)r[j], x[j], s[0]);
  }
  double t = s[0];
#pragma unroll
  for (int v = 1; v < CE; ++v) t += s[v];
  t = warp_sum(t);
  if (lane == 0) out[i] = alpha * t;
}

// part[b][j] = sum_{i in rows of chunk b} M[i*ld + j] * u[i]
template <typename T>
__global__ void k_gemv_cols(const T* __restrict__ M, int64_t rows, int64_t cols, int64_t ld,
                            const double* __restrict__ u, double* __restrict__ part) {
  pdl_wait();
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int nb = gridDim.y;
  const int64_t r0 = rows * blockIdx.y / nb, r1 = rows * (blockIdx.y + 1) / nb;
  if (j >= cols) return;
  double s = 0.0;
  int64_t i = r0;
  for (; i + 8 <= r1; i += 8) {  // eight loads in flight, then the FMAs in row order
    double a[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) a[q] = (double)M[(i + q) * ld + j];
#pragma unroll
    for (int q = 0; q < 8; ++q) s = fma(u[i + q], a[q], s);
  }
  for (; i < r1; ++i) s = fma(u[i], (double)M[i * ld + j], s);
  part[(int64_t)blockIdx.y * cols + j] = s;
}

// Woodbury epilogue: out = (y - (sum_b part[b]) / lam) / nu2   (y = z / lam)
__global__ void k_woodbury_finish(const double* __restrict__ part, int nb, int64_t d,
                                  const double* __restrict__ y, const double* __restrict__ lam,
                                  double nu2, double* __restrict__ out) {
  pdl_wait();
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= d) return;
  double s = 0.0;
  for (int b = 0; b < nb; ++b) s += part[(int64_t)b * d + j];
  out[j] = (y[j] - s / lam[j]) / nu2;
}

__global__ void k_div_vec(const double* __restrict__ z, const double* __restrict__ lam, int64_t d,
                          double* __restrict__ y) {
  pdl_wait();
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < d) y[j] = z[j] / lam[j];
}

int gemv_rows(adask_ctx* ctx, int dtype, const void* M, int64_t rows, int64_t cols, int64_t ld,
              const double* x, double alpha, double* out, int mode, cudaStream_t st) {
  if (rows <= 0) return ADASK_OK;
  const unsigned blocks = (unsigned)cdiv(rows * 32, 256);
  const size_t esz = dtype == ADASK_F64 ? 8 : 4;
  const int vec = ((uintptr_t)M % 16 == 0) && ((size_t)ld * esz) % 16 == 0;
  if (dtype == ADASK_F64)
    ADASK_CUDA(launch_pdl(k_gemv_rows<double>, dim3(blocks), dim3(256), 0, st, (const double*)M, rows, cols, ld, x,
                          alpha, out, mode, vec));
  else
    ADASK_CUDA(launch_pdl(k_gemv_rows<float>, dim3(blocks), dim3(256), 0, st, (const float*)M, rows, cols, ld, x,
                          alpha, out, mode, vec));
  ADASK_LAUNCHED(ctx);
  return ADASK_OK;
}

int woodbury_apply(adask_ctx* ctx, int dtype, const void* SA, int64_t m, int64_t d, int64_t ldsa,
                   const void* Linv, const void* LinvT, int64_t ldl, const double* lam, double nu2,
                   const double* z, double* out, cudaStream_t st) {
  // scratch: y (d), w (m), t (m), u (m), partials (nb * d)
  const int nb = (int)std::min<int64_t>(std::max<int64_t>(1, m / 16), 64);
  const size_t a = 256;
  size_t off_w = align_up((size_t)d * 8, a), off_t = off_w + align_up((size_t)m * 8, a);
  size_t off_u = off_t + align_up((size_t)m * 8, a), off_p = off_u + align_up((size_t)m * 8, a);
  void* wsp = nullptr;
  ADASK_TRY(ctx->ws[WS_GEMV].get(off_p + (size_t)nb * d * 8, st, &wsp));
  char* b = (char*)wsp;
  double *y = (double*)b, *w = (double*)(b + off_w), *t = (double*)(b + off_t);
  double *u = (double*)(b + off_u), *part = (double*)(b + off_p);
  ADASK_CUDA(launch_pdl(k_div_vec, dim3((unsigned)cdiv(d, 256)), dim3(256), 0, st, z, lam, d, y));
  ADASK_LAUNCHED(ctx);
  ADASK_TRY(gemv_rows(ctx, dtype, SA, m, d, ldsa, y, 1.0, w, 0, st));     // w = SA y
  ADASK_TRY(gemv_rows(ctx, dtype, Linv, m, m, ldl, w, 1.0, t, 1, st));    // t = L^-1 w
  ADASK_TRY(gemv_rows(ctx, dtype, LinvT, m, m, ldl, t, 1.0, u, 2, st));   // u = L^-T t
  dim3 g((unsigned)cdiv(d, 256), (unsigned)nb);
  if (dtype == ADASK_F64)
    ADASK_CUDA(launch_pdl(k_gemv_cols<double>, g, dim3(256), 0, st, (const double*)SA, m, d, ldsa, (const double*)u,
                          part));
  else
    ADASK_CUDA(launch_pdl(k_gemv_cols<float>, g, dim3(256), 0, st, (const float*)SA, m, d, ldsa, (const double*)u,
                          part));
  ADASK_LAUNCHED(ctx);
  ADASK_CUDA(launch_pdl(k_woodbury_finish, dim3((unsigned)cdiv(d, 256)), dim3(256), 0, st, (const double*)part, nb,
                        d, (const double*)y, lam, nu2, out));
  ADASK_LAUNCHED(ctx);
  return ADASK_OK;
}

// Triangular solve L y = z (or L^T y = z) for one right-hand side per CTA:
// row-by-row substitution, each row's dot product reduced across the block.
// Not on the solver's hot path (the preconditioner applies explicit
// inverses); it backs the reference's linalg.tri_solve.
template <typename T>
__global__ void k_tri_solve(const T* __restrict__ L, int64_t k, int64_t ldl, int transposed,
                            const double* __restrict__ Z, int64_t ldz, double* __restrict__ Y, int64_t ldy,
                            int* bad) {
  __shared__ double sh[32];
  const double* z = Z + (int64_t)blockIdx.x * ldz;
  double* y = Y + (int64_t)blockIdx.x * ldy;
  for (int64_t s = 0; s < k; ++s) {
    const int64_t i = transposed ? k - 1 - s : s;
    double acc = 0.0;
    if (!transposed) {
      for (int64_t j = threadIdx.x; j < i; j += blockDim.x) acc += (double)L[i * ldl + j] * y[j];
    } else {
      for (int64_t j = i + 1 + threadIdx.x; j < k; j += blockDim.x) acc += (double)L[j * ldl + i] * y[j];
    }
    acc = block_sum(acc, sh);
    if (threadIdx.x == 0) {
      const double dgl = (double)L[i * ldl + i];
      if (dgl == 0.0) atomicExch(bad, 1);
      y[i] = (z[i] - acc) / dgl;
    }
    __syncthreads();
  }
}

}  // namespace adask

using namespace adask;

extern "C" int adask_tri_solve(adask_ctx* ctx, int dtype, const void* L, int64_t k, int64_t ldl, int transposed,
                               const double* Z, int64_t c, int64_t ldz, double* Y, int64_t ldy, void* stream) {
  ADASK_TRY(use_device(ctx));
  if (k < 1 || c < 1 || ldl < k || ldz < k || ldy < k || !L || !Z || !Y)
    return fail(ADASK_E_DIM, "tri_solve: bad shape");
  if (dtype != ADASK_F64 && dtype != ADASK_F32) return fail(ADASK_E_ARG, "bad dtype");
  cudaStream_t st = S(stream);
  void* wsp = nullptr;
  ADASK_TRY(ctx->ws[WS_SMALL].get(256, st, &wsp));
  ADASK_CUDA(cudaMemsetAsync(wsp, 0, sizeof(int), st));
  if (dtype == ADASK_F64)
    k_tri_solve<double><<<(unsigned)c, 256, 0, st>>>((const double*)L, k, ldl, transposed, Z, ldz, Y, ldy, (int*)wsp);
  else
    k_tri_solve<float><<<(unsigned)c, 256, 0, st>>>((const float*)L, k, ldl, transposed, Z, ldz, Y, ldy, (int*)wsp);
  ADASK_LAUNCHED(ctx);
  int bad = 0;
  ADASK_CUDA(cudaMemcpyAsync(&bad, wsp, sizeof(int), cudaMemcpyDeviceToHost, st));
  ADASK_CUDA(cudaStreamSynchronize(st));
  if (bad) return fail(ADASK_E_ARG, "tri_solve: singular triangular factor (zero diagonal)");
  return ADASK_OK;
}
