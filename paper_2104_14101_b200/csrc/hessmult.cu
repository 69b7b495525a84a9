// H X = A^T (A X) + nu^2 Lam X  (- B)       reference: problem.py:89-107
//
// The reference makes two BLAS GEMV passes over A (A @ X, then A.T @ ...).
// Here every row of A is read from HBM exactly once: a CTA streams a tile of R
// rows into registers (128-bit non-allocating loads), forms the R row dots
// y_r = a_r . x with a block reduction, and immediately accumulates
// y_r * a_r into its private partial d-vector.  CTAs own contiguous row
// ranges (static, so the summation order is fixed); a second kernel reduces
// the per-CTA partials in a fixed order and applies the nu^2 Lam X - B
// epilogue.  No floating-point atomics: bitwise reproducible.
//
// Algorithmic bytes per call: n * d * sizeof(T).
#include "common.cuh"
#include "hessmult.cuh"

namespace adask {

template <typename T>
struct Vec16;
template <>
struct Vec16<double> {
  static constexpr int N = 2;
  __device__ static __forceinline__ void load(const double* p, double* v) {
    double2 r;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];"
                 : "=d"(r.x), "=d"(r.y)
                 : "l"(p));
    v[0] = r.x;
    v[1] = r.y;
  }
};
template <>
struct Vec16<float> {
  static constexpr int N = 4;
  __device__ static __forceinline__ void load(const float* p, float* v) {
    float4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(p));
    v[0] = r.x;
    v[1] = r.y;
    v[2] = r.z;
    v[3] = r.w;
  }
};

template <typename T, int VEC>
__device__ __forceinline__ void load_chunk(const T* p, T* v) {
  if constexpr (VEC == 1) {
    v[0] = __ldg(p);
  } else {
    Vec16<T>::load(p, v);
  }
}

// One pass of A^T A x over the row range owned by this CTA.
// Thread t owns column chunks {ch * blockDim + t : ch < NCH}, chunk = VEC
// consecutive columns.  R rows per tile are held in registers between the
// dot and the rank-1 accumulation.
template <typename T, int VEC, int NCH, int R>
__global__ void __launch_bounds__(256) k_hess_fused(const T* __restrict__ A, int64_t n, int64_t d,
                                                    int64_t lda, const double* __restrict__ x,
                                                    double* __restrict__ part) {
  __shared__ double red[2][8][R];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int nw = blockDim.x >> 5;
  const int64_t nchunks = (d + VEC - 1) / VEC;

  double xv[NCH][VEC], acc[NCH][VEC];
  bool act[NCH];
#pragma unroll
  for (int ch = 0; ch < NCH; ++ch) {
    int64_t c = (int64_t)ch * blockDim.x + tid;
    act[ch] = c < nchunks;
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
      int64_t col = c * VEC + v;
      xv[ch][v] = (act[ch] && col < d) ? x[col] : 0.0;
      acc[ch][v] = 0.0;
    }
  }

  // static contiguous row range of this CTA
  const int64_t tiles = (n + R - 1) / R;
  const int64_t t0 = tiles * blockIdx.x / gridDim.x;
  const int64_t t1 = tiles * (blockIdx.x + 1) / gridDim.x;
  int buf = 0;
  for (int64_t tile = t0; tile < t1; ++tile) {
    const int64_t r0 = tile * R;
    T a[R][NCH][VEC];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const bool rok = (r0 + r) < n;
      const T* row = A + (r0 + r) * lda;
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) {
        int64_t c = (int64_t)ch * blockDim.x + tid;
        if (rok && act[ch]) {
          load_chunk<T, VEC>(row + c * VEC, a[r][ch]);
        } else {
#pragma unroll
          for (int v = 0; v < VEC; ++v) a[r][ch][v] = (T)0;
        }
      }
    }
    double dot[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      double s = 0.0;
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
        for (int v = 0; v < VEC; ++v) s = fma((double)a[r][ch][v], xv[ch][v], s);
      dot[r] = warp_sum(s);
    }
    if (lane == 0) {
#pragma unroll
      for (int r = 0; r < R; ++r) red[buf][wid][r] = dot[r];
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < R; ++r) {
      double y = 0.0;
      for (int w = 0; w < nw; ++w) y += red[buf][w][r];
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
        for (int v = 0; v < VEC; ++v) acc[ch][v] = fma(y, (double)a[r][ch][v], acc[ch][v]);
    }
    buf ^= 1;  // double-buffered reduction slots: one barrier per tile
  }
  double* out = part + (int64_t)blockIdx.x * d;
#pragma unroll
  for (int ch = 0; ch < NCH; ++ch) {
    int64_t c = (int64_t)ch * blockDim.x + tid;
    if (!act[ch]) continue;
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
      int64_t col = c * VEC + v;
      if (col < d) out[col] = acc[ch][v];
    }
  }
}

// out[j] = sum_b part[b][j]  (+ nu2 lam[j] x[j] - B[j])   fixed order.
// Block = 32 columns x 8 b-groups.
__global__ void k_hess_finish(const double* __restrict__ part, int nparts, int64_t d,
                              const double* __restrict__ x, double nu2,
                              const double* __restrict__ lam, const double* __restrict__ B,
                              double* __restrict__ out, int epilogue) {
  __shared__ double sh[8][33];
  const int cx = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int64_t j = (int64_t)blockIdx.x * 32 + cx;
  double s = 0.0;
  if (j < d)
    for (int b = g; b < nparts; b += 8) s += part[(int64_t)b * d + j];
  sh[g][cx] = s;
  __syncthreads();
  if (g == 0 && j < d) {
    double t = sh[0][cx];
#pragma unroll
    for (int q = 1; q < 8; ++q) t += sh[q][cx];
    if (epilogue) {
      t += nu2 * (lam[j] * x[j]);
      if (B) t -= B[j];
    }
    out[j] = t;
  }
}

// Two-pass path for rows too wide for the fused register tile:
// y = A x (warp per row), then column-parallel A^T y partials.
template <typename T>
__global__ void k_gemv_rows(const T* __restrict__ A, int64_t n, int64_t d, int64_t lda,
                            const double* __restrict__ x, double* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (row >= n) return;
  const T* a = A + row * lda;
  double s = 0.0;
  for (int64_t j = lane; j < d; j += 32) s = fma((double)a[j], x[j], s);
  s = warp_sum(s);
  if (lane == 0) y[row] = s;
}

template <typename T>
__global__ void k_gemv_cols_part(const T* __restrict__ A, int64_t n, int64_t d, int64_t lda,
                                 const double* __restrict__ y, double* __restrict__ part) {
  const int64_t col = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int nb = gridDim.y;
  const int64_t r0 = n * blockIdx.y / nb, r1 = n * (blockIdx.y + 1) / nb;
  if (col >= d) return;
  double s = 0.0;
  for (int64_t r = r0; r < r1; ++r) s = fma(y[r], (double)A[r * lda + col], s);
  part[(int64_t)blockIdx.y * d + col] = s;
}

template <typename T, int VEC, int NCH, int R>
static int launch_fused(adask_ctx* ctx, const T* A, int64_t n, int64_t d, int64_t lda,
                        const double* x, double* part, int grid, int threads, cudaStream_t st) {
  k_hess_fused<T, VEC, NCH, R><<<grid, threads, 0, st>>>(A, n, d, lda, x, part);
  ADASK_LAUNCHED(ctx);
  return ADASK_OK;
}

// Picks the register-tile shape for (dtype, d, alignment).
template <typename T>
static int hess_partial(adask_ctx* ctx, const T* A, int64_t n, int64_t d, int64_t lda,
                        const double* x, double** part_out, int* nparts_out, cudaStream_t st) {
  constexpr int V16 = 16 / sizeof(T);
  const bool aligned = ((uintptr_t)A % 16 == 0) && ((lda * (int64_t)sizeof(T)) % 16 == 0);
  const int vec = aligned ? V16 : 1;
  const int64_t nchunks = (d + vec - 1) / vec;
  int threads = 256, nch = (int)cdiv(nchunks, 256);
  if (nch <= 1) {
    nch = 1;
    threads = (int)std::max<int64_t>(64, std::min<int64_t>(256, cdiv(nchunks, 32) * 32));
  }
  const bool fused = (aligned && nch <= (sizeof(T) == 8 ? 8 : 4)) || (!aligned && nch <= 16);
  if (!fused) {
    // two-pass fallback
    const int nb = 2 * kNumSMs;
    void* wsp = nullptr;
    size_t bytes = align_up((size_t)n * sizeof(double), 256) + (size_t)nb * d * sizeof(double);
    ADASK_TRY(ctx->ws[WS_HESS].get(bytes, st, &wsp));
    double* y = (double*)wsp;
    double* part = (double*)((char*)wsp + align_up((size_t)n * sizeof(double), 256));
    k_gemv_rows<T><<<(unsigned)cdiv(n * 32, 256), 256, 0, st>>>(A, n, d, lda, x, y);
    ADASK_LAUNCHED(ctx);
    dim3 g2((unsigned)cdiv(d, 256), nb);
    k_gemv_cols_part<T><<<g2, 256, 0, st>>>(A, n, d, lda, y, part);
    ADASK_LAUNCHED(ctx);
    *part_out = part;
    *nparts_out = nb;
    return ADASK_OK;
  }
  // rows per tile: keep ~32 values of A per thread in flight
  const int per_row = nch * vec;
  int R = 32 / per_row;
  R = R >= 16 ? 16 : R >= 8 ? 8 : R >= 4 ? 4 : 2;
  const int64_t tiles = cdiv(n, R);
  const int ctas_per_sm = threads <= 128 ? 4 : 2;
  int grid = (int)std::min<int64_t>(tiles, (int64_t)kNumSMs * ctas_per_sm);
  if (grid < 1) grid = 1;
  void* wsp = nullptr;
  ADASK_TRY(ctx->ws[WS_HESS].get((size_t)grid * d * sizeof(double), st, &wsp));
  double* part = (double*)wsp;
  *part_out = part;
  *nparts_out = grid;
#define L(VV, NN, RR) return launch_fused<T, VV, NN, RR>(ctx, A, n, d, lda, x, part, grid, threads, st)
  if (vec == V16) {
    switch (nch) {
      case 1:
        if (R == 16) L(V16, 1, 16);
        if (R == 8) L(V16, 1, 8);
        L(V16, 1, 4);
      case 2:
        if (R == 8) L(V16, 2, 8);
        L(V16, 2, 4);
      case 3:
      case 4:
        if (R == 4) L(V16, 4, 4);
        L(V16, 4, 2);
      default:
        if constexpr (sizeof(T) == 8) L(V16, 8, 2);
        return fail(ADASK_E_ARG, "hess_mult: unreachable tile shape");
    }
  } else {
    switch (nch) {
      case 1:
        L(1, 1, 16);
      case 2:
        L(1, 2, 16);
      case 3:
      case 4:
        L(1, 4, 8);
      case 5:
      case 6:
      case 7:
      case 8:
        L(1, 8, 4);
      default:
        L(1, 16, 2);
    }
  }
#undef L
}

int hess_mult_impl(adask_ctx* ctx, int dtype, const void* A, int64_t n, int64_t d, int64_t lda,
                   const double* X, int64_t c, int64_t ldx, double nu2, const double* lam,
                   const double* B, int64_t ldb, double* out, int64_t ldo, uint32_t flags,
                   cudaStream_t st) {
  if (n < 0 || d <= 0 || c <= 0 || lda < d || ldx < d || ldo < d || (B && ldb < d))
    return fail(ADASK_E_DIM, "hess_mult: bad shape n=%lld d=%lld c=%lld", (long long)n,
                (long long)d, (long long)c);
  const bool partial = (flags & ADASK_PARTIAL) != 0;
  if (!partial && !lam) return fail(ADASK_E_ARG, "hess_mult: lam required");
  ProfScope prof(ctx, PK_HESS, st, (double)n * d * (dtype == ADASK_F64 ? 8 : 4) * c,
                 4.0 * (double)n * d * c);
  for (int64_t j = 0; j < c; ++j) {
    const double* x = X + j * ldx;
    double* part = nullptr;
    int nparts = 0;
    if (n == 0) {
      // A^T A x = 0
      ADASK_CUDA(cudaMemsetAsync(out + j * ldo, 0, d * sizeof(double), st));
      if (!partial) {
        ADASK_TRY(vec_hess_finish_impl(ctx, out + j * ldo, d, 1, ldo, x, nu2, lam,
                                       B ? B + j * ldb : nullptr, out + j * ldo, st));
      }
      continue;
    }
    if (dtype == ADASK_F64)
      ADASK_TRY(hess_partial<double>(ctx, (const double*)A, n, d, lda, x, &part, &nparts, st));
    else if (dtype == ADASK_F32)
      ADASK_TRY(hess_partial<float>(ctx, (const float*)A, n, d, lda, x, &part, &nparts, st));
    else
      return fail(ADASK_E_ARG, "bad dtype %d", dtype);
    k_hess_finish<<<(unsigned)cdiv(d, 32), 256, 0, st>>>(part, nparts, d, x, nu2, lam,
                                                         B ? B + j * ldb : nullptr,
                                                         out + j * ldo, partial ? 0 : 1);
    ADASK_LAUNCHED(ctx);
  }
  return ADASK_OK;
}

__global__ void k_vec_hess_finish(const double* __restrict__ part, int64_t d, int64_t c, int64_t ld,
                                  const double* __restrict__ X, double nu2,
                                  const double* __restrict__ lam, const double* __restrict__ B,
                                  double* __restrict__ out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= d * c) return;
  int64_t j = i / d, r = i % d;
  double t = part[j * ld + r] + nu2 * (lam[r] * X[j * ld + r]);
  if (B) t -= B[j * ld + r];
  out[j * ld + r] = t;
}

int vec_hess_finish_impl(adask_ctx* ctx, const double* part, int64_t d, int64_t c, int64_t ld,
                         const double* X, double nu2, const double* lam, const double* B,
                         double* out, cudaStream_t st) {
  int64_t tot = d * c;
  if (tot == 0) return ADASK_OK;
  k_vec_hess_finish<<<(unsigned)cdiv(tot, 256), 256, 0, st>>>(part, d, c, ld, X, nu2, lam, B, out);
  ADASK_LAUNCHED(ctx);
  return ADASK_OK;
}

}  // namespace adask

using namespace adask;

extern "C" int adask_hess_mult(adask_ctx* ctx, int dtype, const void* A, int64_t n, int64_t d,
                               int64_t lda, const double* X, int64_t c, int64_t ldx, double nu2,
                               const double* lam, const double* B, int64_t ldb, double* out,
                               int64_t ldo, uint32_t flags, void* stream) {
  ADASK_TRY(use_device(ctx));
  return hess_mult_impl(ctx, dtype, A, n, d, lda, X, c, ldx, nu2, lam, B, ldb, out, ldo, flags,
                        S(stream));
}

extern "C" int adask_vec_hess_finish(adask_ctx* ctx, const double* part, int64_t d, int64_t c,
                                     int64_t ld, const double* X, double nu2, const double* lam,
                                     const double* B, double* out, void* stream) {
  ADASK_TRY(use_device(ctx));
  return vec_hess_finish_impl(ctx, part, d, c, ld, X, nu2, lam, B, out, S(stream));
}
