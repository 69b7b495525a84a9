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
#include "tma.cuh"

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

// TMA-fed variant (the B200 path): one CTA per SM, a producer warp streams
// R-row stages of A into a STAGES-deep SMEM ring with cp.async.bulk
// (mbarrier completion, L2 evict-first), eight consumer warps read their
// 16-byte column chunks from SMEM, release the stage, reduce the R row dots
// across the CTA (one named barrier per stage) and accumulate y_r a_r in
// registers.  Bytes in flight no longer depend on occupancy or registers.
template <typename T, int NCH, int R, int STAGES, int NX>
__global__ void __launch_bounds__(288, 1) k_hess_tma(const T* __restrict__ A, int64_t n, int64_t d,
                                                     int64_t lda, const double* __restrict__ x0,
                                                     const double* __restrict__ x1, double* __restrict__ part0,
                                                     double* __restrict__ part1) {
  // NX = 2: the same pass over A serves two right-hand sides (the PCG
  // proposal direction and the current iterate); every column's arithmetic
  // is the NX = 1 sequence, so each result is bitwise the single-column one
  constexpr int V = 16 / sizeof(T);
  constexpr int NW = 8;  // consumer warps
  extern __shared__ __align__(128) unsigned char hsm[];
  const int64_t stage_elems = (int64_t)R * d;
  T* ring = reinterpret_cast<T*>(hsm);
  uint64_t* full = reinterpret_cast<uint64_t*>(hsm + align_up_dev(STAGES * stage_elems * sizeof(T), 128));
  uint64_t* empty = full + STAGES;
  double* red = reinterpret_cast<double*>(empty + STAGES);  // [NX][2][NW][R], then ybuf [NX][2][R]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t row_begin = n * blockIdx.x / gridDim.x, row_end = n * (blockIdx.x + 1) / gridDim.x;
  const int64_t ntiles = (row_end - row_begin + R - 1) / R;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW);
    }
    fence_barrier_init();
  }
  // A^T A 0 = 0 exactly: an all-zero right-hand side (the solvers' usual
  // x0 = 0 at the first restart) writes zero partials without streaming A
  bool nz = false;
  for (int64_t j = tid; j < d; j += blockDim.x) nz |= (x0[j] != 0.0) || (NX == 2 && x1[j] != 0.0);
  if (!__syncthreads_or(nz)) {
    for (int q = 0; q < NX; ++q) {
      double* out = (q == 0 ? part0 : part1) + (int64_t)blockIdx.x * d;
      for (int64_t j = tid; j < d; j += blockDim.x) out[j] = 0.0;
    }
    return;
  }
  if (warp == NW) {
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      const uint32_t row_bytes = (uint32_t)(d * sizeof(T));
      for (int64_t t = 0; t < ntiles; ++t) {
        const int s = (int)(t % STAGES);
        const uint32_t ph = (uint32_t)((t / STAGES) & 1);
        if (t >= STAGES) mbar_wait(&empty[s], ph ^ 1);
        const int64_t r0 = row_begin + t * R;
        const int rows = (int)min((int64_t)R, row_end - r0);
        mbar_arrive_expect_tx(&full[s], rows * row_bytes);
        T* dst = ring + s * stage_elems;
        if (lda == d) {
          bulk_g2s_evict_first(dst, A + r0 * lda, rows * row_bytes, &full[s], pol);
        } else {
          for (int r = 0; r < rows; ++r)
            bulk_g2s_evict_first(dst + r * d, A + (r0 + r) * lda, row_bytes, &full[s], pol);
        }
      }
    }
    return;
  }
  const int64_t nchunks = d / V;
  double xv[NX][NCH][V], acc[NX][NCH][V];
  bool act[NCH];
#pragma unroll
  for (int ch = 0; ch < NCH; ++ch) {
    const int64_t c = (int64_t)ch * (NW * 32) + tid;
    act[ch] = c < nchunks;
#pragma unroll
    for (int v = 0; v < V; ++v) {
#pragma unroll
      for (int q = 0; q < NX; ++q) {
        const double* xq = q == 0 ? x0 : x1;
        xv[q][ch][v] = act[ch] ? xq[c * V + v] : 0.0;
        acc[q][ch][v] = 0.0;
      }
    }
  }
  int buf = 0;
  for (int64_t t = 0; t < ntiles; ++t) {
    const int s = (int)(t % STAGES);
    const uint32_t ph = (uint32_t)((t / STAGES) & 1);
    const int rows = (int)min((int64_t)R, row_end - (row_begin + t * R));
    mbar_wait(&full[s], ph);
    const T* src = ring + s * stage_elems;
    T a[R][NCH][V];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) {
        const int64_t c = (int64_t)ch * (NW * 32) + tid;
        if (r < rows && act[ch]) {
          if constexpr (sizeof(T) == 8) {
            const double2 qv = *reinterpret_cast<const double2*>(src + r * d + c * V);
            a[r][ch][0] = qv.x;
            a[r][ch][1] = qv.y;
          } else {
            const float4 qv = *reinterpret_cast<const float4*>(src + r * d + c * V);
            a[r][ch][0] = qv.x;
            a[r][ch][1] = qv.y;
            a[r][ch][2] = qv.z;
            a[r][ch][3] = qv.w;
          }
        } else {
#pragma unroll
          for (int v = 0; v < V; ++v) a[r][ch][v] = (T)0;
        }
      }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);  // stage consumed by this warp
#pragma unroll
    for (int q = 0; q < NX; ++q) {
      double dot[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if constexpr (sizeof(T) == 8) {
          double sacc = 0.0;
#pragma unroll
          for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
            for (int v = 0; v < V; ++v) sacc = fma((double)a[r][ch][v], xv[q][ch][v], sacc);
          dot[r] = sacc;
        } else {
          // fp32 data: short per-thread partial in fp32, reduced in fp64
          float sacc = 0.0f;
#pragma unroll
          for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
            for (int v = 0; v < V; ++v) sacc = fmaf((float)a[r][ch][v], (float)xv[q][ch][v], sacc);
          dot[r] = (double)sacc;
        }
      }
      const double tot = warp_multi_sum<R>(dot);
      if ((lane & (32 / R - 1)) == 0) red[((q * 2 + buf) * NW + warp) * R + warp_multi_row<R>(lane)] = tot;
    }
    named_bar_sync(1, NW * 32);
    double* ybuf = red + NX * 2 * NW * R;  // [NX][2][R]
    if (tid < NX * R) {
      const int q = tid / R, r = tid - q * R;
      double y = 0.0;
#pragma unroll
      for (int w = 0; w < NW; ++w) y += red[((q * 2 + buf) * NW + w) * R + r];
      ybuf[(q * 2 + buf) * R + r] = y;
    }
    named_bar_sync(1, NW * 32);
#pragma unroll
    for (int q = 0; q < NX; ++q) {
      if constexpr (sizeof(T) == 8) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const double y = ybuf[(q * 2 + buf) * R + r];
#pragma unroll
          for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
            for (int v = 0; v < V; ++v) acc[q][ch][v] = fma(y, (double)a[r][ch][v], acc[q][ch][v]);
        }
      } else {
        // the R-row rank update in fp32, folded into the fp64 accumulator once per stage
        float stv[NCH][V];
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
          for (int v = 0; v < V; ++v) stv[ch][v] = 0.0f;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const float y = (float)ybuf[(q * 2 + buf) * R + r];
#pragma unroll
          for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
            for (int v = 0; v < V; ++v) stv[ch][v] = fmaf(y, (float)a[r][ch][v], stv[ch][v]);
        }
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
          for (int v = 0; v < V; ++v) acc[q][ch][v] += (double)stv[ch][v];
      }
    }
    buf ^= 1;
  }
#pragma unroll
  for (int q = 0; q < NX; ++q) {
    double* out = (q == 0 ? part0 : part1) + (int64_t)blockIdx.x * d;
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) {
      if (!act[ch]) continue;
      const int64_t c = (int64_t)ch * (NW * 32) + tid;
#pragma unroll
      for (int v = 0; v < V; ++v) out[c * V + v] = acc[q][ch][v];
    }
  }
}

template <typename T, int NCH, int R, int STAGES, int NX = 1>
static int launch_tma(adask_ctx* ctx, const T* A, int64_t n, int64_t d, int64_t lda, const double* x,
                      double* part, int grid, cudaStream_t st, const double* x1 = nullptr,
                      double* part1 = nullptr) {
  const size_t ring = align_up((size_t)STAGES * R * d * sizeof(T), 128);
  const size_t smem = ring + 2 * STAGES * sizeof(uint64_t) + NX * (2 * 8 * R + 2 * R) * sizeof(double);
  auto kern = k_hess_tma<T, NCH, R, STAGES, NX>;
  ADASK_TRY(ensure_smem_attr((const void*)kern, (int)smem));
  kern<<<grid, 288, smem, st>>>(A, n, d, lda, x, x1, part, part1);
  ADASK_LAUNCHED(ctx);
  return ADASK_OK;
}

// TMA path eligibility and dispatch: rows of 16-byte multiples, 16-byte
// aligned base and pitch, d <= 256 * 8 chunks.  Stage = R rows ~ 32 KB.
template <typename T>
static int hess_partial_tma(adask_ctx* ctx, const T* A, int64_t n, int64_t d, int64_t lda,
                            const double* x, double** part_out, int* nparts_out, cudaStream_t st,
                            bool* used, const double* x1 = nullptr, double** part1_out = nullptr) {
  constexpr int V = 16 / sizeof(T);
  *used = false;
  if ((uintptr_t)A % 16 || (d % V) || (lda * (int64_t)sizeof(T)) % 16) return ADASK_OK;
  const int64_t nchunks = d / V;
  int nch = (int)cdiv(nchunks, 256);
  if (nch > 8) return ADASK_OK;
  nch = nch <= 1 ? 1 : nch <= 2 ? 2 : nch <= 4 ? 4 : 8;
  const bool pair = x1 != nullptr;
  if (pair && nch > 4) return ADASK_OK;  // register budget of the two-column tile
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(kNumSMs, cdiv(n, 16)));
  void* wsp = nullptr;
  ADASK_TRY(ctx->ws[WS_HESS].get((size_t)(pair ? 2 : 1) * grid * d * sizeof(double), st, &wsp));
  double* part = (double*)wsp;
  double* part1 = pair ? part + (size_t)grid * d : nullptr;
  *part_out = part;
  if (pair) *part1_out = part1;
  *nparts_out = grid;
  *used = true;
  const int64_t row_bytes = d * (int64_t)sizeof(T);
  if (pair) {
    switch (nch) {
      case 1:
        if (row_bytes <= 2048) return launch_tma<T, 1, 16, 6, 2>(ctx, A, n, d, lda, x, part, grid, st, x1, part1);
        // 16-row stages halve the per-row reduction/barrier overhead of the two
        // columns (2^24 x 1024 fp32: 1.29x -> 1.09x of a single-column pass)
        return launch_tma<T, 1, 16, 3, 2>(ctx, A, n, d, lda, x, part, grid, st, x1, part1);
      case 2:
        return launch_tma<T, 2, 4, 6, 2>(ctx, A, n, d, lda, x, part, grid, st, x1, part1);
      default:
        return launch_tma<T, 4, 2, 6, 2>(ctx, A, n, d, lda, x, part, grid, st, x1, part1);
    }
  }
  switch (nch) {
    case 1:
      if (row_bytes <= 2048) return launch_tma<T, 1, 16, 6>(ctx, A, n, d, lda, x, part, grid, st);
      return launch_tma<T, 1, 8, 6>(ctx, A, n, d, lda, x, part, grid, st);
    case 2:
      return launch_tma<T, 2, 4, 6>(ctx, A, n, d, lda, x, part, grid, st);
    case 4:
      return launch_tma<T, 4, 2, 6>(ctx, A, n, d, lda, x, part, grid, st);
    default:
      return launch_tma<T, 8, 1, 6>(ctx, A, n, d, lda, x, part, grid, st);
  }
}

// out[j] = sum_b part[b][j]  (+ nu2 lam[j] x[j] - B[j])   fixed order.
// Block = 32 columns x 8 b-groups.
__global__ void __launch_bounds__(1024) k_hess_finish(const double* __restrict__ part, int nparts, int64_t d,
                                                      const double* __restrict__ x, double nu2,
                                                      const double* __restrict__ lam,
                                                      const double* __restrict__ B, double* __restrict__ out,
                                                      int epilogue) {
  pdl_wait();
  // 32 columns x 32 partial groups; each thread sums its parts with four
  // independent accumulators (all loads in flight at once), then group 0
  // combines the 32 group sums -- a fixed order, so the result is deterministic
  __shared__ double sh[32][33];
  const int cx = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int64_t j = (int64_t)blockIdx.x * 32 + cx;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  if (j < d) {
    int b = g;
    for (; b + 96 < nparts; b += 128) {
      s0 += part[(int64_t)b * d + j];
      s1 += part[(int64_t)(b + 32) * d + j];
      s2 += part[(int64_t)(b + 64) * d + j];
      s3 += part[(int64_t)(b + 96) * d + j];
    }
    for (; b < nparts; b += 32) s0 += part[(int64_t)b * d + j];
  }
  sh[g][cx] = (s0 + s1) + (s2 + s3);
  __syncthreads();
  if (g == 0 && j < d) {
    double t = sh[0][cx];
#pragma unroll
    for (int q = 1; q < 32; ++q) t += sh[q][cx];
    if (epilogue) {
      t += nu2 * (lam[j] * x[j]);
      if (B) t -= B[j];
    }
    out[j] = t;
  }
}

// Both columns of a pair pass in one launch (blockIdx.y = column).
__global__ void __launch_bounds__(1024) k_hess_finish_pair(const double* __restrict__ part0,
                                                           const double* __restrict__ part1, int nparts, int64_t d,
                                                           const double* __restrict__ x0,
                                                           const double* __restrict__ x1, double nu2,
                                                           const double* __restrict__ lam,
                                                           const double* __restrict__ B0,
                                                           const double* __restrict__ B1, double* __restrict__ out0,
                                                           double* __restrict__ out1, int epilogue) {
  pdl_wait();
  const bool q = blockIdx.y != 0;
  const double* part = q ? part1 : part0;
  const double* x = q ? x1 : x0;
  const double* B = q ? B1 : B0;
  double* out = q ? out1 : out0;
  __shared__ double sh[32][33];
  const int cx = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int64_t j = (int64_t)blockIdx.x * 32 + cx;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  if (j < d) {
    int b = g;
    for (; b + 96 < nparts; b += 128) {
      s0 += part[(int64_t)b * d + j];
      s1 += part[(int64_t)(b + 32) * d + j];
      s2 += part[(int64_t)(b + 64) * d + j];
      s3 += part[(int64_t)(b + 96) * d + j];
    }
    for (; b < nparts; b += 32) s0 += part[(int64_t)b * d + j];
  }
  sh[g][cx] = (s0 + s1) + (s2 + s3);
  __syncthreads();
  if (g == 0 && j < d) {
    double t = sh[0][cx];
#pragma unroll
    for (int r = 1; r < 32; ++r) t += sh[r][cx];
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
    bool used = false;
    const bool tma_ok = getenv("ADASK_NO_TMA") == nullptr;
    if (dtype == ADASK_F64) {
      if (tma_ok)
        ADASK_TRY(hess_partial_tma<double>(ctx, (const double*)A, n, d, lda, x, &part, &nparts, st, &used));
      if (!used) ADASK_TRY(hess_partial<double>(ctx, (const double*)A, n, d, lda, x, &part, &nparts, st));
    } else if (dtype == ADASK_F32) {
      if (tma_ok)
        ADASK_TRY(hess_partial_tma<float>(ctx, (const float*)A, n, d, lda, x, &part, &nparts, st, &used));
      if (!used) ADASK_TRY(hess_partial<float>(ctx, (const float*)A, n, d, lda, x, &part, &nparts, st));
    } else {
      return fail(ADASK_E_ARG, "bad dtype %d", dtype);
    }
    ADASK_CUDA(launch_pdl(k_hess_finish, dim3((unsigned)cdiv(d, 32)), dim3(1024), 0, st, (const double*)part, nparts,
                          d, x, nu2, lam, B ? B + j * ldb : (const double*)nullptr, out + j * ldo,
                          partial ? 0 : 1));
    ADASK_LAUNCHED(ctx);
  }
  return ADASK_OK;
}

// H [x0, x1] in one pass over A (c = 1 problems): out0 = H x0 (- B0), out1 =
// H x1 (- B1); each column bitwise equal to hess_mult_impl's.  *fused = 0 when
// the shape is not eligible (the caller then makes two single-column calls).
int hess_mult_pair_impl(adask_ctx* ctx, int dtype, const void* A, int64_t n, int64_t d, int64_t lda,
                        const double* x0, const double* B0, double* out0, const double* x1, const double* B1,
                        double* out1, double nu2, const double* lam, cudaStream_t st, int* fused, int partial) {
  *fused = 0;
  if (n <= 0 || getenv("ADASK_NO_TMA") || getenv("ADASK_NO_PAIR")) return ADASK_OK;
  ProfScope prof(ctx, PK_HESS, st, (double)n * d * (dtype == ADASK_F64 ? 8 : 4), 8.0 * (double)n * d);
  double *part0 = nullptr, *part1 = nullptr;
  int nparts = 0;
  bool used = false;
  if (dtype == ADASK_F64)
    ADASK_TRY(hess_partial_tma<double>(ctx, (const double*)A, n, d, lda, x0, &part0, &nparts, st, &used, x1, &part1));
  else
    ADASK_TRY(hess_partial_tma<float>(ctx, (const float*)A, n, d, lda, x0, &part0, &nparts, st, &used, x1, &part1));
  if (!used) return ADASK_OK;
  ADASK_CUDA(launch_pdl(k_hess_finish_pair, dim3((unsigned)cdiv(d, 32), 2), dim3(1024), 0, st, (const double*)part0,
                        (const double*)part1, nparts, d, x0, x1, nu2, lam, B0, B1, out0, out1, partial ? 0 : 1));
  ADASK_LAUNCHED(ctx);
  *fused = 1;
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

extern "C" int adask_hess_mult_pair(adask_ctx* ctx, int dtype, const void* A, int64_t n, int64_t d, int64_t lda,
                                    const double* x0, const double* x1, double nu2, const double* lam,
                                    double* out0, double* out1, void* stream) {
  ADASK_TRY(adask::use_device(ctx));
  if (n < 0 || d < 1 || lda < d || !x0 || !x1 || !out0 || !out1 || !lam)
    return adask::fail(ADASK_E_DIM, "hess_mult_pair: bad arguments");
  if (dtype != ADASK_F64 && dtype != ADASK_F32) return adask::fail(ADASK_E_ARG, "bad dtype");
  cudaStream_t st = adask::S(stream);
  int fused = 0;
  ADASK_TRY(adask::hess_mult_pair_impl(ctx, dtype, A, n, d, lda, x0, nullptr, out0, x1, nullptr, out1, nu2, lam, st,
                                       &fused));
  if (fused) return ADASK_OK;
  ADASK_TRY(adask::hess_mult_impl(ctx, dtype, A, n, d, lda, x0, 1, d, nu2, lam, nullptr, d, out0, d, 0, st));
  return adask::hess_mult_impl(ctx, dtype, A, n, d, lda, x1, 1, d, nu2, lam, nullptr, d, out1, d, 0, st);
}
