// SJLT / CountSketch  S*A                       reference: embeddings.py:105-129
//
// Reference: rows = rng.integers(0, m, n) (buckets), signs = rng.integers(0, 2, n)
// drawn from one PCG64 stream (buckets first, then signs), S = csr(m x n), SA =
// S @ A via scipy csr_matvecs, which for every bucket b accumulates
// y_b += sign_i * A[i, :] over the bucket's rows in ascending i.
//
// B200 path (bit-exact in fp64):
//   1. buckets and signs of the local rows from the PCG64 stream by jump-ahead
//      (rng.cu), rejection-exact for any m;
//   2. stable radix sort of (bucket, row) pairs (CUB, integer keys) and bucket
//      offsets from an integer histogram + exclusive scan;
//   3. per-bucket accumulation in ascending row order, one CTA per (bucket,
//      column panel), 128-bit coalesced row loads with 8 rows in flight; no
//      floating-point atomics, so SA is bitwise identical to the reference.
// Algorithmic bytes: (n + m) * d * sizeof(T).
#include <cub/cub.cuh>
#include <cstdlib>

#include "common.cuh"
#include "rng.cuh"
#include "sjlt.cuh"

namespace adask {

__global__ void k_iota_i32(int32_t* v, int64_t n, int32_t s) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = (int32_t)(i / s);
}

__global__ void k_hist(const int32_t* __restrict__ keys, int64_t n, int32_t* __restrict__ cnt) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) atomicAdd(&cnt[keys[i]], 1);  // integer: order-independent
}

template <typename T, int VEC, int UNROLL>
__global__ void __launch_bounds__(128) k_bucket_accumulate(
    const T* __restrict__ A, int64_t d, int64_t lda, const int32_t* __restrict__ order,
    const int32_t* __restrict__ start, const int32_t* __restrict__ sgn, int32_t sgn_stride,
    int64_t m, double scale, int use_scale, T* __restrict__ SA, int64_t ldsa, int accumulate) {
  const int64_t col0 = ((int64_t)blockIdx.y * blockDim.x + threadIdx.x) * VEC;
  if (col0 >= d) return;
  const bool full = col0 + VEC <= d;
  for (int64_t b = blockIdx.x; b < m; b += gridDim.x) {
    const int32_t p0 = start[b], p1 = start[b + 1];
    double acc[VEC];
#pragma unroll
    for (int v = 0; v < VEC; ++v) acc[v] = 0.0;
    // entry indices of the next group are fetched one group ahead, so the row
    // loads of a group do not wait behind their own index loads
    int32_t en[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) en[u] = (p0 + u < p1) ? __ldg(order + p0 + u) : -1;
    for (int32_t p = p0; p < p1; p += UNROLL) {
      int32_t ec[UNROLL];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) ec[u] = en[u];
      T a[UNROLL][VEC];
      int32_t sg[UNROLL];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        const int32_t e = ec[u];  // entry index (row * s + t); -1 past the bucket
        sg[u] = e >= 0 ? __ldg(sgn + e) : 0;
        const int64_t row = e < 0 ? 0 : (sgn_stride == 1 ? e : e / sgn_stride);
        const T* src = A + row * lda + col0;
        if (e < 0) {
#pragma unroll
          for (int v = 0; v < VEC; ++v) a[u][v] = (T)0;
        } else if (full && VEC > 1) {
          if constexpr (VEC == 2 && sizeof(T) == 8) {
            const double2 t = __ldg(reinterpret_cast<const double2*>(src));
            a[u][0] = (T)t.x;
            a[u][VEC - 1] = (T)t.y;
          } else if constexpr (VEC == 4 && sizeof(T) == 4) {
            const float4 t = __ldg(reinterpret_cast<const float4*>(src));
            a[u][0] = (T)t.x;
            a[u][1 % VEC] = (T)t.y;
            a[u][2 % VEC] = (T)t.z;
            a[u][VEC - 1] = (T)t.w;
          } else {
#pragma unroll
            for (int v = 0; v < VEC; ++v) a[u][v] = __ldg(src + v);
          }
        } else {
#pragma unroll
          for (int v = 0; v < VEC; ++v) a[u][v] = (col0 + v < d) ? __ldg(src + v) : (T)0;
        }
      }
      const int32_t pn = p + UNROLL;
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) en[u] = (pn + u < p1) ? __ldg(order + pn + u) : -1;
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        if (ec[u] >= 0) {
#pragma unroll
          for (int v = 0; v < VEC; ++v) {
            double x = (double)a[u][v];
            if (use_scale) {
              // s > 1: y += (sign / sqrt(s)) * x, product then sum (no contraction)
              double coef = sg[u] ? scale : -scale;
              acc[v] = __dadd_rn(acc[v], __dmul_rn(coef, x));
            } else {
              acc[v] = __dadd_rn(acc[v], sg[u] ? x : -x);  // exact +-x
            }
          }
        }
      }
    }
    T* dst = SA + b * ldsa + col0;
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
      if (col0 + v < d) {
        double r = acc[v];
        if (accumulate) r = (double)dst[v] + r;
        dst[v] = (T)r;
      }
    }
  }
}

template <typename T>
static int launch_accumulate(adask_ctx* ctx, const T* A, int64_t d, int64_t lda,
                             const int32_t* order, const int32_t* start, const int32_t* sgn,
                             int32_t s, int64_t m, T* SA, int64_t ldsa, int accumulate,
                             cudaStream_t st) {
  {
    int launched = 0;
    ADASK_TRY(sjlt_accumulate_pipe(ctx, sizeof(T) == 8 ? ADASK_F64 : ADASK_F32, A, d, lda, order, start, sgn, s, m,
                                   SA, ldsa, accumulate, st, &launched));
    if (launched) return ADASK_OK;
  }
  constexpr int VEC = 16 / sizeof(T);
  const bool aligned = ((uintptr_t)A % 16 == 0) && ((lda * (int64_t)sizeof(T)) % 16 == 0);
  const int threads = 128;
  const double scale = 1.0 / sqrt((double)s);
  const int use_scale = s > 1;
  const int64_t narrow_below = getenv("ADASK_SJLT_NARROW") ? atoll(getenv("ADASK_SJLT_NARROW")) : 4 * kNumSMs;
  if (m * cdiv(d, (int64_t)threads * VEC) < narrow_below) {
    // few, long buckets: one thread per column and 16 rows in flight per
    // thread (twice the threads and the same bytes in flight per thread)
    int64_t panels = cdiv(d, (int64_t)threads);
    int64_t gx = std::min<int64_t>(m, std::max<int64_t>(1, (int64_t)kNumSMs * 32 / panels));
    dim3 grid((unsigned)gx, (unsigned)panels);
    k_bucket_accumulate<T, 1, 16><<<grid, threads, 0, st>>>(A, d, lda, order, start, sgn, s, m, scale,
                                                            use_scale, SA, ldsa, accumulate);
  } else if (aligned) {
    int64_t panels = cdiv(d, (int64_t)threads * VEC);
    int64_t gx = std::min<int64_t>(m, std::max<int64_t>(1, (int64_t)kNumSMs * 32 / panels));
    dim3 grid((unsigned)gx, (unsigned)panels);
    k_bucket_accumulate<T, VEC, 8><<<grid, threads, 0, st>>>(A, d, lda, order, start, sgn, s, m,
                                                             scale, use_scale, SA, ldsa, accumulate);
  } else {
    int64_t panels = cdiv(d, (int64_t)threads);
    int64_t gx = std::min<int64_t>(m, std::max<int64_t>(1, (int64_t)kNumSMs * 32 / panels));
    dim3 grid((unsigned)gx, (unsigned)panels);
    k_bucket_accumulate<T, 1, 8><<<grid, threads, 0, st>>>(A, d, lda, order, start, sgn, s, m,
                                                           scale, use_scale, SA, ldsa, accumulate);
  }
  ADASK_LAUNCHED(ctx);
  return ADASK_OK;
}

// Sort `nent` entries by key (stable) and build bucket offsets start[0..m].
// keys/vals live in WS_SORT; returns device pointers to sorted entry order
// and start offsets.
int bucket_sort(adask_ctx* ctx, const int32_t* keys, int64_t nent, int64_t m, int32_t s,
                const int32_t** order_out, const int32_t** start_out, cudaStream_t st) {
  int end_bit = 1;
  while ((1ll << end_bit) < m) ++end_bit;
  size_t temp_sort = 0, temp_scan = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, temp_sort, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                  (const int32_t*)nullptr, (int32_t*)nullptr, (int)nent, 0, end_bit,
                                  st);
  cub::DeviceScan::ExclusiveSum(nullptr, temp_scan, (int32_t*)nullptr, (int32_t*)nullptr,
                                (int)(m + 1), st);
  size_t temp = std::max(temp_sort, temp_scan);
  const size_t a = 256;
  size_t off_vals = 0;
  size_t off_keys_out = off_vals + align_up((size_t)nent * 4, a);
  size_t off_vals_out = off_keys_out + align_up((size_t)nent * 4, a);
  size_t off_cnt = off_vals_out + align_up((size_t)nent * 4, a);
  size_t off_start = off_cnt + align_up((size_t)(m + 1) * 4, a);
  size_t off_temp = off_start + align_up((size_t)(m + 1) * 4, a);
  void* wsp = nullptr;
  ADASK_TRY(ctx->ws[WS_SORT].get(off_temp + temp + a, st, &wsp));
  char* base = (char*)wsp;
  int32_t* vals = (int32_t*)(base + off_vals);
  int32_t* keys_out = (int32_t*)(base + off_keys_out);
  int32_t* vals_out = (int32_t*)(base + off_vals_out);
  int32_t* cnt = (int32_t*)(base + off_cnt);
  int32_t* start = (int32_t*)(base + off_start);
  void* tmp = base + off_temp;
  // values = entry index (row-major rows[j*s + t] -> entry j*s+t)
  k_iota_i32<<<(unsigned)cdiv(nent, 256), 256, 0, st>>>(vals, nent, 1);
  ADASK_LAUNCHED(ctx);
  size_t ts = temp;
  cudaError_t e = cub::DeviceRadixSort::SortPairs(tmp, ts, (const uint32_t*)keys, (uint32_t*)keys_out,
                                                  vals, vals_out, (int)nent, 0, end_bit, st);
  if (e != cudaSuccess) return fail(ADASK_E_CUDA, "radix sort: %s", cudaGetErrorString(e));
  ctx->launches++;
  ADASK_CUDA(cudaMemsetAsync(cnt, 0, (size_t)(m + 1) * 4, st));
  k_hist<<<(unsigned)cdiv(nent, 256), 256, 0, st>>>(keys, nent, cnt);
  ADASK_LAUNCHED(ctx);
  ts = temp;
  e = cub::DeviceScan::ExclusiveSum(tmp, ts, cnt, start, (int)(m + 1), st);
  if (e != cudaSuccess) return fail(ADASK_E_CUDA, "scan: %s", cudaGetErrorString(e));
  ctx->launches++;
  *order_out = vals_out;
  *start_out = start;
  (void)s;
  return ADASK_OK;
}

__global__ void k_rows_to_keys(const int64_t* __restrict__ rows, int64_t n, int32_t* __restrict__ keys) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) keys[i] = (int32_t)rows[i];
}

int sketch_sjlt_impl(adask_ctx* ctx, int dtype, const void* A, int64_t n_local, int64_t d,
                     int64_t lda, int64_t row0, int64_t n_total, int64_t m, int64_t s,
                     const adask_pcg64* g, const int64_t* rows_host, uint64_t sign_first,
                     void* SA, int64_t ldsa, uint32_t flags, cudaStream_t st) {
  if (m < 1) return fail(ADASK_E_SKETCH_TOO_LARGE, "sketch size must be a positive integer, got %lld",
                         (long long)m);
  if (s < 1 || s > m)
    return fail(ADASK_E_SPARSITY, "need 1 <= s <= m = %lld, got s = %lld", (long long)m, (long long)s);
  if (d < 1 || lda < d || ldsa < d || n_local < 0 || row0 < 0 || row0 + n_local > n_total)
    return fail(ADASK_E_DIM, "sketch_sjlt: bad shape");
  if (m > 0x7FFFFFFFll || n_total * s > 0x7FFFFFFFll)
    return fail(ADASK_E_ARG, "sketch_sjlt: sizes beyond int32 indexing");
  if (dtype != ADASK_F64 && dtype != ADASK_F32) return fail(ADASK_E_ARG, "bad dtype");
  const int64_t nent = n_local * s;
  const size_t esz = dtype == ADASK_F64 ? 8 : 4;
  ProfScope prof(ctx, PK_SJLT, st, (double)(n_local + m) * d * esz);
  const int accumulate = (flags & ADASK_ACCUMULATE) ? 1 : 0;
  if (nent == 0) {
    if (!accumulate)
      ADASK_CUDA(cudaMemset2DAsync(SA, (size_t)ldsa * esz, 0, (size_t)d * esz, (size_t)m, st));
    return ADASK_OK;
  }
  // keys (buckets) and signs for the local entries (WS_SRHT slot: WS_RNG backs
  // the rejection list of pcg_integers_impl)
  const size_t a = 256;
  int32_t* keys = nullptr;
  int32_t* sgn = nullptr;
  uint64_t sfirst = sign_first;
  if (s == 1) {
    void* w2 = nullptr;
    ADASK_TRY(ctx->ws[WS_SRHT].get(2 * align_up((size_t)nent * 4, a), st, &w2));
    keys = (int32_t*)w2;
    sgn = (int32_t*)((char*)w2 + align_up((size_t)nent * 4, a));
    uint64_t next = 0;
    ADASK_TRY(pcg_integers_impl(ctx, g, 0, row0, n_local, n_total, (uint32_t)m, keys, &next, st));
    sfirst = next;
  } else {
    if (!rows_host) return fail(ADASK_E_ARG, "sketch_sjlt: s > 1 needs host row picks");
    void* w2 = nullptr;
    for (int64_t i = 0; i < nent; ++i)
      if (rows_host[i] < 0 || rows_host[i] >= m)
        return fail(ADASK_E_ARG, "sketch_sjlt: row pick %lld out of range", (long long)rows_host[i]);
    ADASK_TRY(ctx->ws[WS_SRHT].get(2 * align_up((size_t)nent * 4, a) + align_up((size_t)nent * 8, a),
                                   st, &w2));
    keys = (int32_t*)w2;
    sgn = (int32_t*)((char*)w2 + align_up((size_t)nent * 4, a));
    int64_t* rows_dev = (int64_t*)((char*)w2 + 2 * align_up((size_t)nent * 4, a));
    ADASK_CUDA(cudaMemcpyAsync(rows_dev, rows_host, (size_t)nent * 8, cudaMemcpyHostToDevice, st));
    k_rows_to_keys<<<(unsigned)cdiv(nent, 256), 256, 0, st>>>(rows_dev, nent, keys);
    ADASK_LAUNCHED(ctx);
    ADASK_CUDA(cudaStreamSynchronize(st));  // rows_host may be pageable and caller-owned
  }
  // signs: integers(0, 2, size = n_total * s), local items [row0*s, row0*s + nent)
  ADASK_TRY(pcg_integers_impl(ctx, g, sfirst, row0 * s, nent, n_total * s, 2u, sgn, nullptr, st));
  const int32_t* order = nullptr;
  const int32_t* start = nullptr;
  ADASK_TRY(bucket_sort(ctx, keys, nent, m, (int32_t)s, &order, &start, st));
  if (dtype == ADASK_F64)
    return launch_accumulate<double>(ctx, (const double*)A, d, lda, order, start, sgn, (int32_t)s, m,
                                     (double*)SA, ldsa, accumulate, st);
  return launch_accumulate<float>(ctx, (const float*)A, d, lda, order, start, sgn, (int32_t)s, m,
                                  (float*)SA, ldsa, accumulate, st);
}

}  // namespace adask

using namespace adask;

extern "C" int adask_sketch_sjlt(adask_ctx* ctx, int dtype, const void* A, int64_t n_local, int64_t d,
                                 int64_t lda, int64_t row0, int64_t n_total, int64_t m, int64_t s,
                                 const adask_pcg64* g, const int64_t* rows_host,
                                 uint64_t sign_u32_first, void* SA, int64_t ldsa, uint32_t flags,
                                 void* stream) {
  ADASK_TRY(use_device(ctx));
  return sketch_sjlt_impl(ctx, dtype, A, n_local, d, lda, row0, n_total, m, s, g, rows_host,
                          sign_u32_first, SA, ldsa, flags, S(stream));
}
