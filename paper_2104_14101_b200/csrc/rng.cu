// Device-side randomness: parallel, bit-exact evaluation of numpy's
// Generator.integers(0, m, size=count) stream (PCG64 + Lemire, including
// rejections for non-power-of-two m), and the Philox4x32-10 Gaussian sketch
// entries.
//
// integers(0, m) in the reference: embeddings.py:96 (SRHT signs, m = 2),
// :118 (SJLT buckets), :124 (SJLT signs).  Each item is a 32-bit draw mapped
// by Lemire's multiply-shift; draw j is the low (even j) or high (odd j) half
// of 64-bit output j/2 (numpy next_uint32 buffering).  Item i uses the i-th
// accepted draw, so with the sorted list R of rejected draw positions,
// a_i = first + i + k*, k* = min{k : k == |R| or R[k] - k > first + i}.
#include <algorithm>
#include <vector>

#include "common.cuh"
#include "pcg64.cuh"
#include "rng.cuh"

namespace adask {

static inline bool thr_is_zero(uint32_t m) { return lemire_threshold(m) == 0; }

__global__ void k_pcg_scan_rejects(GenState g, uint64_t first, uint64_t window, uint32_t m,
                                   uint32_t thr, uint64_t* rejects, unsigned long long* nrej,
                                   uint64_t cap) {
  const uint64_t per = 64;
  uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint64_t j0 = first + t * per;
  if (j0 >= first + window) return;
  uint64_t j1 = min(j0 + per, first + window);
  U32Stream s(g, j0);
  for (uint64_t j = j0; j < j1; ++j) {
    uint32_t u = s.next();
    if (lemire_reject(u, m, thr)) {
      unsigned long long pos = atomicAdd(nrej, 1ull);
      if (pos < cap) rejects[pos] = j;
    }
  }
}

template <typename OutT, int PER>
__global__ void k_pcg_integers(GenState g, uint64_t first, int64_t item0, int64_t count, uint32_t m,
                               const uint64_t* __restrict__ R, int64_t nR, OutT* __restrict__ out) {
  int64_t i0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * PER;
  if (i0 >= count) return;
  int64_t i1 = (i0 + PER < count ? i0 + PER : count);
  // k* by binary search over the monotone predicate R[k] - k > first + item
  const uint64_t item = (uint64_t)(item0 + i0);
  int64_t lo = 0, hi = nR;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if ((int64_t)(R[mid] - (uint64_t)mid) > (int64_t)(first + item)) hi = mid;
    else lo = mid + 1;
  }
  int64_t k = lo;
  uint64_t j = first + item + (uint64_t)k;
  U32Stream s(g, j);
  for (int64_t i = i0; i < i1;) {
    uint32_t u = s.next();
    if (k < nR && R[k] == j) {
      ++k;
      ++j;
      continue;
    }
    out[i] = (OutT)lemire_value(u, m);
    ++i;
    ++j;
  }
}

// Fast path without rejections (power-of-two m): contiguous draws.
template <typename OutT, int PER>
__global__ void k_pcg_integers_norej(GenState g, uint64_t first, int64_t count, uint32_t m,
                                     OutT* __restrict__ out) {
  int64_t i0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * PER;
  if (i0 >= count) return;
  int64_t i1 = (i0 + PER < count ? i0 + PER : count);
  U32Stream s(g, first + (uint64_t)i0);
  for (int64_t i = i0; i < i1; ++i) out[i] = (OutT)lemire_value(s.next(), m);
}

// Sign bits of integers(0, 2, size=count) packed 32 per word (bit e of word w
// = draw first + 32w + e; 1 -> +1).  m = 2 never rejects (Lemire threshold 0).
__global__ void k_pcg_sign_bits(GenState g, uint64_t first, int64_t count, uint32_t* __restrict__ words) {
  const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t i0 = w * 32;
  if (i0 >= count) return;
  const int64_t n = count - i0 < 32 ? count - i0 : 32;
  U32Stream s(g, first + (uint64_t)i0);
  uint32_t bits = 0;
  for (int e = 0; e < n; ++e) bits |= (lemire_value(s.next(), 2u) & 1u) << e;
  words[w] = bits;
}

int pcg_sign_bits_impl(adask_ctx* ctx, const adask_pcg64* g, uint64_t first, int64_t count,
                       uint32_t* words, cudaStream_t st) {
  if (count <= 0) return ADASK_OK;
  const int64_t nw = cdiv(count, 32);
  k_pcg_sign_bits<<<(unsigned)cdiv(nw, 256), 256, 0, st>>>(GenState::from(*g), first, count, words);
  ADASK_LAUNCHED(ctx);
  return ADASK_OK;
}

int pcg_integers_impl(adask_ctx* ctx, const adask_pcg64* g, uint64_t first, int64_t item0,
                      int64_t count, int64_t total_items, uint32_t m, int32_t* out, uint64_t* next,
                      cudaStream_t st) {
  if (!g || m == 0 || count < 0 || item0 < 0 || total_items < item0 + count)
    return fail(ADASK_E_ARG, "pcg64_integers: bad arguments");
  if (total_items == 0) {
    if (next) *next = first;
    return ADASK_OK;
  }
  GenState gs = GenState::from(*g);
  if (m == 1) {  // rng == 0: numpy returns `off` without consuming draws
    ADASK_CUDA(cudaMemsetAsync(out, 0, (size_t)count * sizeof(int32_t), st));
    if (next) *next = first;
    return ADASK_OK;
  }
  if (count == 0 && thr_is_zero(m)) {
    if (next) *next = first + (uint64_t)total_items;
    return ADASK_OK;
  }
  constexpr int PER = 32;
  const int threads = 256;
  const uint32_t thr = lemire_threshold(m);
  if (thr == 0) {
    int64_t blocks = cdiv(cdiv(count, PER), threads);
    k_pcg_integers_norej<int32_t, PER><<<(unsigned)blocks, threads, 0, st>>>(
        gs, first + (uint64_t)item0, count, m, out);
    ADASK_LAUNCHED(ctx);
    if (next) *next = first + (uint64_t)total_items;
    return ADASK_OK;
  }
  // Rejection-aware path.  Expected rejections: total_items * thr / 2^32.
  uint64_t slack = 1024 + (uint64_t)((double)total_items * ((double)thr / 4294967296.0) * 2.0);
  for (int attempt = 0; attempt < 8; ++attempt) {
    uint64_t window = (uint64_t)total_items + slack;
    uint64_t cap = slack;
    void* wsp = nullptr;
    size_t bytes = sizeof(unsigned long long) + cap * sizeof(uint64_t) + 64;
    ADASK_TRY(ctx->ws[WS_RNG].get(bytes, st, &wsp));
    unsigned long long* d_n = reinterpret_cast<unsigned long long*>(wsp);
    uint64_t* d_R = reinterpret_cast<uint64_t*>(reinterpret_cast<char*>(wsp) + 64);
    ADASK_CUDA(cudaMemsetAsync(d_n, 0, sizeof(unsigned long long), st));
    uint64_t nthreads = (window + 63) / 64;
    k_pcg_scan_rejects<<<(unsigned)cdiv((int64_t)nthreads, threads), threads, 0, st>>>(
        gs, first, window, m, thr, d_R, d_n, cap);
    ADASK_LAUNCHED(ctx);
    unsigned long long nrej = 0;
    ADASK_CUDA(cudaMemcpyAsync(&nrej, d_n, sizeof(nrej), cudaMemcpyDeviceToHost, st));
    ADASK_CUDA(cudaStreamSynchronize(st));
    if (nrej > cap || window - nrej < (uint64_t)total_items) {
      slack = 2 * slack + 2 * nrej;
      continue;
    }
    std::vector<uint64_t> R((size_t)nrej);
    if (nrej) {
      ADASK_CUDA(cudaMemcpyAsync(R.data(), d_R, nrej * sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
      ADASK_CUDA(cudaStreamSynchronize(st));
      std::sort(R.begin(), R.end());
      ADASK_CUDA(cudaMemcpyAsync(d_R, R.data(), nrej * sizeof(uint64_t), cudaMemcpyHostToDevice, st));
    }
    if (count > 0) {
      int64_t blocks = cdiv(cdiv(count, PER), threads);
      k_pcg_integers<int32_t, PER><<<(unsigned)blocks, threads, 0, st>>>(gs, first, item0, count, m,
                                                                           d_R, (int64_t)nrej, out);
      ADASK_LAUNCHED(ctx);
    }
    if (next) {
      // last consumed index a_{total-1} = first + total - 1 + k*
      uint64_t target = first + (uint64_t)total_items - 1;
      int64_t k = 0;
      while (k < (int64_t)nrej && (int64_t)(R[(size_t)k] - (uint64_t)k) <= (int64_t)target) ++k;
      *next = target + (uint64_t)k + 1;
    }
    if (nrej) ADASK_CUDA(cudaStreamSynchronize(st));  // R (host vector) must outlive the copy
    return ADASK_OK;
  }
  return fail(ADASK_E_ARG, "pcg64_integers: rejection window did not converge");
}

// ---------------------------------------------------------------- Philox normals
template <typename T>
__global__ void k_philox_gaussian(int64_t krow0, int64_t mk, int64_t col0, int64_t ncols, uint32_t k0, uint32_t k1,
                                  double sc, T* __restrict__ out, int64_t ldo) {
  // one thread per (column, group of four global sketch rows); grid.y tiles
  // the groups covering rows [krow0, krow0 + mk)
  const int64_t g = (krow0 >> 2) + blockIdx.y;
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncols) return;
  double z[4];
  gaussian_quad_f64((uint64_t)(col0 + c), (uint32_t)g, k0, k1, z);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int64_t k = 4 * g + q;
    if (k >= krow0 && k < krow0 + mk) out[(k - krow0) * ldo + c] = (T)(z[q] / sc);
  }
}

// Rows [krow0, krow0 + mk) of the m_total-row Gaussian S (scale 1/sqrt(m_total)).
int philox_gaussian_rows(adask_ctx* ctx, int dtype, int64_t krow0, int64_t mk, int64_t m_total, int64_t col0,
                         int64_t ncols, uint64_t key, void* out, int64_t ldo, cudaStream_t st) {
  if (mk <= 0 || ncols <= 0) return ADASK_OK;
  const int64_t groups = ((krow0 + mk - 1) >> 2) - (krow0 >> 2) + 1;
  if (groups > 65535) return fail(ADASK_E_ARG, "philox_gaussian: more than 262140 rows per call");
  dim3 grid((unsigned)cdiv(ncols, 256), (unsigned)groups);
  const double sc = sqrt((double)m_total);
  const uint32_t k0 = (uint32_t)key, k1 = (uint32_t)(key >> 32);
  if (dtype == ADASK_F64)
    k_philox_gaussian<double><<<grid, 256, 0, st>>>(krow0, mk, col0, ncols, k0, k1, sc, (double*)out, ldo);
  else
    k_philox_gaussian<float><<<grid, 256, 0, st>>>(krow0, mk, col0, ncols, k0, k1, sc, (float*)out, ldo);
  ADASK_LAUNCHED(ctx);
  return ADASK_OK;
}

// The same entries stored transposed: out[(i - col0) * ldo + (k - krow0)] =
// S[k, i] (rows = columns of S = rows of A), the K-outer operand of the DMMA
// sketch GEMM.  Consecutive threads take consecutive row groups of one column.
template <typename T>
__global__ void k_philox_gaussian_t(int64_t krow0, int64_t mk, int64_t col0, int64_t ncols, int64_t groups,
                                    uint32_t k0, uint32_t k1, double sc, T* __restrict__ out, int64_t ldo) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= ncols * groups) return;
  const int64_t c = t / groups;
  const int64_t g = (krow0 >> 2) + (t - c * groups);
  double z[4];
  gaussian_quad_f64((uint64_t)(col0 + c), (uint32_t)g, k0, k1, z);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int64_t k = 4 * g + q;
    if (k >= krow0 && k < krow0 + mk) out[c * ldo + (k - krow0)] = (T)(z[q] / sc);
  }
}

int philox_gaussian_rows_t(adask_ctx* ctx, int dtype, int64_t krow0, int64_t mk, int64_t m_total, int64_t col0,
                           int64_t ncols, uint64_t key, void* out, int64_t ldo, cudaStream_t st) {
  if (mk <= 0 || ncols <= 0) return ADASK_OK;
  const int64_t groups = ((krow0 + mk - 1) >> 2) - (krow0 >> 2) + 1;
  const double sc = sqrt((double)m_total);
  const uint32_t k0 = (uint32_t)key, k1 = (uint32_t)(key >> 32);
  const unsigned grid = (unsigned)cdiv(ncols * groups, 256);
  if (dtype == ADASK_F64)
    k_philox_gaussian_t<double><<<grid, 256, 0, st>>>(krow0, mk, col0, ncols, groups, k0, k1, sc, (double*)out, ldo);
  else
    k_philox_gaussian_t<float><<<grid, 256, 0, st>>>(krow0, mk, col0, ncols, groups, k0, k1, sc, (float*)out, ldo);
  ADASK_LAUNCHED(ctx);
  return ADASK_OK;
}

}  // namespace adask

using namespace adask;

extern "C" int adask_pcg64_integers(adask_ctx* ctx, const adask_pcg64* g, uint64_t u32_first,
                                    int64_t count, uint32_t m, int32_t* out,
                                    uint64_t* u32_next_host, void* stream) {
  ADASK_TRY(use_device(ctx));
  return pcg_integers_impl(ctx, g, u32_first, 0, count, count, m, out, u32_next_host, S(stream));
}

extern "C" int adask_philox_gaussian(adask_ctx* ctx, int dtype, int64_t m, int64_t col0,
                                     int64_t ncols, uint64_t key, void* out, int64_t ldo,
                                     void* stream) {
  ADASK_TRY(use_device(ctx));
  if (m <= 0 || ncols < 0 || col0 < 0 || ldo < ncols || !out)
    return fail(ADASK_E_ARG, "philox_gaussian: bad arguments");
  if (ncols == 0) return ADASK_OK;
  return philox_gaussian_rows(ctx, dtype, 0, m, m, col0, ncols, key, out, ldo, S(stream));
}

// Host evaluation of the Gaussian entry definition (for CPU-side pinning of
// the oracle restatement; the device kernels use the same function).
extern "C" int adask_philox_gaussian_host(int64_t m, int64_t col0, int64_t ncols, uint64_t key,
                                          double* out, int64_t ldo) {
  if (m <= 0 || ncols < 0 || col0 < 0 || ldo < ncols || (ncols > 0 && !out))
    return fail(ADASK_E_ARG, "philox_gaussian_host: bad arguments");
  const double sc = sqrt((double)m);
  for (int64_t g = 0; 4 * g < m; ++g)
    for (int64_t i = col0; i < col0 + ncols; ++i) {
      double z[4];
      gaussian_quad_f64((uint64_t)i, (uint32_t)g, (uint32_t)key, (uint32_t)(key >> 32), z);
      for (int q = 0; q < 4 && 4 * g + q < m; ++q) out[(4 * g + q) * ldo + (i - col0)] = z[q] / sc;
    }
  return ADASK_OK;
}
