// Gaussian sketch SA = S A, S = N(0, 1/m)          reference: embeddings.py:66-73
//
// S[k, i] = Philox4x32-10 / Box-Muller normal (rng.cuh) divided by sqrt(m),
// keyed by the sketch seed and indexed by (sketch row k, GLOBAL row i of A),
// so a row-sharded A gives per-shard partial sketches that sum to the full
// one.  fp64: S^T is generated in L2-sized chunks and multiplied on the FP64
// tensor cores (DMMA, gram.cu gemm_tn_tc); fp32 without ADASK_TF32 (or
// unaligned fp64): S chunks + the FP32/FP64-pipe GEMM (gemm.cu).  The TF32
// tensor-core path with S generated on the fly in shared memory is
// gauss_tc.cu (ADASK_TF32).
#include "common.cuh"
#include "gemm.cuh"
#include "rng.cuh"

namespace adask {

int gauss_tc_impl(adask_ctx* ctx, const float* A, int64_t n_local, int64_t d, int64_t lda,
                  int64_t row0, int64_t m, uint64_t key, float* SA, int64_t ldsa, bool accumulate,
                  cudaStream_t st, int64_t kg0, int64_t m_total);

}  // namespace adask

using namespace adask;

// Rows [k0, k0 + mk) of the m_total-row sketch (S scaled by 1/sqrt(m_total)),
// written to SA rows 0 .. mk-1.  adask_sketch_gaussian is k0 = 0, mk = m_total;
// incremental growth (driver.cu) computes only the new rows.
extern "C" int adask_sketch_gaussian_rows(adask_ctx* ctx, int dtype, const void* A, int64_t n_local, int64_t d,
                                          int64_t lda, int64_t row0, int64_t m_total, int64_t k0, int64_t mk,
                                          uint64_t key, void* SA, int64_t ldsa, uint32_t flags, void* stream) {
  ADASK_TRY(use_device(ctx));
  if (m_total < 1 || mk < 1 || k0 < 0 || k0 + mk > m_total)
    return fail(ADASK_E_SKETCH_TOO_LARGE, "sketch rows [%lld, %lld) of m = %lld", (long long)k0,
                (long long)(k0 + mk), (long long)m_total);
  if (n_local < 0 || d < 1 || lda < d || ldsa < d || row0 < 0)
    return fail(ADASK_E_DIM, "sketch_gaussian: bad shape");
  if (dtype != ADASK_F64 && dtype != ADASK_F32) return fail(ADASK_E_ARG, "bad dtype");
  cudaStream_t st = S(stream);
  const size_t esz = dtype == ADASK_F64 ? 8 : 4;
  const bool accumulate = (flags & ADASK_ACCUMULATE) != 0;
  ProfScope prof(ctx, PK_GAUSS, st, (double)n_local * d * esz, 2.0 * (double)mk * n_local * d);
  // tcgen05 path needs 16-byte aligned rows (TMA) and a 4-aligned row offset; otherwise the FP32-pipe GEMM
  if ((flags & ADASK_TF32) && dtype == ADASK_F32 && lda % 4 == 0 && ((uintptr_t)A & 15) == 0 && k0 % 4 == 0) {
    return gauss_tc_impl(ctx, (const float*)A, n_local, d, lda, row0, mk, key, (float*)SA, ldsa, accumulate, st,
                         k0, m_total);
  }
  if (n_local == 0) {
    if (!accumulate) ADASK_CUDA(cudaMemset2DAsync(SA, ldsa * esz, 0, d * esz, mk, st));
    return ADASK_OK;
  }
  // fp64 with 16-byte aligned rows of A: FP64 tensor cores (DMMA).  S^T is
  // generated once per chunk of rows of A (a tile-local on-the-fly generator
  // would repeat the fp64 Box-Muller d / 128 times on the same FP64 pipe the
  // DMMAs use).  ADASK_GAUSS_DMMA=0: the FP64-pipe GEMM;
  // ADASK_GAUSS_CHUNK_MB: S^T bytes per chunk.
  static const bool dmma_on = !(getenv("ADASK_GAUSS_DMMA") && atoi(getenv("ADASK_GAUSS_DMMA")) == 0);
  static const int64_t chunk_mb = getenv("ADASK_GAUSS_CHUNK_MB") ? atoll(getenv("ADASK_GAUSS_CHUNK_MB")) : 256;
  if (dmma_on && dtype == ADASK_F64 && ((uintptr_t)A & 15) == 0 && (lda * esz) % 16 == 0 &&
      ((uintptr_t)SA & 7) == 0) {
    const int64_t lds = (mk + 1) / 2 * 2;
    int64_t nc = (int64_t)((chunk_mb << 20) / (lds * (int64_t)esz));
    nc = std::max<int64_t>(256, nc / 256 * 256);
    nc = std::min<int64_t>(nc, n_local);
    void* wsp = nullptr;
    ADASK_TRY(ctx->ws[WS_GAUSS].get((size_t)lds * nc * esz, st, &wsp));
    for (int64_t c0 = 0; c0 < n_local; c0 += nc) {
      const int64_t w = std::min<int64_t>(nc, n_local - c0);
      ADASK_TRY(philox_gaussian_rows_t(ctx, dtype, k0, mk, m_total, row0 + c0, w, key, wsp, lds, st));
      const void* Ac = (const char*)A + (size_t)c0 * lda * esz;
      ADASK_TRY(gram::gemm_tn_tc(ctx, dtype, wsp, lds, Ac, lda, w, mk, d, SA, ldsa, c0 > 0 || accumulate, st));
    }
    return ADASK_OK;
  }
  // chunk of S columns (rows of A) so that S_chunk stays <= 256 MiB
  int64_t nc = (int64_t)((256ll << 20) / ((int64_t)mk * (int64_t)esz));
  nc = std::max<int64_t>(256, nc / 256 * 256);
  nc = std::min<int64_t>(nc, n_local);
  void* wsp = nullptr;
  ADASK_TRY(ctx->ws[WS_GAUSS].get((size_t)mk * nc * esz, st, &wsp));
  for (int64_t c0 = 0; c0 < n_local; c0 += nc) {
    const int64_t w = std::min<int64_t>(nc, n_local - c0);
    ADASK_TRY(philox_gaussian_rows(ctx, dtype, k0, mk, m_total, row0 + c0, w, key, wsp, w, st));
    const void* Ac = (const char*)A + (size_t)c0 * lda * esz;
    const double beta = (c0 > 0 || accumulate) ? 1.0 : 0.0;
    ADASK_TRY(gemm_impl(ctx, dtype, mk, d, w, 1.0, wsp, w, false, Ac, lda, false, nullptr, beta, SA, ldsa, 0.0,
                        nullptr, false, st));
  }
  return ADASK_OK;
}

extern "C" int adask_sketch_gaussian(adask_ctx* ctx, int dtype, const void* A, int64_t n_local,
                                     int64_t d, int64_t lda, int64_t row0, int64_t m, uint64_t key,
                                     void* SA, int64_t ldsa, uint32_t flags, void* stream) {
  if (m < 1) return fail(ADASK_E_SKETCH_TOO_LARGE, "sketch size must be a positive integer, got %lld",
                         (long long)m);
  return adask_sketch_gaussian_rows(ctx, dtype, A, n_local, d, lda, row0, m, 0, m, key, SA, ldsa, flags, stream);
}

// SA = S A for an explicit m x n sketch matrix S (device, row-major, lds):
// the Gaussian sketch with the reference's own draw (numpy ziggurat normals
// of default_rng(seed), embeddings.py:71-72, generated on the host by the
// caller) when bitwise-equal randomness to the reference is wanted (the
// opt-in rng="numpy" mode of embeddings.set_gaussian_rng).
extern "C" int adask_sketch_dense(adask_ctx* ctx, int dtype, const void* Smat, int64_t m, int64_t n, int64_t lds,
                                  const void* A, int64_t d, int64_t lda, void* SA, int64_t ldsa, void* stream) {
  ADASK_TRY(use_device(ctx));
  if (m < 1 || n < 0 || d < 1 || lds < n || lda < d || ldsa < d) return fail(ADASK_E_DIM, "sketch_dense: bad shape");
  if (dtype != ADASK_F64 && dtype != ADASK_F32) return fail(ADASK_E_ARG, "bad dtype");
  cudaStream_t st = S(stream);
  const size_t esz = dtype == ADASK_F64 ? 8 : 4;
  ProfScope prof(ctx, PK_GAUSS, st, (double)n * d * esz, 2.0 * (double)m * n * d);
  if (n == 0) {
    ADASK_CUDA(cudaMemset2DAsync(SA, ldsa * esz, 0, d * esz, m, st));
    return ADASK_OK;
  }
  return gemm_impl(ctx, dtype, m, d, n, 1.0, Smat, lds, false, A, lda, false, nullptr, 0.0, SA, ldsa, 0.0, nullptr,
                   false, st);
}
