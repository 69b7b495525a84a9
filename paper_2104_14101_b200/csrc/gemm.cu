// Register-blocked SMEM-tiled GEMM for fp64 (DFMA) and fp32 (FFMA), used by
// the preconditioner Gram / capacitance matrices (preconditioner.py:69-73),
// the blocked Cholesky / triangular inverse (linalg.py:30-55) and the
// materialized-S Gaussian sketch (embeddings.py:71-73).
//
// C = alpha * opA(A) diag(kscale) opB(B) + beta * C + diag_add      (M x N)
// opA(i,k) = TA ? A[k*lda + i] : A[i*lda + k];  opB(k,j) = TB ? B[j*ldb + k] : B[k*ldb + j]
// `lower` restricts the work and the writes to j <= i (SYRK-style).
// 128 x 128 CTA tile, 16 x 16 threads with 8 x 8 register micro-tiles
// (16-byte interleaved so SMEM reads are conflict-free), double-buffered SMEM
// with register prefetch, optional deterministic split-K (fixed-order
// reduction of the per-split partials).  fp64 has no tcgen05 kind on sm_100a;
// this is the FP64-pipe path.  The fp32 tensor-core (TF32 tcgen05) path for
// the Gaussian sketch lives in gauss_tc.cu.
#include "common.cuh"
#include "gemm.cuh"

namespace adask {

struct GemmArgs {
  int64_t M, N, K;
  const void* A;
  int64_t lda;
  const void* B;
  int64_t ldb;
  const double* kscale;
  double alpha, beta;
  void* C;
  int64_t ldc;
  double dscal;
  const double* dvec;
  int lower;
  int splits;
  double* part;  // splits > 1: [splits][M][N] partials
};

template <typename T>
struct GemmCfg {
  static constexpr int BM = 128, BN = 128;
  static constexpr int BK = sizeof(T) == 8 ? 8 : 16;
  static constexpr int V = 16 / sizeof(T);  // elements per 16-byte vector
  static constexpr int TM = 8, TN = 8;
  static constexpr int LPT = BM * BK / 256;  // loads per thread per operand
  static constexpr int PAD = V;
};

template <typename T, bool TRANS, bool IS_A>
__device__ __forceinline__ void gemm_load(const GemmArgs& g, int64_t mn0, int64_t k0,
                                          T (&r)[GemmCfg<T>::LPT]) {
  using Cf = GemmCfg<T>;
  const int t = threadIdx.x;
  const T* P = reinterpret_cast<const T*>(IS_A ? g.A : g.B);
  const int64_t ld = IS_A ? g.lda : g.ldb;
  const int64_t MN = IS_A ? g.M : g.N;
  // contiguous along k when (IS_A && !TRANS) || (!IS_A && TRANS)
  constexpr bool KCONT = IS_A ? !TRANS : TRANS;
  if constexpr (KCONT) {
    constexpr int TPR = Cf::BK / Cf::LPT;  // threads per row
    const int row = t / TPR, kk = (t % TPR) * Cf::LPT;
    const int64_t gi = mn0 + row;
#pragma unroll
    for (int e = 0; e < Cf::LPT; ++e) {
      const int64_t gk = k0 + kk + e;
      r[e] = (gi < MN && gk < g.K) ? P[gi * ld + gk] : (T)0;
    }
  } else {
    constexpr int TPR = Cf::BM / Cf::LPT;
    const int kr = t / TPR, ii = (t % TPR) * Cf::LPT;
    const int64_t gk = k0 + kr;
#pragma unroll
    for (int e = 0; e < Cf::LPT; ++e) {
      const int64_t gi = mn0 + ii + e;
      r[e] = (gi < MN && gk < g.K) ? P[gk * ld + gi] : (T)0;
    }
  }
}

template <typename T, bool TRANS, bool IS_A>
__device__ __forceinline__ void gemm_store(const GemmArgs& g, int64_t k0, const T (&r)[GemmCfg<T>::LPT],
                                           T* sm /*[BK][BM+PAD]*/) {
  using Cf = GemmCfg<T>;
  constexpr int LDS = Cf::BM + Cf::PAD;
  const int t = threadIdx.x;
  constexpr bool KCONT = IS_A ? !TRANS : TRANS;
  if constexpr (KCONT) {
    constexpr int TPR = Cf::BK / Cf::LPT;
    const int row = t / TPR, kk = (t % TPR) * Cf::LPT;
#pragma unroll
    for (int e = 0; e < Cf::LPT; ++e) {
      T v = r[e];
      if (IS_A && g.kscale) {
        const int64_t gk = k0 + kk + e;
        if (gk < g.K) v = (T)((double)v * g.kscale[gk]);
      }
      sm[(kk + e) * LDS + row] = v;
    }
  } else {
    constexpr int TPR = Cf::BM / Cf::LPT;
    const int kr = t / TPR, ii = (t % TPR) * Cf::LPT;
    double ks = 1.0;
    if (IS_A && g.kscale) {
      const int64_t gk = k0 + kr;
      if (gk < g.K) ks = g.kscale[gk];
    }
#pragma unroll
    for (int e = 0; e < Cf::LPT; ++e) {
      T v = r[e];
      if (IS_A && g.kscale) v = (T)((double)v * ks);
      sm[kr * LDS + ii + e] = v;
    }
  }
}

template <typename T, bool TA, bool TB>
__global__ void __launch_bounds__(256, 1) k_gemm(GemmArgs g) {
  using Cf = GemmCfg<T>;
  constexpr int BM = Cf::BM, BN = Cf::BN, BK = Cf::BK, V = Cf::V;
  constexpr int LDS = BM + Cf::PAD;
  __shared__ __align__(16) T As[2][BK * LDS];
  __shared__ __align__(16) T Bs[2][BK * LDS];

  const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;
  if (g.lower && n0 > m0 + BM - 1) return;
  const int tid = threadIdx.x, tr = tid / 16, tc = tid % 16;

  const int64_t ktiles = (g.K + BK - 1) / BK;
  const int64_t kt0 = ktiles * blockIdx.z / g.splits, kt1 = ktiles * (blockIdx.z + 1) / g.splits;

  T acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = (T)0;

  T ra[Cf::LPT], rb[Cf::LPT];
  int buf = 0;
  if (kt0 < kt1) {
    gemm_load<T, TA, true>(g, m0, kt0 * BK, ra);
    gemm_load<T, TB, false>(g, n0, kt0 * BK, rb);
    gemm_store<T, TA, true>(g, kt0 * BK, ra, As[0]);
    gemm_store<T, TB, false>(g, kt0 * BK, rb, Bs[0]);
  }
  __syncthreads();
  for (int64_t kt = kt0; kt < kt1; ++kt) {
    const bool more = kt + 1 < kt1;
    if (more) {
      gemm_load<T, TA, true>(g, m0, (kt + 1) * BK, ra);
      gemm_load<T, TB, false>(g, n0, (kt + 1) * BK, rb);
    }
    const T* as = As[buf];
    const T* bs = Bs[buf];
#pragma unroll
    for (int k = 0; k < BK; ++k) {
      T a[8], b[8];
#pragma unroll
      for (int q = 0; q < 8 / V; ++q) {
#pragma unroll
        for (int v = 0; v < V; ++v) {
          a[q * V + v] = as[k * LDS + q * 16 * V + tr * V + v];
          b[q * V + v] = bs[k * LDS + q * 16 * V + tc * V + v];
        }
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
    if (more) {
      gemm_store<T, TA, true>(g, (kt + 1) * BK, ra, As[buf ^ 1]);
      gemm_store<T, TB, false>(g, (kt + 1) * BK, rb, Bs[buf ^ 1]);
    }
    __syncthreads();
    buf ^= 1;
  }

  // epilogue
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t gi = m0 + (i / V) * 16 * V + tr * V + (i % V);
    if (gi >= g.M) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int64_t gj = n0 + (j / V) * 16 * V + tc * V + (j % V);
      if (gj >= g.N) continue;
      if (g.lower && gj > gi) continue;
      if (g.splits > 1) {
        g.part[((int64_t)blockIdx.z * g.M + gi) * g.N + gj] = (double)acc[i][j];
      } else {
        T* c = reinterpret_cast<T*>(g.C) + gi * g.ldc + gj;
        double v = g.alpha * (double)acc[i][j];
        if (g.beta != 0.0) v += g.beta * (double)(*c);
        if (gi == gj && g.dscal != 0.0) v += g.dscal * (g.dvec ? g.dvec[gi] : 1.0);
        *c = (T)v;
      }
    }
  }
}

template <typename T>
__global__ void k_gemm_splitk_reduce(GemmArgs g) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= g.M * g.N) return;
  const int64_t gi = idx / g.N, gj = idx % g.N;
  if (g.lower && gj > gi) return;
  double s = 0.0;
  for (int z = 0; z < g.splits; ++z) s += g.part[(int64_t)z * g.M * g.N + idx];
  T* c = reinterpret_cast<T*>(g.C) + gi * g.ldc + gj;
  double v = g.alpha * s;
  if (g.beta != 0.0) v += g.beta * (double)(*c);
  if (gi == gj && g.dscal != 0.0) v += g.dscal * (g.dvec ? g.dvec[gi] : 1.0);
  *c = (T)v;
}

template <typename T, bool TA, bool TB>
static int launch_gemm(adask_ctx* ctx, GemmArgs g, cudaStream_t st) {
  dim3 grid((unsigned)cdiv(g.N, 128), (unsigned)cdiv(g.M, 128), (unsigned)g.splits);
  k_gemm<T, TA, TB><<<grid, 256, 0, st>>>(g);
  ADASK_LAUNCHED(ctx);
  if (g.splits > 1) {
    k_gemm_splitk_reduce<T><<<(unsigned)cdiv(g.M * g.N, 256), 256, 0, st>>>(g);
    ADASK_LAUNCHED(ctx);
  }
  return ADASK_OK;
}

int gemm_impl(adask_ctx* ctx, int dtype, int64_t M, int64_t N, int64_t K, double alpha,
              const void* A, int64_t lda, bool ta, const void* B, int64_t ldb, bool tb,
              const double* kscale, double beta, void* C, int64_t ldc, double dscal,
              const double* dvec, bool lower, cudaStream_t st, int ws_slot) {
  if (M <= 0 || N <= 0) return ADASK_OK;
  GemmArgs g{};
  g.M = M;
  g.N = N;
  g.K = K;
  g.A = A;
  g.lda = lda;
  g.B = B;
  g.ldb = ldb;
  g.kscale = kscale;
  g.alpha = alpha;
  g.beta = beta;
  g.C = C;
  g.ldc = ldc;
  g.dscal = dscal;
  g.dvec = dvec;
  g.lower = lower ? 1 : 0;
  // split-K so that the grid covers >= ~2 waves of 148 SMs when K is deep
  int64_t tiles = cdiv(M, 128) * cdiv(N, 128);
  if (lower) tiles = (tiles + cdiv(M, 128)) / 2;
  const int bk = dtype == ADASK_F64 ? 8 : 16;
  const int64_t ktiles = cdiv(K, bk);
  int splits = 1;
  while (tiles * splits < 2 * kNumSMs && ktiles / (splits * 2) >= 16 && splits < 64) splits *= 2;
  g.splits = splits;
  if (splits > 1) {
    void* wsp = nullptr;
    ADASK_TRY(ctx->ws[ws_slot].get((size_t)splits * M * N * sizeof(double), st, &wsp));
    g.part = (double*)wsp;
  }
  if (K <= 0) {
    // C = beta C + diag
    g.splits = 1;
  }
#define GO(TT)                                                    \
  do {                                                            \
    if (!ta && !tb) return launch_gemm<TT, false, false>(ctx, g, st); \
    if (!ta && tb) return launch_gemm<TT, false, true>(ctx, g, st);   \
    if (ta && !tb) return launch_gemm<TT, true, false>(ctx, g, st);   \
    return launch_gemm<TT, true, true>(ctx, g, st);                   \
  } while (0)
  if (dtype == ADASK_F64) GO(double);
  GO(float);
#undef GO
}

}  // namespace adask
