// Preconditioner Grams (preconditioner.py:69-73) and the dense A^T A of
// RegularizedProblem.hessian / direct_solve (problem.py:109-111, 144-149) on
// the FP64 tensor cores: mma.sync f64 (SASS DMMA.8x8x4), the only tensor-core
// kind with fp64 operands on sm_100a (tcgen05 has no f64 kind).
//
//   dense    ("cholesky-d", m >= d):  M = SA^T SA + nu^2 diag(lam)          (d x d)
//   woodbury ("woodbury-m", m <  d):  M = (SA * (1/lam)) SA^T + nu^2 I      (m x m)
//
// Both are SYRK-shaped: only the lower triangle of 128 x 128 C tiles is
// computed.  The dense Gram reduces over the ROWS of SA ("K-outer": both
// operand tiles are row slabs of SA, 128 contiguous columns each); the
// Woodbury capacitance reduces over the COLUMNS ("K-contiguous": operand tiles
// are 128 rows x 128 bytes), with the reference's elementwise SA * (1/lam)
// product formed in registers on the A-side fragments (same rounding as the
// reference's T = SA * (1.0 / lam)).  fp32 data (configs 3-4) is converted to
// fp64 at the fragment load, so the fp32 Grams accumulate in fp64.
//
// Kernel: 256 threads (8 warps as 2 x 4, warp tile 64 x 32 = 4 x 4
// m16n8k4 MMAs), cp.async pipeline (3 stages of 256-byte-deep operand tiles
// on the K-outer side, 4 stages of 128-byte-deep ones on the K-contiguous side)
// with padded pitches that make every fragment load (LDS.128 for fp64,
// LDS.64 for fp32) bank-conflict free, and a fragment-to-C index permutation
// that lets one 16-byte load feed two MMA rows (K-outer) or two k steps
// (K-contiguous).  Deterministic split-K: per-split fp64 partial tiles are
// summed in split order by k_gram_reduce, which also adds nu^2 Lam.
#include "common.cuh"
#include "gemm.cuh"

// bytes of reduction depth per pipeline stage of the K-outer kernels: 256 with
// three stages measured 2-3% faster than 128 with four (one CTA barrier per
// 32 instead of 16 fp64 reduction steps); the K-contiguous side stays at 128
#ifndef GRAM_KO_DEPTH
#define GRAM_KO_DEPTH 256
#endif
namespace adask {
namespace gram {

constexpr int BT = 128;     // C tile edge
constexpr int NT = 256;     // threads: 8 warps, 2 (rows) x 4 (cols)

template <typename T, bool KC>
struct Lay {
  static constexpr int ES = (int)sizeof(T);
  // reduction depth per stage: 128 bytes (K-contiguous), GRAM_KO_DEPTH bytes (K-outer)
  static constexpr int BK = (KC ? 128 : GRAM_KO_DEPTH) / ES;
  static constexpr int NSTAGE = (!KC && GRAM_KO_DEPTH > 128) ? 3 : 4;
  static constexpr int V = 16 / ES;     // elements per 16-byte chunk
  // K-outer: [BK][PITCH] (rows = reduction index, 128 C indices per row);
  // K-contiguous: [BT][PITCH] (rows = C index, BK reduction values per row)
  static constexpr int PITCH_B = KC ? (128 + (ES == 8 ? 64 : 32)) : (BT * ES + 32);
  static constexpr int PITCH = PITCH_B / ES;
  static constexpr int ROWS = KC ? BT : BK;
  static constexpr int OP_BYTES = ROWS * PITCH_B;
  static constexpr int STAGE_BYTES = 2 * OP_BYTES;
  static constexpr int SMEM = NSTAGE * STAGE_BYTES;
  static constexpr int NQ = ROWS * (KC ? BK : BT) / V / 256;  // 16-byte chunks per thread and operand tile
};

struct Args {
  const void* X;     // operand matrix (row-major, ld elements, 16-byte aligned rows)
  int64_t ld;
  int64_t K;         // reduction length
  int64_t N;         // C is N x N
  const double* rl;  // K-contiguous only: 1/lam, padded to a multiple of BK (nullable)
  int nb;            // C tiles per dimension
  int splits;
  int64_t kchunk;    // reduction values per split (multiple of BK)
  void* M;           // output (splits == 1), lower triangle, ldm
  int64_t ldm;
  double nu2;        // diagonal add nu2 * (lam ? lam[i] : 1)
  const double* lam;
  double* part;      // splits > 1: [tile][split][BT][BT] fp64 partials
};

__device__ __forceinline__ void cp_async16(uint32_t saddr, const void* g, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(saddr), "l"(g), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ void dmma(double (&c)[4], double a0, double a1, double b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a0), "d"(a1), "d"(b0));
}

// two consecutive elements at p (16- or 8-byte aligned) as doubles
template <typename T>
__device__ __forceinline__ double2 lds2(const T* p) {
  if constexpr (sizeof(T) == 8) {
    return *reinterpret_cast<const double2*>(p);
  } else {
    const float2 f = *reinterpret_cast<const float2*>(p);
    return make_double2((double)f.x, (double)f.y);
  }
}

// Lower-triangle tile t -> (bi, bj), bj <= bi.
__device__ __forceinline__ void tile_of(int t, int& bi, int& bj) {
  int i = (int)((sqrtf(8.0f * (float)t + 1.0f) - 1.0f) * 0.5f);
  while ((i + 1) * (i + 2) / 2 <= t) ++i;
  while (i * (i + 1) / 2 > t) --i;
  bi = i;
  bj = t - i * (i + 1) / 2;
}

// Issue the cp.async copies of one operand tile (C-index block c0) for the
// reduction slab [k0, k0 + BK) (zero-filled past kend / N).
template <typename T, bool KC>
__device__ __forceinline__ void load_tile(const void* Xv, int64_t ld, int64_t N, uint32_t sbase, int64_t c0,
                                          int64_t k0, int64_t kend) {
  using Lt = Lay<T, KC>;
  const T* X = reinterpret_cast<const T*>(Xv);
#pragma unroll
  for (int q = 0; q < Lt::NQ; ++q) {
    const int c = threadIdx.x + NT * q;  // chunk index within the operand tile
    int r, cc;
    int64_t grow, gcol;
    int bytes;
    if constexpr (!KC) {
      r = c / (BT / Lt::V);
      cc = (c % (BT / Lt::V)) * Lt::V;
      grow = k0 + r;
      gcol = c0 + cc;
      const int64_t left = N - gcol;
      bytes = (grow < kend && left > 0) ? (int)(left >= Lt::V ? 16 : left * Lt::ES) : 0;
    } else {
      r = c / (Lt::BK / Lt::V);
      cc = (c % (Lt::BK / Lt::V)) * Lt::V;
      grow = c0 + r;
      gcol = k0 + cc;
      const int64_t left = kend - gcol;
      bytes = (grow < N && left > 0) ? (int)(left >= Lt::V ? 16 : left * Lt::ES) : 0;
    }
    const T* g = bytes ? X + grow * ld + gcol : X;
    cp_async16(sbase + (uint32_t)(r * Lt::PITCH_B + cc * Lt::ES), g, bytes);
  }
}

template <typename T, bool KC, typename OUT>
__global__ void __launch_bounds__(NT, 1) k_gram_dmma(Args a) {
  using Lt = Lay<T, KC>;
  extern __shared__ __align__(128) unsigned char smem[];
  pdl_wait();
  const int tile = blockIdx.x / a.splits, split = blockIdx.x % a.splits;
  int bi, bj;
  tile_of(tile, bi, bj);
  const bool diag = bi == bj;
  const int64_t ci = (int64_t)bi * BT, cj = (int64_t)bj * BT;
  const int64_t kbeg = (int64_t)split * a.kchunk;
  const int64_t kend = min(a.K, kbeg + a.kchunk);
  const int nst = kend > kbeg ? (int)((kend - kbeg + Lt::BK - 1) / Lt::BK) : 0;
  const uint32_t s0 = (uint32_t)__cvta_generic_to_shared(smem);

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, tig = lane & 3;
  const int wm = warp >> 2, wn = warp & 3;  // warp tile rows wm*64, cols wn*32
  // warps whose 64 x 32 band lies outside C (small N) or strictly above the
  // diagonal of a diagonal tile skip the fragment loads and MMAs
  const bool active = (ci + wm * 64 < a.N) && (cj + wn * 32 < a.N) && !(diag && wn * 32 > wm * 64 + 63);

  double acc[4][4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[i][j][e] = 0.0;

  auto issue = [&](int stage_slot, int st_idx) {
    const uint32_t sb = s0 + (uint32_t)(stage_slot * Lt::STAGE_BYTES);
    const int64_t k0 = kbeg + (int64_t)st_idx * Lt::BK;
    load_tile<T, KC>(a.X, a.ld, a.N, sb, ci, k0, kend);
    if (!diag) load_tile<T, KC>(a.X, a.ld, a.N, sb + Lt::OP_BYTES, cj, k0, kend);
  };

#pragma unroll
  for (int s = 0; s < Lt::NSTAGE - 1; ++s) {
    if (s < nst) issue(s, s);
    cp_commit();
  }
  for (int it = 0; it < nst; ++it) {
    cp_wait<Lt::NSTAGE - 2>();
    __syncthreads();
    {
      const int nx = it + Lt::NSTAGE - 1;
      if (nx < nst) issue(nx % Lt::NSTAGE, nx);
      cp_commit();
    }
    if (!active) continue;
    const unsigned char* sb = smem + (it % Lt::NSTAGE) * Lt::STAGE_BYTES;
    const T* As = reinterpret_cast<const T*>(sb);
    const T* Bs = reinterpret_cast<const T*>(diag ? sb : sb + Lt::OP_BYTES);
    if constexpr (!KC) {
      // k4 step q: MMA row g <-> tile row 2g, row g+8 <-> 2g+1 (one 16-byte
      // load per lane feeds both); n subtile ni = 2np+e <-> tile col
      // 16np + 2c + e for MMA col c.
#pragma unroll
      for (int q = 0; q < Lt::BK / 4; ++q) {
        const T* arow = As + (4 * q + tig) * Lt::PITCH + wm * 64 + 2 * g;
        const T* brow = Bs + (4 * q + tig) * Lt::PITCH + wn * 32 + 2 * g;
        double2 av[4], bv[2];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) av[mi] = lds2<T>(arow + 16 * mi);
#pragma unroll
        for (int np = 0; np < 2; ++np) bv[np] = lds2<T>(brow + 16 * np);
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) {
          dmma(acc[mi][0], av[mi].x, av[mi].y, bv[0].x);
          dmma(acc[mi][1], av[mi].x, av[mi].y, bv[0].y);
          dmma(acc[mi][2], av[mi].x, av[mi].y, bv[1].x);
          dmma(acc[mi][3], av[mi].x, av[mi].y, bv[1].y);
        }
      }
    } else {
      // step pair s: lane tig takes reduction index 8s + 2 tig (step 2s) and
      // 8s + 2 tig + 1 (step 2s + 1), so one 16-byte load covers both steps.
      const int64_t k0 = kbeg + (int64_t)it * Lt::BK;
#pragma unroll
      for (int s = 0; s < Lt::BK / 8; ++s) {
        double2 r2 = make_double2(1.0, 1.0);
        if (a.rl) r2 = __ldg(reinterpret_cast<const double2*>(a.rl + k0 + 8 * s + 2 * tig));
        double2 bv[4];
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) bv[ni] = lds2<T>(Bs + (wn * 32 + 8 * ni + g) * Lt::PITCH + 8 * s + 2 * tig);
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) {
          double2 v0 = lds2<T>(As + (wm * 64 + 16 * mi + g) * Lt::PITCH + 8 * s + 2 * tig);
          double2 v1 = lds2<T>(As + (wm * 64 + 16 * mi + g + 8) * Lt::PITCH + 8 * s + 2 * tig);
          v0.x *= r2.x;  // T = SA * (1/lam), preconditioner.py:72
          v0.y *= r2.y;
          v1.x *= r2.x;
          v1.y *= r2.y;
#pragma unroll
          for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni], v0.x, v1.x, bv[ni].x);
#pragma unroll
          for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni], v0.y, v1.y, bv[ni].y);
        }
      }
    }
  }
  cp_wait<0>();

  // epilogue: C fragment c0 (MMA row g, col 2tig), c1 (g, 2tig+1), c2 (g+8, 2tig), c3 (g+8, 2tig+1)
  if (!active && a.splits == 1) return;
  const bool direct = a.splits == 1;
  double* part = direct ? nullptr : a.part + ((int64_t)tile * a.splits + split) * (BT * BT);
  OUT* M = reinterpret_cast<OUT*>(a.M);
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        int r, c;
        if constexpr (!KC) {
          r = wm * 64 + 16 * mi + 2 * g + (e >> 1);
          c = wn * 32 + 16 * (ni >> 1) + 2 * (2 * tig + (e & 1)) + (ni & 1);
        } else {
          r = wm * 64 + 16 * mi + g + 8 * (e >> 1);
          c = wn * 32 + 8 * ni + 2 * tig + (e & 1);
        }
        const double v = acc[mi][ni][e];
        if (!direct) {
          part[r * BT + c] = v;
        } else {
          const int64_t gr = ci + r, gc = cj + c;
          if (gr < a.N && gc <= gr) {
            double out = v;
            if (gr == gc && a.nu2 != 0.0) out += a.nu2 * (a.lam ? a.lam[gr] : 1.0);
            M[gr * a.ldm + gc] = (OUT)out;
          }
        }
      }
}

template <typename OUT>
__global__ void k_gram_reduce(Args a) {
  pdl_wait();
  const int tile = blockIdx.x;
  int bi, bj;
  tile_of(tile, bi, bj);
  const int64_t ci = (int64_t)bi * BT, cj = (int64_t)bj * BT;
  const double* P = a.part + (int64_t)tile * a.splits * (BT * BT);
  OUT* M = reinterpret_cast<OUT*>(a.M);
  for (int e = blockIdx.y * blockDim.x + threadIdx.x; e < BT * BT; e += gridDim.y * blockDim.x) {
    const int r = e / BT, c = e % BT;
    const int64_t gr = ci + r, gc = cj + c;
    if (gr >= a.N || gc > gr) continue;
    double v = 0.0;
    for (int s = 0; s < a.splits; ++s) v += P[(int64_t)s * (BT * BT) + e];
    if (gr == gc && a.nu2 != 0.0) v += a.nu2 * (a.lam ? a.lam[gr] : 1.0);
    M[gr * a.ldm + gc] = (OUT)v;
  }
}

// strided copy into a 16-byte aligned, zero-padded buffer (odd shapes only)
template <typename T>
__global__ void k_pack(const T* X, int64_t rows, int64_t cols, int64_t ld, T* out, int64_t ldo) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= rows * ldo) return;
  const int64_t i = e / ldo, j = e - i * ldo;
  out[e] = j < cols ? X[i * ld + j] : (T)0;
}

__global__ void k_recip_pad(const double* lam, int64_t d, int64_t dpad, double* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < dpad) out[i] = i < d ? 1.0 / lam[i] : 0.0;
}

// Split-K factor from a small cost model (units ~ one 128x128x(128 B) stage
// of one CTA, ~2 us on the FP64 tensor pipe): waves x (prologue + stages per
// split) + the fixed-order reduction of the partial tiles.
int choose_splits(int tiles, int64_t ksteps) {
  int best = 1;
  double best_cost = 1e300;
  for (int s = 1; s <= 256 && s <= ksteps; ++s) {
    const int64_t ctas = (int64_t)tiles * s;
    const double waves = std::ceil((double)ctas / kNumSMs);
    const double per = 1.0 + (double)cdiv(ksteps, s);
    const double red = s > 1 ? 1.0 + 0.02 * (double)tiles * s / kNumSMs * 8.0 : 0.0;
    const double cost = waves * per + red;
    if (cost < best_cost - 1e-9) {
      best_cost = cost;
      best = s;
    }
  }
  return best;
}

template <typename T, bool KC, typename OUT>
int run(adask_ctx* ctx, Args a, cudaStream_t st) {
  using Lt = Lay<T, KC>;
  a.nb = (int)cdiv(a.N, BT);
  const int tiles = a.nb * (a.nb + 1) / 2;
  const int64_t ksteps = cdiv(a.K, Lt::BK);
  a.splits = choose_splits(tiles, ksteps);
  a.kchunk = cdiv(ksteps, a.splits) * Lt::BK;
  a.splits = (int)cdiv(a.K, a.kchunk);  // no empty split
  if (a.splits < 1) a.splits = 1;
  if (a.splits > 1) {
    void* w = nullptr;
    ADASK_TRY(ctx->ws[WS_GEMM].get((size_t)tiles * a.splits * BT * BT * sizeof(double), st, &w));
    a.part = (double*)w;
  }
  auto kern = k_gram_dmma<T, KC, OUT>;
  ADASK_TRY(ensure_smem_attr((const void*)kern, Lt::SMEM));
  ADASK_CUDA(launch_pdl(kern, dim3((unsigned)(tiles * a.splits)), dim3(NT), (size_t)Lt::SMEM, st, a));
  ctx->launches++;
  if (a.splits > 1) {
    // one element per thread: the split loads of every element are in flight at once
    ADASK_CUDA(launch_pdl(k_gram_reduce<OUT>, dim3((unsigned)tiles, BT * BT / 256), dim3(256), 0, st, a));
    ctx->launches++;
  }
  return ADASK_OK;
}

// ---------------------------------------------------------------------------
// Rectangular C (M x N) = X^T Y (+ C), X K x M and Y K x N row-major: the same
// K-outer DMMA tile kernel over a full tile grid.  Used by the fp64 Gaussian
// sketch (gauss.cu): X = S^T chunk (Philox normals, generated once per chunk
// and L2-resident), Y = the rows of A of the chunk.  Deterministic split-K.
struct RArgs {
  const void* X;
  int64_t ldx;
  const void* Y;
  int64_t ldy;
  int64_t K, M, N;
  int nbn;           // C tiles per row of tiles
  int splits;
  int64_t kchunk;
  void* C;
  int64_t ldc;
  int accumulate;
  double* part;      // splits > 1: [tile][split][BT][BT]
};

template <typename T, typename OUT>
__global__ void __launch_bounds__(NT, 1) k_gemm_tn_dmma(RArgs a) {
  using Lt = Lay<T, false>;
  extern __shared__ __align__(128) unsigned char smem[];
  pdl_wait();
  const int tile = blockIdx.x / a.splits, split = blockIdx.x % a.splits;
  const int bi = tile / a.nbn, bj = tile % a.nbn;
  const int64_t ci = (int64_t)bi * BT, cj = (int64_t)bj * BT;
  const int64_t kbeg = (int64_t)split * a.kchunk;
  const int64_t kend = min(a.K, kbeg + a.kchunk);
  const int nst = kend > kbeg ? (int)((kend - kbeg + Lt::BK - 1) / Lt::BK) : 0;
  const uint32_t s0 = (uint32_t)__cvta_generic_to_shared(smem);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, tig = lane & 3;
  const int wm = warp >> 2, wn = warp & 3;
  const bool active = (ci + wm * 64 < a.M) && (cj + wn * 32 < a.N);

  double acc[4][4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[i][j][e] = 0.0;

  auto issue = [&](int stage_slot, int st_idx) {
    const uint32_t sb = s0 + (uint32_t)(stage_slot * Lt::STAGE_BYTES);
    const int64_t k0 = kbeg + (int64_t)st_idx * Lt::BK;
    load_tile<T, false>(a.X, a.ldx, a.M, sb, ci, k0, kend);
    load_tile<T, false>(a.Y, a.ldy, a.N, sb + Lt::OP_BYTES, cj, k0, kend);
  };
#pragma unroll
  for (int s = 0; s < Lt::NSTAGE - 1; ++s) {
    if (s < nst) issue(s, s);
    cp_commit();
  }
  for (int it = 0; it < nst; ++it) {
    cp_wait<Lt::NSTAGE - 2>();
    __syncthreads();
    {
      const int nx = it + Lt::NSTAGE - 1;
      if (nx < nst) issue(nx % Lt::NSTAGE, nx);
      cp_commit();
    }
    if (!active) continue;
    const unsigned char* sb = smem + (it % Lt::NSTAGE) * Lt::STAGE_BYTES;
    const T* As = reinterpret_cast<const T*>(sb);
    const T* Bs = reinterpret_cast<const T*>(sb + Lt::OP_BYTES);
#pragma unroll
    for (int q = 0; q < Lt::BK / 4; ++q) {  // fragment <-> C index permutation as in k_gram_dmma
      const T* arow = As + (4 * q + tig) * Lt::PITCH + wm * 64 + 2 * g;
      const T* brow = Bs + (4 * q + tig) * Lt::PITCH + wn * 32 + 2 * g;
      double2 av[4], bv[2];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) av[mi] = lds2<T>(arow + 16 * mi);
#pragma unroll
      for (int np = 0; np < 2; ++np) bv[np] = lds2<T>(brow + 16 * np);
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) {
        dmma(acc[mi][0], av[mi].x, av[mi].y, bv[0].x);
        dmma(acc[mi][1], av[mi].x, av[mi].y, bv[0].y);
        dmma(acc[mi][2], av[mi].x, av[mi].y, bv[1].x);
        dmma(acc[mi][3], av[mi].x, av[mi].y, bv[1].y);
      }
    }
  }
  cp_wait<0>();
  if (!active && a.splits == 1) return;
  const bool direct = a.splits == 1;
  double* part = direct ? nullptr : a.part + ((int64_t)tile * a.splits + split) * (BT * BT);
  OUT* C = reinterpret_cast<OUT*>(a.C);
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int r = wm * 64 + 16 * mi + 2 * g + (e >> 1);
        const int c = wn * 32 + 16 * (ni >> 1) + 2 * (2 * tig + (e & 1)) + (ni & 1);
        const double v = acc[mi][ni][e];
        if (!direct) {
          part[r * BT + c] = v;
        } else {
          const int64_t gr = ci + r, gc = cj + c;
          if (gr < a.M && gc < a.N) {
            OUT* o = C + gr * a.ldc + gc;
            *o = (OUT)(a.accumulate ? (double)*o + v : v);
          }
        }
      }
}

template <typename OUT>
__global__ void k_gemm_tn_reduce(RArgs a) {
  pdl_wait();
  const int tile = blockIdx.x;
  const int bi = tile / a.nbn, bj = tile % a.nbn;
  const int64_t ci = (int64_t)bi * BT, cj = (int64_t)bj * BT;
  const double* P = a.part + (int64_t)tile * a.splits * (BT * BT);
  OUT* C = reinterpret_cast<OUT*>(a.C);
  for (int e = blockIdx.y * blockDim.x + threadIdx.x; e < BT * BT; e += gridDim.y * blockDim.x) {
    const int r = e / BT, c = e % BT;
    const int64_t gr = ci + r, gc = cj + c;
    if (gr >= a.M || gc >= a.N) continue;
    double v = 0.0;
    for (int s = 0; s < a.splits; ++s) v += P[(int64_t)s * (BT * BT) + e];
    OUT* o = C + gr * a.ldc + gc;
    *o = (OUT)(a.accumulate ? (double)*o + v : v);
  }
}

// C (M x N, dtype) = X^T Y (+ C): X K x M, Y K x N, both `dtype`, 16-byte
// aligned rows (the caller checks).
int gemm_tn_tc(adask_ctx* ctx, int dtype, const void* X, int64_t ldx, const void* Y, int64_t ldy, int64_t K,
               int64_t M, int64_t N, void* C, int64_t ldc, bool accumulate, cudaStream_t st) {
  if (M < 1 || N < 1) return ADASK_OK;
  RArgs a{};
  a.X = X;
  a.ldx = ldx;
  a.Y = Y;
  a.ldy = ldy;
  a.K = K;
  a.M = M;
  a.N = N;
  a.C = C;
  a.ldc = ldc;
  a.accumulate = accumulate ? 1 : 0;
  a.nbn = (int)cdiv(N, BT);
  const int tiles = (int)cdiv(M, BT) * a.nbn;
  const int BK = dtype == ADASK_F64 ? Lay<double, false>::BK : Lay<float, false>::BK;
  const int64_t ksteps = std::max<int64_t>(1, cdiv(K, BK));
  a.splits = choose_splits(tiles, ksteps);
  a.kchunk = cdiv(ksteps, a.splits) * BK;
  a.splits = (int)std::max<int64_t>(1, cdiv(K, a.kchunk));
  if (a.splits > 1) {
    void* w = nullptr;
    ADASK_TRY(ctx->ws[WS_GEMM].get((size_t)tiles * a.splits * BT * BT * sizeof(double), st, &w));
    a.part = (double*)w;
  }
  if (dtype == ADASK_F64) {
    auto kern = k_gemm_tn_dmma<double, double>;
    ADASK_TRY(ensure_smem_attr((const void*)kern, Lay<double, false>::SMEM));
    ADASK_CUDA(launch_pdl(kern, dim3((unsigned)(tiles * a.splits)), dim3(NT), (size_t)Lay<double, false>::SMEM, st, a));
  } else {
    auto kern = k_gemm_tn_dmma<float, float>;
    ADASK_TRY(ensure_smem_attr((const void*)kern, Lay<float, false>::SMEM));
    ADASK_CUDA(launch_pdl(kern, dim3((unsigned)(tiles * a.splits)), dim3(NT), (size_t)Lay<float, false>::SMEM, st, a));
  }
  ctx->launches++;
  if (a.splits > 1) {
    if (dtype == ADASK_F64)
      ADASK_CUDA(launch_pdl(k_gemm_tn_reduce<double>, dim3((unsigned)tiles, BT * BT / 256), dim3(256), 0, st, a));
    else
      ADASK_CUDA(launch_pdl(k_gemm_tn_reduce<float>, dim3((unsigned)tiles, BT * BT / 256), dim3(256), 0, st, a));
    ctx->launches++;
  }
  return ADASK_OK;
}

// C (N x N, lower) = X^T X (K-outer: X is K x N) or (X D) X^T (K-contiguous:
// X is N x K, D = diag(rl)), + nu2 (lam or 1) on the diagonal, into M (dtype).
int gram_tc(adask_ctx* ctx, int dtype, const void* X, int64_t ld, int64_t K, int64_t N, bool kc,
            const double* rl, double nu2, const double* lam, void* M, int64_t ldm, bool out_f64, cudaStream_t st) {
  const int es = dtype == ADASK_F64 ? 8 : 4;
  const int64_t cols = kc ? K : N, rows = kc ? N : K;
  if (N < 1) return ADASK_OK;
  Args a{};
  a.X = X;
  a.ld = ld;
  a.K = K;
  a.N = N;
  a.rl = rl;
  a.M = M;
  a.ldm = ldm;
  a.nu2 = nu2;
  a.lam = lam;
  if (((uintptr_t)X % 16) != 0 || (ld * es) % 16 != 0) {
    // odd shapes (tests, tiny problems): pack into a 16-byte aligned copy
    const int64_t ldp = cdiv(cols * es, 16) * 16 / es;
    void* w = nullptr;
    ADASK_TRY(ctx->ws[WS_GRAM_PACK].get((size_t)(rows * ldp) * es + 256, st, &w));
    const int64_t tot = rows * ldp;
    if (tot > 0) {
      if (dtype == ADASK_F64)
        k_pack<double><<<(unsigned)cdiv(tot, 256), 256, 0, st>>>((const double*)X, rows, cols, ld, (double*)w, ldp);
      else
        k_pack<float><<<(unsigned)cdiv(tot, 256), 256, 0, st>>>((const float*)X, rows, cols, ld, (float*)w, ldp);
      ADASK_LAUNCHED(ctx);
    }
    a.X = w;
    a.ld = ldp;
  }
  if (dtype == ADASK_F64)
    return kc ? run<double, true, double>(ctx, a, st) : run<double, false, double>(ctx, a, st);
  if (out_f64 && !kc) return run<float, false, double>(ctx, a, st);  // fp32 data, fp64 Hessian (direct_solve)
  return kc ? run<float, true, float>(ctx, a, st) : run<float, false, float>(ctx, a, st);
}

}  // namespace gram

int gram_dense(adask_ctx* ctx, int dtype, const void* SA, int64_t m, int64_t d, int64_t ldsa, double nu2,
               const double* lam, void* M, int64_t ldm, cudaStream_t st) {
  return gram::gram_tc(ctx, dtype, SA, ldsa, m, d, false, nullptr, nu2, lam, M, ldm, false, st);
}

int gram_woodbury(adask_ctx* ctx, int dtype, const void* SA, int64_t m, int64_t d, int64_t ldsa, double nu2,
                  const double* lam, void* M, int64_t ldm, cudaStream_t st) {
  // 1/lam, zero-padded to a multiple of the deepest stage (32 values)
  const int64_t dpad = cdiv(d, 32) * 32 + 32;
  void* w = nullptr;
  ADASK_TRY(ctx->ws[WS_GRAM_RL].get((size_t)dpad * sizeof(double), st, &w));
  gram::k_recip_pad<<<(unsigned)cdiv(dpad, 256), 256, 0, st>>>(lam, d, dpad, (double*)w);
  ADASK_LAUNCHED(ctx);
  return gram::gram_tc(ctx, dtype, SA, ldsa, d, m, true, (const double*)w, nu2, nullptr, M, ldm, false, st);
}

}  // namespace adask
