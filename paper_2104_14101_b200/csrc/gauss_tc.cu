// TF32 tensor-core Gaussian sketch  SA = S A  (tcgen05 + TMEM + TMA), fp32.
//                                     reference: embeddings.py:66-73
//
// S (m x n) never exists in memory.  A CTA pair (2-CTA cluster) computes a
// 256 x 512 tile of SA over a slice of the rows of A with
// tcgen05.mma.cta_group::2.kind::tf32 (M = 256, N = 256, K = 8, two MMAs per
// K step), the accumulators in TMEM (each CTA: its 128 rows x 512 columns).
// Per 32-row stage of A, each CTA's 16 generator warps write its 128 x 32
// tile of S (the Gaussian entry definition of rng.cuh: gaussian_quad_f64,
// evaluated in fast fp32) straight into shared memory in the MN-major
// SWIZZLE_128B_BASE32B operand layout (one Philox call = four sketch rows =
// one 16-byte chunk),
// its TMA warp loads its half of the A tile (CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B),
// and the even CTA's MMA thread issues the MMAs and commits to both CTAs'
// ring barriers (4-stage ring, 48 KB per stage).  The epilogue warps drain
// TMEM with tcgen05.ld.  Split-K partial tiles are summed in slice order by
// a second kernel (deterministic).
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "pcg64.cuh"
#include "umma.cuh"

namespace adask {

namespace {

constexpr int BM = 128;  // sketch rows per CTA (TMEM lanes); a CTA pair covers 256
#ifndef ADASK_TC_BK
#define ADASK_TC_BK 32
#endif
constexpr int BK = ADASK_TC_BK;  // rows of A per pipeline stage
constexpr int NGEN = 16;  // generator / epilogue warps (one stage row each per pass)
constexpr int KQ = BK / NGEN;  // Philox calls per generator thread per stage
constexpr int THREADS = 64 + 32 * NGEN;

// Per CTA of the pair: NH MMAs of N = 256 per K step; this CTA holds 128 of
// each MMA's 256 columns (the peer holds the other 128).
template <int NH>
struct TcCfg {
  static constexpr int BN = 256 * NH;          // columns per pair tile (TMEM columns per CTA)
  static constexpr int BOXES = 4 * NH;         // 32-column TMA boxes this CTA loads per stage
  static constexpr int S_BYTES = BM * BK * 4;       // this CTA's 128 sketch rows
  static constexpr int B_BYTES = BOXES * BK * 128;  // this CTA's half of the A tile
  static constexpr int STAGE_BYTES = S_BYTES + B_BYTES;
  static constexpr int STAGES = (200 * 1024) / STAGE_BYTES < 12 ? (200 * 1024) / STAGE_BYTES : 12;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;
  static constexpr uint32_t TMEM_COLS = BN;
};

__device__ __forceinline__ float sqrt_approx(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float lg2_approx(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float unit23(uint32_t w) {  // (w >> 9) * 2^-23, exact
  return __uint_as_float(0x3F800000u | (w >> 9)) - 1.0f;
}

// gaussian_quad_f64 (rng.cuh) in fast fp32 for NQ counters at once (the
// rounds are interleaved so the NQ dependency chains overlap): Philox4x32-10
// with precomputed round keys, Box-Muller on MUFU lg2 / sqrt / sin / cos.
// cos(2 pi u) is evaluated as -cos(2 pi (u - 1/2)) to keep the MUFU argument
// in [-pi, pi).
template <int NQ>
__device__ __forceinline__ void gaussian_quads_fast(const uint64_t* i, uint32_t g, const uint32_t* rk0,
                                                    const uint32_t* rk1, float4* out) {
  uint32_t x[NQ], y[NQ], z[NQ], w[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    x[q] = (uint32_t)i[q];
    y[q] = (uint32_t)(i[q] >> 32);
    z[q] = g;
    w[q] = 0u;
  }
#pragma unroll
  for (int r = 0; r < 10; ++r)
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const uint64_t p0 = (uint64_t)0xD2511F53u * x[q], p1 = (uint64_t)0xCD9E8D57u * z[q];
      x[q] = (uint32_t)(p1 >> 32) ^ y[q] ^ rk0[r];
      y[q] = (uint32_t)p1;
      z[q] = (uint32_t)(p0 >> 32) ^ w[q] ^ rk1[r];
      w[q] = (uint32_t)p0;
    }
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const float ra = sqrt_approx(-1.3862943611198906f * lg2_approx(1.0f - unit23(x[q])));
    const float rc = sqrt_approx(-1.3862943611198906f * lg2_approx(1.0f - unit23(z[q])));
    float sa, ca, sc, cc;
    __sincosf(6.2831853071795865f * (unit23(y[q]) - 0.5f), &sa, &ca);
    __sincosf(6.2831853071795865f * (unit23(w[q]) - 0.5f), &sc, &cc);
    out[q] = make_float4(-ra * ca, -ra * sa, -rc * cc, -rc * sc);
  }
}

// mbarrier wait that traps (instead of hanging the GPU) after ~10 s
__device__ __forceinline__ void wait_or_trap(uint64_t* bar, uint32_t parity, int tag) {
  const uint32_t a = smem_u32(bar);
  uint32_t ok = 0;
  long long t0 = 0;
  for (uint32_t spin = 0;; ++spin) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
    if (ok) return;
    if ((spin & 1023) == 0) {
      const long long t = clock64();
      if (spin == 0)
        t0 = t;
      else if (t - t0 > 20000000000ll) {
        printf("k_gauss_tc: block %d thread %d stuck on barrier tag %d parity %u\n", (int)blockIdx.x,
               (int)threadIdx.x, tag, parity);
        __trap();
      }
    }
  }
}
__device__ __forceinline__ void st_shared_v4(uint32_t addr, float4 v) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}

// One CTA pair (a 2-CTA cluster) computes a 256 x BN tile of SA over one
// split-K slice of the rows of A with tcgen05.mma.cta_group::2 (M = 256):
// CTA r holds sketch rows [128 r, 128 r + 128) of the tile (its S tile and
// its TMEM accumulator) and, of every MMA's 256 columns, the 128 starting
// at 128 r (its half of each A tile).  The even CTA issues the MMAs; both
// CTAs' TMA loads and S tiles complete the even CTA's ring barrier, and its
// commits release the ring slot in both CTAs.
template <int NH>
__global__ void __launch_bounds__(THREADS, 1)
    k_gauss_tc(const __grid_constant__ CUtensorMap amap, int64_t n_local, int64_t d, int64_t row0, int64_t m,
               uint32_t key0, uint32_t key1, float scale, int64_t k_per_slice, int m_pairs, int n_tiles,
               float* __restrict__ out, int64_t ldo, int64_t slice_stride, int vec_ok, int64_t kg0, int dbg) {
  using C = TcCfg<NH>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* done = empty + C::STAGES;
  uint32_t* tmem_slot = (uint32_t*)(done + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t cr = blockIdx.x & 1u;  // rank in the pair (1-D clusters of 2)
  int c = (int)(blockIdx.x >> 1);
  const int mp = c % m_pairs;
  c /= m_pairs;
  const int nt = c % n_tiles;
  const int slice = c / n_tiles;
  const int64_t m0 = (int64_t)mp * (2 * BM) + (int64_t)cr * BM, n0 = (int64_t)nt * C::BN;
  const int64_t kb = (int64_t)slice * k_per_slice;
  const int64_t ke = kb + k_per_slice < n_local ? kb + k_per_slice : n_local;
  const int nk = (int)((ke - kb + BK - 1) / BK);

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 3);  // even CTA's producer (expect_tx) + both generator groups
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    fence_barrier_init();
  }
  if (warp == 1) umma::tmem_alloc_pair(tmem_slot, C::TMEM_COLS);
  umma::fence_before_sync();
  __syncthreads();
  umma::cluster_sync();
  umma::fence_after_sync();
  const uint32_t tbase = *tmem_slot;
  const uint32_t full_lead = umma::mapa(smem_u32(full), 0u);  // the even CTA's ring barriers
  const bool trace = (dbg & 128) != 0 && blockIdx.x < 2;   // per-role cycle accounting
  long long tr0 = 0, tr1 = 0;
  const long long t_start = clock64();

  if (warp == 0) {
    // ---------------------------------------------------------- TMA producer
    if (lane == 0) {
      umma::tma_prefetch_map(&amap);
      const int pf = (dbg >> 8) & 63;  // experimental: L2 prefetch distance in stages
      for (int it = 0; it < nk; ++it) {
        const int s = it % C::STAGES;
        const uint32_t ph = (uint32_t)(it / C::STAGES) & 1u;
        const long long tw = trace ? clock64() : 0;
        wait_or_trap(&empty[s], ph ^ 1u, 1);
        if (trace) tr0 += clock64() - tw;
        uint8_t* bst = smem + s * C::STAGE_BYTES + C::S_BYTES;
        const uint32_t bar = full_lead + (uint32_t)(s * 8);
        if (cr == 0) mbar_arrive_expect_tx(&full[s], (dbg & 8) ? 0u : 2u * C::B_BYTES);
        if (dbg & 8) continue;  // timing probe: no A traffic
        const int32_t krow = (int32_t)(kb + (int64_t)it * BK);
        if (pf > 0 && it + pf < nk) {  // warm L2 for the stage pf ahead
#pragma unroll
          for (int h = 0; h < NH; ++h)
#pragma unroll
            for (int j = 0; j < 4; ++j)
              umma::tma_prefetch_2d(&amap, (int32_t)(n0 + 256 * h + 128 * (int)cr + 32 * j), krow + pf * BK);
        }
#pragma unroll
        for (int h = 0; h < NH; ++h)
#pragma unroll
          for (int j = 0; j < 4; ++j)
            umma::tma_load_2d_pair(bst + (h * 4 + j) * (BK * 128), &amap,
                                   (int32_t)(n0 + 256 * h + 128 * (int)cr + 32 * j), krow, bar);
      }
      if (trace) out[16 * blockIdx.x + 0] = (float)tr0;
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------- MMA issuer (even CTA)
    if (cr == 0 && lane == 0) {
      constexpr uint32_t idesc = umma::idesc_tf32(2 * BM, 256, true, true);
      for (int it = 0; it < nk; ++it) {
        const int s = it % C::STAGES;
        const uint32_t ph = (uint32_t)(it / C::STAGES) & 1u;
        const long long tw = trace ? clock64() : 0;
        wait_or_trap(&full[s], ph, 2);
        if (trace) tr0 += clock64() - tw;
        umma::fence_after_sync();
        const uint32_t sa = smem_u32(smem + s * C::STAGE_BYTES);
        const uint32_t sb = sa + C::S_BYTES;
#pragma unroll
        for (int ks = 0; ks < BK / 8; ++ks) {
          const uint64_t ad = umma::sdesc(sa + ks * 1024, BK * 128, 512, umma::LAYOUT_SW128_BASE32B);
#pragma unroll
          for (int h = 0; h < NH; ++h) {
            const uint64_t bd =
                umma::sdesc(sb + h * 4 * (BK * 128) + ks * 1024, BK * 128, 512, umma::LAYOUT_SW128_BASE32B);
            umma::mma_tf32_pair(tbase + h * 256, ad, bd, idesc, (uint32_t)(it | ks));
          }
        }
        umma::mma_commit_pair_mc(&empty[s], 0x3);  // the slot is free in both CTAs
      }
      umma::mma_commit_pair_mc(done, 0x3);
      if (trace) out[16 * blockIdx.x + 1] = (float)tr0;
    }
    __syncwarp();
  } else {
    // ---------------------------------------------------------- S generators
    const int gt = threadIdx.x - 64;  // 0 .. 32 NGEN - 1
    const int rg = gt & 31;           // tile rows 4rg .. 4rg+3
    const int kk0 = gt >> 5;          // stage rows kk0 + NGEN q, q < KQ
    const uint32_t grp = (uint32_t)(((kg0 + m0) >> 2) + rg);  // global sketch-row group
    uint32_t rk0[10], rk1[10];
#pragma unroll
    for (int r = 0; r < 10; ++r) {
      rk0[r] = key0 + (uint32_t)r * 0x9E3779B9u;
      rk1[r] = key1 + (uint32_t)r * 0xBB67AE85u;
    }
    // MN-major SW128_BASE32B: MN group (rg >> 3) at BK*128 bytes, K row kk at
    // 128 B, 32-byte chunk ((rg >> 1) & 3) XOR (kk & 3), 16-byte half rg & 1
    const uint32_t soff = (uint32_t)((rg >> 3) * (BK * 128) + kk0 * 128 + ((((rg >> 1) & 3) ^ (kk0 & 3)) << 5) +
                                     ((rg & 1) << 4));
    const uint64_t gi0 = (uint64_t)(row0 + kb + kk0);
    // GU stages per trip: GU x KQ independent Philox / Box-Muller chains
    constexpr int GU = KQ >= 2 ? 1 : 2;
    for (int it0 = 0; it0 < nk; it0 += GU) {
      float4 z[GU][KQ];
      uint64_t gi[GU * KQ];
#pragma unroll
      for (int u = 0; u < GU; ++u)
#pragma unroll
        for (int q = 0; q < KQ; ++q) gi[u * KQ + q] = gi0 + (uint64_t)(it0 + u) * BK + NGEN * q;
      if (dbg & 4) {  // timing probe: no generation
#pragma unroll
        for (int u = 0; u < GU; ++u)
#pragma unroll
          for (int q = 0; q < KQ; ++q) z[u][q] = make_float4(0.f, 0.f, 0.f, 0.f);
      } else if (dbg == 1) {  // S[r, k] = [r == k mod 128] (layout debugging)
#pragma unroll
        for (int u = 0; u < GU; ++u)
#pragma unroll
          for (int q = 0; q < KQ; ++q) {
            const int kl = (int)((gi[u * KQ + q] - (uint64_t)row0) & 127);
            z[u][q] = make_float4(4 * rg == kl, 4 * rg + 1 == kl, 4 * rg + 2 == kl, 4 * rg + 3 == kl);
          }
      } else {
        gaussian_quads_fast<GU * KQ>(gi, grp, rk0, rk1, &z[0][0]);
      }
#pragma unroll
      for (int u = 0; u < GU; ++u) {
        const int it = it0 + u;
        if (it >= nk) break;
        const int s = it % C::STAGES;
        const uint32_t ph = (uint32_t)(it / C::STAGES) & 1u;
        const long long tw = trace ? clock64() : 0;
        wait_or_trap(&empty[s], ph ^ 1u, 3);
        if (trace) tr0 += clock64() - tw;
        const uint32_t sdst = smem_u32(smem + s * C::STAGE_BYTES) + soff;
#pragma unroll
        for (int q = 0; q < KQ; ++q) st_shared_v4(sdst + NGEN * 128 * q, z[u][q]);
        umma::fence_proxy_async_smem();
        const long long tb = trace ? clock64() : 0;
        named_bar_sync(1, 32 * NGEN);
        if (trace) tr1 += clock64() - tb;
        if (gt == 0) {
          if (cr == 0)
            mbar_arrive(&full[s]);
          else
            umma::mbar_arrive_remote(full_lead + (uint32_t)(s * 8));
        }
      }
    }
    // ---------------------------------------------------------- epilogue
    const long long tw = trace ? clock64() : 0;
    wait_or_trap(done, 0, 4);
    if (trace && gt == 0) {
      out[16 * blockIdx.x + 2] = (float)tr0;
      out[16 * blockIdx.x + 3] = (float)tr1;
      out[16 * blockIdx.x + 4] = (float)(tw - t_start);
      out[16 * blockIdx.x + 5] = (float)(clock64() - t_start);
      out[16 * blockIdx.x + 6] = (float)nk;
    }
    umma::fence_after_sync();
    const int q = warp & 3;            // TMEM lane quarter this warp may read
    const int half = (warp - 2) >> 2;  // column part
    constexpr int CW = C::BN / (NGEN / 4);
    const int64_t row = m0 + 32 * q + lane;
    float* orow = out + (int64_t)slice * slice_stride + row * ldo + n0;
#pragma unroll 1
    for (int cc = 0; cc < CW; cc += 16) {
      const int col = half * CW + cc;
      float v[16];
      umma::tmem_ld16(tbase + ((uint32_t)(32 * q) << 16) + (uint32_t)col, v);
      if (row < m && n0 + col < d && dbg != 2 && !(dbg & 128)) {
        if (vec_ok && n0 + col + 16 <= d) {
#pragma unroll
          for (int j = 0; j < 16; j += 4)
            *(float4*)(orow + col + j) =
                make_float4(v[j] * scale, v[j + 1] * scale, v[j + 2] * scale, v[j + 3] * scale);
        } else {
          for (int j = 0; j < 16 && n0 + col + j < d; ++j) orow[col + j] = v[j] * scale;
        }
      }
    }
  }
  umma::fence_before_sync();
  __syncthreads();
  umma::cluster_sync();  // no CTA leaves while its peer may still signal it or read its smem
  if (warp == 1) {
    umma::fence_after_sync();
    umma::tmem_dealloc_pair(tbase, C::TMEM_COLS);
  }
}

// SA (+)= sum over slices of the partial tiles, in slice order.
__global__ void k_slice_sum(const float* __restrict__ P, int slices, int64_t slice_stride, int64_t m,
                            int64_t d, float* __restrict__ SA, int64_t ldsa, int accumulate) {
  const int64_t total = m * d;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / d, c = e - r * d;
    float acc = accumulate ? SA[r * ldsa + c] : 0.0f;
    for (int s = 0; s < slices; ++s) acc += P[(int64_t)s * slice_stride + e];
    SA[r * ldsa + c] = acc;
  }
}

template <int NH>
int launch_tc(adask_ctx* ctx, const CUtensorMap& map, int64_t n_local, int64_t d, int64_t row0, int64_t m,
              uint64_t key, int64_t k_per_slice, int m_pairs, int n_tiles, int slices, float* out, int64_t ldo,
              int64_t slice_stride, int64_t kg0, int64_t m_total, cudaStream_t st) {
  using C = TcCfg<NH>;
  static bool attr = false;
  if (!attr) {
    ADASK_TRY(ensure_smem_attr((const void*)k_gauss_tc<NH>, C::SMEM));
    attr = true;
  }
  const float scale = (float)(1.0 / sqrt((double)m_total));
  const int vec_ok = (ldo % 4 == 0) && (((uintptr_t)out & 15) == 0);
  const int dbg = getenv("ADASK_TC_DEBUG") ? atoi(getenv("ADASK_TC_DEBUG")) : 0;
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3((unsigned)(2ll * m_pairs * n_tiles * slices));
  lc.blockDim = dim3(THREADS);
  lc.dynamicSmemBytes = C::SMEM;
  lc.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  ADASK_CUDA(cudaLaunchKernelEx(&lc, k_gauss_tc<NH>, map, n_local, d, row0, m, (uint32_t)key, (uint32_t)(key >> 32),
                                scale, k_per_slice, m_pairs, n_tiles, out, ldo, slice_stride, vec_ok, kg0, dbg));
  ADASK_LAUNCHED(ctx);
  return ADASK_OK;
}

}  // namespace

// Rows [kg0, kg0 + m) of the m_total-row sketch (kg0 a multiple of 4).
int gauss_tc_impl(adask_ctx* ctx, const float* A, int64_t n_local, int64_t d, int64_t lda, int64_t row0,
                  int64_t m, uint64_t key, float* SA, int64_t ldsa, bool accumulate, cudaStream_t st, int64_t kg0,
                  int64_t m_total) {
  if (kg0 % 4 != 0) return fail(ADASK_E_ARG, "TF32 Gaussian sketch: row offset must be a multiple of 4");
  if (n_local == 0) {
    if (!accumulate) ADASK_CUDA(cudaMemset2DAsync(SA, ldsa * 4, 0, d * 4, m, st));
    return ADASK_OK;
  }
  if (lda % 4 != 0 || ((uintptr_t)A & 15) != 0)
    return fail(ADASK_E_ARG, "TF32 Gaussian sketch: rows of A must be 16-byte aligned (lda %% 4 == 0)");
  if (n_local >= (1ll << 31) || d >= (1ll << 31))
    return fail(ADASK_E_ARG, "TF32 Gaussian sketch: A too large for one tensor map");
  const int NH = d > 256 ? 2 : 1;
  const int BN = 256 * NH;
  const int m_pairs = (int)cdiv(m, 2 * BM), n_tiles = (int)cdiv(d, BN);
  const int64_t pairs = (int64_t)m_pairs * n_tiles;
  const int64_t nk_total = cdiv(n_local, BK);
  // split-K: minimise waves x (stages per slice + prologue/epilogue cost),
  // 74 pairs (148 SMs) per wave
  int best = 1;
  double best_cost = 1e300;
  for (int s = 1; s <= 64 && s <= nk_total; ++s) {
    const int64_t waves = cdiv(pairs * s, (int64_t)(kNumSMs / 2));
    const double cost = (double)waves * ((double)cdiv(nk_total, s) + 24.0);
    if (cost < best_cost * 0.999) {
      best_cost = cost;
      best = s;
    }
  }
  const int64_t k_per_slice = cdiv(nk_total, best) * BK;
  const int slices = (int)cdiv(n_local, k_per_slice);
  CUtensorMap map;
  ADASK_TRY(tensor_map_f32_sw128(&map, A, n_local, d, lda, 32, BK, true));
  float* out = SA;
  int64_t ldo = ldsa, slice_stride = 0;
  if (slices > 1 || accumulate) {
    void* wsp = nullptr;
    ADASK_TRY(ctx->ws[WS_GAUSS].get((size_t)slices * m * d * 4, st, &wsp));
    out = (float*)wsp;
    ldo = d;
    slice_stride = m * d;
  }
  if (NH == 2)
    ADASK_TRY(launch_tc<2>(ctx, map, n_local, d, row0, m, key, k_per_slice, m_pairs, n_tiles, slices, out, ldo,
                           slice_stride, kg0, m_total, st));
  else
    ADASK_TRY(launch_tc<1>(ctx, map, n_local, d, row0, m, key, k_per_slice, m_pairs, n_tiles, slices, out, ldo,
                           slice_stride, kg0, m_total, st));
  if (out != SA) {
    const int64_t total = m * d;
    const int blocks = (int)std::min<int64_t>(cdiv(total, 256), 4 * kNumSMs);
    k_slice_sum<<<blocks, 256, 0, st>>>(out, slices, slice_stride, m, d, SA, ldsa, accumulate ? 1 : 0);
    ADASK_LAUNCHED(ctx);
  }
  return ADASK_OK;
}

}  // namespace adask
