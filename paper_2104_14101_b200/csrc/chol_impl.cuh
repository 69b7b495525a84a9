// Tile-size-generic body of the cooperative Cholesky kernel (included by
// chol.cu inside namespaces chol64 / chol32 with NB defined).
constexpr int NBP = NB + 1;  // padded SMEM row pitch (doubles)
constexpr int kCholThreads = 256;

struct CholArgs {
  void* M;    // kp x kp, lower = input; reused as scratch
  void* L;    // kp x kp output (upper pre-zeroed)
  void* Li;   // kp x kp output L^-1 (upper pre-zeroed)
  void* LiT;  // kp x kp output L^-T (lower pre-zeroed)
  int kp, nblk, k;
  int* info;
  unsigned long long* tlog;  // optional phase timestamps (ADASK_CHOL_TRACE)
  int slow_diag;             // 1: unblocked pivot loop (ADASK_CHOL_SLOWDIAG, comparison)
  int fused_inv;             // 1: L^-1 by rows inside the factorization's phases
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define TMARK(idx)                                                   \
  do {                                                               \
    if (a.tlog && blockIdx.x == 0 && threadIdx.x == 0) a.tlog[idx] = gtimer(); \
  } while (0)

// 64 x 64 tile <-> SMEM (fp64), 16-byte vector accesses, all loads in flight.
template <typename T>
__device__ __forceinline__ void tile_load(double (*s)[NBP], const T* base, int ld, int bi, int bj) {
  const T* p = base + (int64_t)bi * NB * ld + (int64_t)bj * NB;
  constexpr int V = 16 / sizeof(T);            // elements per vector
  constexpr int PER = NB * NB / V / kCholThreads;  // vectors per thread
  using VT = typename std::conditional<sizeof(T) == 8, double2, float4>::type;
  VT v[PER];
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int idx = threadIdx.x + kCholThreads * q;
    const int r = idx / (NB / V), c = (idx % (NB / V)) * V;
    v[q] = *reinterpret_cast<const VT*>(p + (int64_t)r * ld + c);
  }
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int idx = threadIdx.x + kCholThreads * q;
    const int r = idx / (NB / V), c = (idx % (NB / V)) * V;
    const T* e = reinterpret_cast<const T*>(&v[q]);
#pragma unroll
    for (int u = 0; u < V; ++u) s[r][c + u] = (double)e[u];
  }
}

// Split tile load: global -> registers (fetch, issued early) and registers ->
// SMEM (put), so the next tile's loads overlap the current tile product.
template <typename T>
struct TileRegs {
  using VT = typename std::conditional<sizeof(T) == 8, double2, float4>::type;
  static constexpr int V = 16 / sizeof(T);
  static constexpr int PER = NB * NB / V / kCholThreads;
  VT v[PER];
};
template <typename T>
__device__ __forceinline__ void tile_fetch(TileRegs<T>& R, const T* base, int ld, int bi, int bj) {
  using X = TileRegs<T>;
  const T* p = base + (int64_t)bi * NB * ld + (int64_t)bj * NB;
#pragma unroll
  for (int q = 0; q < X::PER; ++q) {
    const int idx = threadIdx.x + kCholThreads * q;
    const int r = idx / (NB / X::V), c = (idx % (NB / X::V)) * X::V;
    R.v[q] = *reinterpret_cast<const typename X::VT*>(p + (int64_t)r * ld + c);
  }
}
template <typename T>
__device__ __forceinline__ void tile_put(double (*s)[NBP], const TileRegs<T>& R) {
  using X = TileRegs<T>;
#pragma unroll
  for (int q = 0; q < X::PER; ++q) {
    const int idx = threadIdx.x + kCholThreads * q;
    const int r = idx / (NB / X::V), c = (idx % (NB / X::V)) * X::V;
    const T* e = reinterpret_cast<const T*>(&R.v[q]);
#pragma unroll
    for (int u = 0; u < X::V; ++u) s[r][c + u] = (double)e[u];
  }
}

template <typename T>
__device__ __forceinline__ void tile_store(T* base, int ld, int bi, int bj, const double (*s)[NBP],
                                           bool transpose = false, int lower_only = 0) {
  T* p = base + (int64_t)bi * NB * ld + (int64_t)bj * NB;
  constexpr int V = 16 / sizeof(T);
  constexpr int PER = NB * NB / V / kCholThreads;
  using VT = typename std::conditional<sizeof(T) == 8, double2, float4>::type;
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int idx = threadIdx.x + kCholThreads * q;
    const int r = idx / (NB / V), c = (idx % (NB / V)) * V;
    VT v;
    T* e = reinterpret_cast<T*>(&v);
#pragma unroll
    for (int u = 0; u < V; ++u) {
      double x = transpose ? s[c + u][r] : s[r][c + u];
      if (lower_only == 1 && c + u > r) x = 0.0;  // lower triangle of the tile
      if (lower_only == 2 && c + u < r) x = 0.0;  // upper triangle of the tile
      e[u] = (T)x;
    }
    *reinterpret_cast<VT*>(p + (int64_t)r * ld + c) = v;
  }
}

// acc[a][b] += sum_k A[r_a][k] * (TB ? B[c_b][k] : B[k][c_b]),
// r_a = tr + 16a, c_b = tc + 16b.
constexpr int TM = NB / 16;  // per-thread micro-tile edge (16 x 16 thread grid)

template <bool TB>
__device__ __forceinline__ void tile_mma(const double (*A)[NBP], const double (*B)[NBP],
                                         double acc[TM][TM]) {
  const int tr = threadIdx.x >> 4, tc = threadIdx.x & 15;
#pragma unroll 8
  for (int k = 0; k < NB; ++k) {
    double a[TM], b[TM];
#pragma unroll
    for (int i = 0; i < TM; ++i) a[i] = A[tr + 16 * i][k];
#pragma unroll
    for (int j = 0; j < TM; ++j) b[j] = TB ? B[tc + 16 * j][k] : B[k][tc + 16 * j];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TM; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
  }
}

__device__ __forceinline__ void acc_to_tile(double (*C)[NBP], const double acc[TM][TM], double scale) {
  const int tr = threadIdx.x >> 4, tc = threadIdx.x & 15;
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TM; ++j) C[tr + 16 * i][tc + 16 * j] = scale * acc[i][j];
}

__device__ __forceinline__ void acc_zero(double acc[TM][TM]) {
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TM; ++j) acc[i][j] = 0.0;
}

__device__ __forceinline__ unsigned long long gtimer2() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Lower-triangle enumeration ordered by decreasing column: the trailing
// triangle {j < l <= i < 64} of pivot step j is the prefix of length
// (63 - j)(64 - j) / 2.  Entry = i | l << 8.
__device__ void build_tri_table(unsigned short* tab) {
  for (int e = threadIdx.x; e < NB * (NB - 1) / 2; e += blockDim.x) {
    // invert the prefix sums: column l holds 64 - l entries
    int l = NB - 1, base = 0;
    while (e >= base + (NB - l)) {
      base += NB - l;
      --l;
    }
    const int i = l + (e - base);
    tab[e] = (unsigned short)(i | (l << 8));
  }
}

// Factor the 64 x 64 tile in S (lower triangle read) in place -- L, strict
// upper zeroed -- and write X = L^-1.  Compact, rolled loops throughout: this
// runs once per panel, so straight-line unrolled code would stream through a
// cold instruction cache.  Factor: one pivot per step, the live trailing
// triangle spread evenly over the CTA via the precomputed table.  Inverse:
// warp w owns columns 8w..8w+7, lanes own rows lane and lane+32, finalized
// rows broadcast by shuffles (no block barrier inside the loop).
__device__ void diag_factor(double (*S)[NBP], double (*X)[NBP], const unsigned short* tab, int* info,
                            int goff, int kvalid, unsigned long long* tl = nullptr, int slow = 0) {
  __shared__ double rinv[NB];
  if (tl && threadIdx.x == 0) tl[0] = gtimer2();
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  if constexpr (NB == 32) {
    // Blocked pivot loop (same floating-point operations in the same order as
    // the unblocked loop below, so the factor is bitwise the same): four panels
    // of 8 pivots.  Warp 0 factors the 32 - jb rows of a panel in registers
    // (lane = row; multipliers broadcast by shuffles, no block barrier per
    // pivot); the whole CTA then applies the panel's 8 rank-1 updates to the
    // trailing triangle, pivot by pivot for every element.
    if (!slow) {
#ifndef ADASK_CHOL_PW
#define ADASK_CHOL_PW 8
#endif
      constexpr int PW = ADASK_CHOL_PW;  // panel width (pivots per warp-register panel)
#pragma unroll 1
      for (int jb = 0; jb < NB; jb += PW) {
        if (warp == 0) {
          const unsigned FULL = 0xffffffffu;
          const int i = jb + lane;
          double r[PW];
#pragma unroll
          for (int q = 0; q < PW; ++q) r[q] = i < NB ? S[i][jb + q] : 0.0;
#pragma unroll
          for (int p = 0; p < PW; ++p) {
            const double pj = __shfl_sync(FULL, r[p], p);
            const double rd = rsqrt(pj);
            if (lane == 0) {
              if ((!(pj > 0.0) || !isfinite(pj)) && goff + jb + p < kvalid) atomicCAS(info, 0, goff + jb + p + 1);
              rinv[jb + p] = rd;
            }
            const double l = lane > p ? r[p] * rd : (lane == p ? pj * rd : r[p]);
            r[p] = l;
#pragma unroll
            for (int q = p + 1; q < PW; ++q) {
              const double lq = __shfl_sync(FULL, l, q);
              if (lane >= q) r[q] = fma(-l, lq, r[q]);
            }
          }
          if (i < NB) {
#pragma unroll
            for (int q = 0; q < PW; ++q) S[i][jb + q] = r[q];
          }
        }
        __syncthreads();
        const int base = jb + PW;
        // 16 x 16 thread grid over the trailing triangle (no integer division)
        for (int ii = base + (t >> 4); ii < NB; ii += 16)
          for (int ll = base + (t & 15); ll <= ii; ll += 16) {
            double v = S[ii][ll];
#pragma unroll
            for (int p = 0; p < PW; ++p) v = fma(-S[ii][jb + p], S[ll][jb + p], v);
            S[ii][ll] = v;
          }
        __syncthreads();
      }
    }
  }
#pragma unroll 1
  for (int j = 0; j < (NB == 32 && !slow ? 0 : NB); ++j) {
    const double pj = S[j][j];
    const double rd = rsqrt(pj);
    if (t > j && t < NB) S[t][j] *= rd;
    if (t == 0) {
      if ((!(pj > 0.0) || !isfinite(pj)) && goff + j < kvalid) atomicCAS(info, 0, goff + j + 1);
      rinv[j] = rd;
    }
    __syncthreads();
    if (t == 0) S[j][j] = pj * rd;
    const int T = (NB - 1 - j) * (NB - j) / 2;
#pragma unroll 1
    for (int e = t; e < T; e += kCholThreads) {
      const int il = tab[e], i = il & 0xff, l = il >> 8;
      S[i][l] = fma(-S[i][j], S[l][j], S[i][l]);
    }
    __syncthreads();
  }
  if (tl && threadIdx.x == 0) tl[1] = gtimer2();
  for (int e = t; e < NB * NB; e += blockDim.x) {
    const int i = e / NB, j = e % NB;
    if (j > i) S[i][j] = 0.0;
  }
  __syncthreads();
  if constexpr (NB == 32) {
    if (!slow) {
      // X = L^-1 by 2 x 2 blocks of 16: the two diagonal blocks are inverted
      // concurrently (warps 0-3 and 4-7, row-sequential as below but 16 steps),
      // then X21 = -X22 (L21 X11) with two 16 x 16 x 16 products (X12 = 0 is
      // the scratch for L21 X11)
      const int half = warp >> 2, o = 16 * half, cw = o + (warp & 3) * 4;
      double acc[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[q] = (o + lane == cw + q) ? 1.0 : 0.0;
#pragma unroll 1
      for (int i = 0; i < 16; ++i) {
        const double ri = rinv[o + i];
        double xi[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const double v = __shfl_sync(0xffffffffu, acc[q], i);
          xi[q] = (cw + q <= o + i) ? v * ri : 0.0;
        }
        if (lane == i) {
#pragma unroll
          for (int q = 0; q < 4; ++q) acc[q] = xi[q];
        }
        const double lri = (lane > i && lane < 16) ? S[o + lane][o + i] : 0.0;
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[q] = fma(-lri, xi[q], acc[q]);
      }
      if (lane < 16) {
#pragma unroll
        for (int q = 0; q < 4; ++q) X[o + lane][cw + q] = acc[q];
      }
      __syncthreads();
      const int rr = t >> 4, cc = t & 15;
      double sum = 0.0;
#pragma unroll
      for (int k = 0; k < 16; ++k) sum = fma(S[16 + rr][k], X[k][cc], sum);
      X[rr][16 + cc] = sum;  // (L21 X11)[rr][cc]
      __syncthreads();
      double u = 0.0;
#pragma unroll
      for (int k = 0; k < 16; ++k) u = fma(X[16 + rr][16 + k], X[k][16 + cc], u);
      __syncthreads();
      X[16 + rr][cc] = -u;
      X[rr][16 + cc] = 0.0;
      __syncthreads();
      if (tl && threadIdx.x == 0) tl[2] = gtimer2();
      return;
    }
  }
  constexpr int CPW = NB / 8;  // columns per warp
  constexpr int RPL = NB / 32; // rows per lane
  double acc[RPL][CPW];
  const int c0 = warp * CPW;
#pragma unroll
  for (int h = 0; h < RPL; ++h)
#pragma unroll
    for (int q = 0; q < CPW; ++q) acc[h][q] = (lane + 32 * h == c0 + q) ? 1.0 : 0.0;
#pragma unroll 1
  for (int i = 0; i < NB; ++i) {
    const int owner = i & 31, hi = i >> 5;
    const double ri = rinv[i];
    double xi[CPW];
#pragma unroll
    for (int q = 0; q < CPW; ++q) {
      double v = (RPL > 1 && hi) ? acc[RPL - 1][q] : acc[0][q];
      v = __shfl_sync(0xffffffffu, v, owner);
      xi[q] = (c0 + q <= i) ? v * ri : 0.0;
    }
    if (lane == owner) {
#pragma unroll
      for (int q = 0; q < CPW; ++q) {
        if (RPL > 1 && hi) acc[RPL - 1][q] = xi[q];
        else acc[0][q] = xi[q];
      }
    }
#pragma unroll
    for (int h = 0; h < RPL; ++h) {
      const int r = lane + 32 * h;
      const double lri = r > i ? S[r][i] : 0.0;
#pragma unroll
      for (int q = 0; q < CPW; ++q) acc[h][q] = fma(-lri, xi[q], acc[h][q]);
    }
  }
#pragma unroll
  for (int h = 0; h < RPL; ++h)
#pragma unroll
    for (int q = 0; q < CPW; ++q) X[lane + 32 * h][c0 + q] = acc[h][q];
  __syncthreads();
  if (tl && threadIdx.x == 0) tl[2] = gtimer2();
}

// Fused inverse (a.fused_inv), X = L^-1 by block rows, interleaved with the
// factorization's phases so it runs on the CTAs the shrinking trailing update
// leaves idle:
//   row s:     X_sl = -Dinv_s T_sl (l < s),  X_ss = Dinv_s (stored at factor time)
//   update p:  T_il = sum_{q=l}^{p} L_iq X_ql for i > p, l <= p  (one term per step)
// T lives in M's strictly-lower tiles left of the active panel (A_il is dead
// once its trsm ran).  Update p runs in the trsm phase of panel p+1 (L_{*,p}
// and row p of X are final), row s in the syrk phase of panel s (T_sl has all
// its terms); X is written to Li and, transposed, to LiT.
// Work items continue the phase's round-robin after `skip` items (CTA b takes
// item u when u = b (mod G)); skip < 0: all CTAs, from item 0.
template <typename T>
__device__ __forceinline__ void inv_update(const CholArgs& a, int p, int skip, double (*sA)[NBP], double (*sB)[NBP],
                                           double (*sC)[NBP], double (&acc)[TM][TM]) {
  const T* L = reinterpret_cast<const T*>(a.L);
  const T* Li = reinterpret_cast<const T*>(a.Li);
  T* M = reinterpret_cast<T*>(a.M);
  const int ld = a.kp, G = gridDim.x, b = blockIdx.x;
  const int nl = p + 1, nupd = (a.nblk - p - 1) * nl;
  int q = b - skip % G;
  if (q < 0) q += G;
  // software-pipelined: the next item's three tiles are in flight during
  // the current product
  TileRegs<T> ra, rb, rc;
  if (q < nupd) {
    const int i = p + 1 + q / nl, l = q % nl;
    tile_fetch<T>(ra, L, ld, i, p);
    tile_fetch<T>(rb, Li, ld, p, l);
    if (l < p) tile_fetch<T>(rc, M, ld, i, l);
  }
  for (; q < nupd; q += G) {
    const int i = p + 1 + q / nl, l = q % nl;
    tile_put<T>(sA, ra);
    tile_put<T>(sB, rb);
    if (l < p) tile_put<T>(sC, rc);
    __syncthreads();
    const int qn = q + G;
    if (qn < nupd) {
      const int in = p + 1 + qn / nl, ln = qn % nl;
      tile_fetch<T>(ra, L, ld, in, p);
      tile_fetch<T>(rb, Li, ld, p, ln);
      if (ln < p) tile_fetch<T>(rc, M, ld, in, ln);
    }
    acc_zero(acc);
    tile_mma<false>(sA, sB, acc);
    {
      const int tr = threadIdx.x >> 4, tc = threadIdx.x & 15;
#pragma unroll
      for (int x = 0; x < TM; ++x)
#pragma unroll
        for (int y = 0; y < TM; ++y) {
          double& c = sC[tr + 16 * x][tc + 16 * y];
          c = l < p ? c + acc[x][y] : acc[x][y];
        }
    }
    __syncthreads();
    tile_store<T>(M, ld, i, l, sC);
    __syncthreads();
  }
}

// Row s of X.  skip >= 0: the syrk phase's CTAs >= 1 (CTA 0 factors the next
// diagonal tile) continue their round-robin after `skip` tiles; skip < 0: all.
template <typename T>
__device__ __forceinline__ void inv_row(const CholArgs& a, int s, int skip, double (*sA)[NBP], double (*sB)[NBP],
                                        double (*sC)[NBP], double (&acc)[TM][TM]) {
  T* Li = reinterpret_cast<T*>(a.Li);
  T* LiT = reinterpret_cast<T*>(a.LiT);
  const T* M = reinterpret_cast<const T*>(a.M);
  const int ld = a.kp, b = blockIdx.x;
  int W = gridDim.x, me = b;
  if (skip >= 0 && W > 1) {
    if (b == 0) return;
    W -= 1;
    me = b - 1;
  } else if (skip < 0) {
    skip = 0;
  }
  int l = me - skip % W;
  if (l < 0) l += W;
  for (; l < s; l += W) {
    tile_load<T>(sA, Li, ld, s, s);
    tile_load<T>(sB, M, ld, s, l);
    __syncthreads();
    acc_zero(acc);
    tile_mma<false>(sA, sB, acc);
    acc_to_tile(sC, acc, -1.0);
    __syncthreads();
    tile_store<T>(Li, ld, s, l, sC);
    tile_store<T>(LiT, ld, l, s, sC, true, 0);
    __syncthreads();
  }
}

template <typename T>
__global__ void __launch_bounds__(kCholThreads, 1) k_chol_coop(CholArgs a) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double csm[];
  double(*sA)[NBP] = reinterpret_cast<double(*)[NBP]>(csm);
  double(*sB)[NBP] = reinterpret_cast<double(*)[NBP]>(csm + NB * NBP);
  double(*sC)[NBP] = reinterpret_cast<double(*)[NBP]>(csm + 2 * NB * NBP);
  double(*sD)[NBP] = reinterpret_cast<double(*)[NBP]>(csm + 3 * NB * NBP);  // second buffers of the
  double(*sE)[NBP] = reinterpret_cast<double(*)[NBP]>(csm + 4 * NB * NBP);  // pipelined inverse
  T* M = reinterpret_cast<T*>(a.M);
  T* L = reinterpret_cast<T*>(a.L);
  T* Li = reinterpret_cast<T*>(a.Li);
  T* LiT = reinterpret_cast<T*>(a.LiT);
  const int ld = a.kp, nblk = a.nblk;
  const int G = gridDim.x, b = blockIdx.x;
  double acc[TM][TM];
  __shared__ unsigned short tri_tab[NB * (NB - 1) / 2];
  build_tri_table(tri_tab);
  __syncthreads();
  TMARK(0);

  // prologue: diagonal block 0
  if (b == 0) {
    tile_load<T>(sA, M, ld, 0, 0);
    __syncthreads();
    TMARK(3 * nblk + 4);
    diag_factor(sA, sB, tri_tab, a.info, 0, a.k, a.tlog ? a.tlog + 3 * nblk + 8 : nullptr, a.slow_diag);
    TMARK(3 * nblk + 5);
    tile_store<T>(L, ld, 0, 0, sA, false, 1);
    tile_store<T>(Li, ld, 0, 0, sB, false, 1);
    if (a.fused_inv) tile_store<T>(LiT, ld, 0, 0, sB, true, 2);
    __syncthreads();
    TMARK(3 * nblk + 6);
  }
  grid.sync();
  TMARK(1);
  for (int j = 0; j + 1 < nblk; ++j) {
    // ---- trsm: L_ij = A_ij Dinv_j^T, i > j
    bool have = false;
    for (int i = j + 1 + b; i < nblk; i += G) {
      if (!have) {
        tile_load<T>(sB, Li, ld, j, j);
        have = true;
      }
      tile_load<T>(sA, M, ld, i, j);
      __syncthreads();
      acc_zero(acc);
      tile_mma<true>(sA, sB, acc);
      acc_to_tile(sC, acc, 1.0);
      __syncthreads();
      tile_store<T>(L, ld, i, j, sC);
      __syncthreads();
    }
    // fused inverse, update of step j-1 on the idle CTAs (after the trsm rows)
    if (a.fused_inv && j >= 1) inv_update<T>(a, j - 1, nblk - j - 1, sA, sB, sC, acc);
    grid.sync();
    TMARK(2 + 3 * j);
    // ---- syrk: A_il -= L_ij L_lj^T for j < l <= i.  CTA 0 owns the next
    // diagonal tile and factors it right away (lookahead); the other CTAs
    // share the remaining tiles.
    const int Tn = nblk - j - 1;
    const int ntiles = Tn * (Tn + 1) / 2;
    const int t_first = (G == 1 || b == 0) ? 0 : b;
    const int t_step = G == 1 ? 1 : (b == 0 ? ntiles : G - 1);
    for (int t = t_first; t < ntiles; t += t_step) {
      int ii = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
      while ((ii + 1) * (ii + 2) / 2 <= t) ++ii;
      while (ii * (ii + 1) / 2 > t) --ii;
      const int ll = t - ii * (ii + 1) / 2;
      const int i = j + 1 + ii, l = j + 1 + ll;
      tile_load<T>(sA, L, ld, i, j);
      tile_load<T>(sB, L, ld, l, j);
      tile_load<T>(sC, M, ld, i, l);
      __syncthreads();
      acc_zero(acc);
      tile_mma<true>(sA, sB, acc);
      {
        const int tr = threadIdx.x >> 4, tc = threadIdx.x & 15;
#pragma unroll
        for (int x = 0; x < TM; ++x)
#pragma unroll
          for (int y = 0; y < TM; ++y) sC[tr + 16 * x][tc + 16 * y] -= acc[x][y];
      }
      __syncthreads();
      if (t == 0) {
        // the updated diagonal tile j+1 is final: factor it now
        diag_factor(sC, sB, tri_tab, a.info, (j + 1) * NB, a.k, nullptr, a.slow_diag);
        tile_store<T>(L, ld, j + 1, j + 1, sC, false, 1);
        tile_store<T>(Li, ld, j + 1, j + 1, sB, false, 1);
        if (a.fused_inv) tile_store<T>(LiT, ld, j + 1, j + 1, sB, true, 2);
      } else {
        tile_store<T>(M, ld, i, l, sC);
      }
      __syncthreads();
    }
    // fused inverse, row j of L^-1 after the syrk tiles (CTAs >= 1)
    if (a.fused_inv && j >= 1) inv_row<T>(a, j, G == 1 ? 0 : ntiles - 1, sA, sB, sC, acc);
    grid.sync();
    TMARK(3 + 3 * j);
  }
  TMARK(3 * nblk + 1);
  if (a.fused_inv) {
    // the last block row: update of step nblk-2, then row nblk-1
    if (nblk >= 2) {
      inv_update<T>(a, nblk - 2, 0, sA, sB, sC, acc);
      grid.sync();
      inv_row<T>(a, nblk - 1, -1, sA, sB, sC, acc);
      grid.sync();
    }
    TMARK(3 * nblk + 2);
    TMARK(3 * nblk + 3);
    return;
  }

  // ---- inverse by recursive doubling: I21 = -I22 (L21 I11), scratch in M
  for (int s = 1; s < nblk; s <<= 1) {
    // step a: Tmp(i, l) = sum_{p=l}^{b0+s-1} L(i, p) Li(p, l),  i in 2-range, l in 1-range
    const int npairs = (nblk + 2 * s - 1) / (2 * s);
    int work = 0;
    for (int q = 0; q < npairs; ++q) {
      const int b0 = q * 2 * s, r2 = min(s, nblk - (b0 + s));
      if (r2 > 0) work += r2 * s;
    }
    for (int t = b; t < work; t += G) {
      int q = 0, tt = t, b0 = 0, r2 = 0;
      for (;; ++q) {
        b0 = q * 2 * s;
        r2 = min(s, nblk - (b0 + s));
        const int w = r2 > 0 ? r2 * s : 0;
        if (tt < w) break;
        tt -= w;
      }
      const int i = b0 + s + tt / s, l = b0 + tt % s;
      acc_zero(acc);
      {
        // double-buffered: the next (L, Li) tile pair is in flight during
        // the current product; one barrier per product
        TileRegs<T> ra, rb;
        tile_fetch<T>(ra, L, ld, i, l);
        tile_fetch<T>(rb, Li, ld, l, l);
        int cur = 0;
        for (int p = l; p < b0 + s; ++p) {
          tile_put<T>(cur ? sD : sA, ra);
          tile_put<T>(cur ? sE : sB, rb);
          __syncthreads();
          if (p + 1 < b0 + s) {
            tile_fetch<T>(ra, L, ld, i, p + 1);
            tile_fetch<T>(rb, Li, ld, p + 1, l);
          }
          tile_mma<false>(cur ? sD : sA, cur ? sE : sB, acc);
          cur ^= 1;
        }
        __syncthreads();
      }
      acc_to_tile(sC, acc, 1.0);
      __syncthreads();
      tile_store<T>(M, ld, i, l, sC);
      __syncthreads();
    }
    grid.sync();
    // step b: Li(i, l) = -sum_{p=b0+s}^{i} Li(i, p) Tmp(p, l)
    for (int t = b; t < work; t += G) {
      int q = 0, tt = t, b0 = 0, r2 = 0;
      for (;; ++q) {
        b0 = q * 2 * s;
        r2 = min(s, nblk - (b0 + s));
        const int w = r2 > 0 ? r2 * s : 0;
        if (tt < w) break;
        tt -= w;
      }
      const int i = b0 + s + tt / s, l = b0 + tt % s;
      acc_zero(acc);
      {
        TileRegs<T> ra, rb;
        tile_fetch<T>(ra, Li, ld, i, b0 + s);
        tile_fetch<T>(rb, M, ld, b0 + s, l);
        int cur = 0;
        for (int p = b0 + s; p <= i; ++p) {
          tile_put<T>(cur ? sD : sA, ra);
          tile_put<T>(cur ? sE : sB, rb);
          __syncthreads();
          if (p + 1 <= i) {
            tile_fetch<T>(ra, Li, ld, i, p + 1);
            tile_fetch<T>(rb, M, ld, p + 1, l);
          }
          tile_mma<false>(cur ? sD : sA, cur ? sE : sB, acc);
          cur ^= 1;
        }
        __syncthreads();
      }
      acc_to_tile(sC, acc, -1.0);
      __syncthreads();
      tile_store<T>(Li, ld, i, l, sC);
      __syncthreads();
    }
    grid.sync();
  }

  TMARK(3 * nblk + 2);
  // ---- L^-T: LiT(l, i) = Li(i, l)^T for l <= i
  const int nt = nblk * (nblk + 1) / 2;
  for (int t = b; t < nt; t += G) {
    int ii = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
    while ((ii + 1) * (ii + 2) / 2 <= t) ++ii;
    while (ii * (ii + 1) / 2 > t) --ii;
    const int ll = t - ii * (ii + 1) / 2;
    tile_load<T>(sA, Li, ld, ii, ll);
    __syncthreads();
    tile_store<T>(LiT, ld, ll, ii, sA, true, ii == ll ? 2 : 0);
    __syncthreads();
  }
  grid.sync();
  TMARK(3 * nblk + 3);
}


inline int launch(adask_ctx* ctx, int dtype, void* M, int64_t k, int64_t kp, void* L, void* Li, void* LiT,
                  int* info, unsigned long long* tlog, cudaStream_t st, int* grid_out) {
  const int nblk = (int)(kp / NB);
  const char* fi = getenv("ADASK_CHOL_INV");
  CholArgs a{M, L, Li, LiT, (int)kp, nblk, (int)k, info, tlog, getenv("ADASK_CHOL_SLOWDIAG") ? 1 : 0,
             // fused inverse up to 64 block rows (k = 2048 at NB = 32): its per-step
             // updates are single tile products, which lose to the doubling's long
             // chains once the updates outnumber the SMs several times over
             // (k = 1024: 528 -> 478 us; k = 2048: even; k = 4096: +4%)
             fi ? (atoi(fi) != 0) : (nblk <= 64)};
  const int smem = 5 * NB * NBP * (int)sizeof(double);
  void* fn = dtype == ADASK_F64 ? (void*)k_chol_coop<double> : (void*)k_chol_coop<float>;
  ADASK_TRY(ensure_smem_attr(fn, smem));
  static int per_sm_cache[2] = {-1, -1}, nsm_cache = -1;  // per dtype; one device type per process
  int& per_sm = per_sm_cache[dtype == ADASK_F64 ? 0 : 1];
  if (per_sm < 0) ADASK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kCholThreads, smem));
  if (nsm_cache < 0) cudaDeviceGetAttribute(&nsm_cache, cudaDevAttrMultiProcessorCount, ctx->device);
  int nsm = nsm_cache;
  if (per_sm < 1) return fail(ADASK_E_CUDA, "chol: kernel cannot be resident");
  int grid = nsm;  // one CTA per SM
  const int maxwork = nblk * (nblk + 1) / 2;
  if (grid > maxwork) grid = maxwork > 1 ? maxwork : 1;
  if (const char* g = getenv("ADASK_CHOL_GRID")) grid = atoi(g) > 0 ? atoi(g) : 1;
  void* args[] = {&a};
  ADASK_CUDA(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kCholThreads), args, smem, st));
  ADASK_LAUNCHED(ctx);
  *grid_out = grid;
  return ADASK_OK;
}
