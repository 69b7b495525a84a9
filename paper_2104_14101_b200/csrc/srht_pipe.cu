// Pipelined two-pass pruned FWHT for the SRHT          reference: embeddings.py:81-102,
//                                                                 linalg.py:62-88
//
// Same butterfly DAG as srht.cu (stages h = 1, 2, 4, ... in bit order, so the
// result is bitwise the reference's), different machine schedule:
//
//   * persistent CTAs (one per SM), items = (row tile, column panel), column
//     panels fastest so the grid sweeps whole rows of A together;
//   * a producer warp streams each 1024-row x 64-byte tile into a 2-stage
//     shared-memory ring with ONE 3-D TMA tensor-map load (the view
//     {columns, row/32, row%32} lands the tile as [e][q], row q*32 + e; rows
//     past n arrive as zeros = the reference's zero padding) plus, by bulk
//     copy, the tile's sign words (pass 1) or its slice of the output-row map
//     (pass 2);
//   * 8 consumer warps run bits 0-4 in registers straight from the stage
//     (fp32 as packed pairs: one FADD2 per two butterflies), release it, and
//     run bits 5-9 in a scratch tile whose rows are permuted r ^ ((r>>5)&3) so
//     that every warp access covers the four 32-byte bank groups;
//   * emit: pass 1 writes Z straight from registers when every slot is
//     needed, else copies out only the needed slots; pass 2 copies out the
//     selected rows, scaled exactly as the reference's two steps (or writes the
//     two half transforms of an 11-bit pass 2, combined by k_srht_combine);
//   * fp64 with m >= 512 hands Z to the tile kernel's pass 2 (srht.cu), which
//     is faster on the short 2^(L-10)-point transforms.
//
// Bytes: pass 1 reads n_pad x d (A, zero rows free) and writes nslots*G x d of
// Z; pass 2 reads Z and writes m x d.  Both passes are HBM streams.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "srht.cuh"
#include "tma.cuh"
#include "umma.cuh"

namespace adask {
namespace {

enum { P1 = 0, P2 = 1 };


// 3-D tensor-map tile load, completion on an mbarrier
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int32_t c0, int32_t c1, int32_t c2,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(smem_u32(dst)),
      "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
constexpr int kNW = 8;                    // consumer warps
constexpr int kThreads = (kNW + 1) * 32;  // + one producer warp
constexpr int kSmemBudget = 220 * 1024;

struct PipeArgs {
  int64_t n_items, npanels, d;
  int64_t n_valid;          // pass 1: rows of A (rows past it are zero padding)
  int nslots;               // pass 1: needed slots (rows of a row block that reach Z)
  // pass 1
  const uint32_t* sgn;      // packed sign bits (1 -> +1) or null
  const int32_t* lo2slot;   // B entries or null (identity)
  void* Z;                  // Z[(slot*G + blk)*d + col]
  int64_t G;
  // pass 2
  const int32_t* map2;      // tile-row -> output row k (-1: none), padded; null = identity
  void* out;
  int64_t ldo;
  double c1, c2;
  int accumulate;
  int vec_out;              // out rows 16-byte aligned (ldo and base)
  int64_t ldz;              // row pitch of Z (d rounded up to 16 bytes)
  int b1;                   // pass-1 bits (identity map of pass 2: k = (hi << b1) | slot)
};

template <int LOG, int LOGT, int SEGB, typename T, int MODE>
struct PipeShape {
  static constexpr int W = SEGB / (int)sizeof(T);  // columns per panel
  static constexpr int BT = 1 << LOGT;             // tile rows
  static constexpr int NB0 = LOG < 5 ? LOG : 5;    // bits of round 0
  static constexpr int E0 = 1 << NB0;
  static constexpr int QB = BT / E0;               // round-0 units per column lane
  static constexpr int TILE = BT * SEGB;
  static constexpr int MAPB = MODE == P2 ? BT * 4 : BT / 8;  // pass 2: row map; pass 1: sign bits
  static constexpr int STAGE = (TILE + MAPB + 127) / 128 * 128;
  static constexpr int STAGES = 2;
  // scratch tile (rounds >= 1 and copy-out), then the pass-1 lo -> slot map
  // or the pass-2 row map of the tile being finished
  static constexpr int MAPX = MODE == P1 ? (4 << LOG) : BT * 4;
  static constexpr size_t OFF_SCR = (size_t)STAGES * STAGE;
  static constexpr size_t OFF_MAP = OFF_SCR + TILE;
  static constexpr size_t OFF_BAR = OFF_MAP + MAPX;
  static constexpr size_t SMEM = OFF_BAR + 2 * STAGES * 8;
  static constexpr int ROUNDS = (LOG + 4) / 5;
  static_assert(SMEM <= 227 * 1024, "shared memory");
  static_assert(LOGT >= LOG && LOG >= 2, "tile shape");
  static_assert(QB <= 256, "TMA box");
};

// 8-byte butterfly lanes: one fp64 value, or the two fp32 values of one row in
// adjacent columns (packed FADD2: one instruction per two butterflies)
template <typename T>
struct Lane8;
template <>
struct Lane8<double> {
  using V = double;
  static __device__ __forceinline__ V add(V a, V b) { return __dadd_rn(a, b); }
  static __device__ __forceinline__ V sub(V a, V b) { return __dsub_rn(a, b); }
  static __device__ __forceinline__ V neg_if(V v, bool neg) { return neg ? -v : v; }
};
template <>
struct Lane8<float> {
  using V = unsigned long long;
  static __device__ __forceinline__ V add(V a, V b) {
    V r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
  }
  static __device__ __forceinline__ V sub(V a, V b) {
    V r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
  }
  static __device__ __forceinline__ V neg_if(V v, bool neg) { return v ^ (neg ? 0x8000000080000000ull : 0ull); }
};

// butterflies over bits [0, NB) of v, where v[e] holds element e ^ X; for the
// first SWB stages the operands are swapped where bit s of X is set (exactly
// the reference's a + b and a - b on the logical elements)
template <typename T, int NB, int SWB>
__device__ __forceinline__ void butterflies_x(typename Lane8<T>::V* v, int X) {
  using L = Lane8<T>;
  using V = typename L::V;
#pragma unroll
  for (int s = 0; s < NB; ++s) {
    const int h = 1 << s;
    const bool f = s < SWB && ((X >> s) & 1);
#pragma unroll
    for (int e = 0; e < (1 << NB); ++e) {
      if (!(e & h)) {
        if (s < SWB) {
          const V a = f ? v[e + h] : v[e];  // logical lower
          const V b = f ? v[e] : v[e + h];  // logical upper
          const V su = L::add(a, b), di = L::sub(a, b);
          v[e] = f ? di : su;
          v[e + h] = f ? su : di;
        } else {
          const V a = v[e], b = v[e + h];
          v[e] = L::add(a, b);
          v[e + h] = L::sub(a, b);
        }
      }
    }
  }
}

template <typename T>
__device__ __forceinline__ T pipe_scale(T v, double c1, double c2) {
  if (c1 == 0.0) return v;
  if constexpr (sizeof(T) == 8) {
    double r = __ddiv_rn((double)v, c1);
    if (c2 != 0.0) r = __dmul_rn(r, c2);
    return (T)r;
  } else {
    float r = __fdiv_rn((float)v, (float)c1);
    if (c2 != 0.0) r = __fmul_rn(r, (float)c2);
    return (T)r;
  }
}

__device__ __forceinline__ int prow(int q, int e, int lo, int hi) {
  return (q & ((1 << lo) - 1)) | (e << lo) | ((q >> lo) << hi);
}

// Scratch layout: logical tile row r lives at row r ^ ((r >> NB0) & 3), so
// that the warp's units (consecutive q in round 0, consecutive low row bits
// afterwards) always cover the four 32-byte bank groups evenly.
template <int NB0>
__device__ __forceinline__ int sphys(int r) {
  return r ^ ((r >> NB0) & 3);
}

// Scratch row of element e of a unit whose rows are base + (e << LO): the
// XOR in sphys only touches row bits 0-1 and depends on bits NB0, NB0+1, so
// phys(e) = P[e & 3] + ((e >> 2) << (LO + 2)) with four per-unit bases --
// every other address is an immediate offset.
template <int NB0, int LO, int E>
__device__ __forceinline__ void unit_bases(int base, int* P) {
#pragma unroll
  for (int k = 0; k < 4 && k < E; ++k) P[k] = sphys<NB0>(base + (k << LO));
}

// Round over bits [LO, LO + NB) of the scratch tile, in place.  Units are
// processed UG at a time (all loads, then butterflies, then stores) so short
// rounds keep enough shared-memory loads in flight.
template <typename T, int BT, int W8, int NB, int NB0, int LO, int NT>
__device__ __forceinline__ void pipe_round(typename Lane8<T>::V* scr, int tid) {
  using V = typename Lane8<T>::V;
  constexpr int E = 1 << NB;
  constexpr int UNITS = BT * W8 / E;
  constexpr int HI = LO + NB;
  constexpr int UG0 = 32 / E > 0 ? 32 / E : 1;
  constexpr int UG = UG0 < UNITS / NT ? UG0 : (UNITS / NT > 0 ? UNITS / NT : 1);
  static_assert(UNITS % (NT * UG) == 0, "round units");
#pragma unroll 1
  for (int u0 = tid; u0 < UNITS; u0 += NT * UG) {
    V v[UG][E];
    int rw[UG][4];
#pragma unroll
    for (int g = 0; g < UG; ++g) {
      const int u = u0 + g * NT;
      const int c = u % W8, q = u / W8;
      int P[4];
      unit_bases<NB0, LO, E>(prow(q, 0, LO, HI), P);
#pragma unroll
      for (int k = 0; k < 4; ++k) rw[g][k] = P[k] * W8 + c;
#pragma unroll
      for (int e = 0; e < E; ++e) v[g][e] = scr[rw[g][e & 3] + ((e >> 2) << (LO + 2)) * W8];
    }
#pragma unroll
    for (int g = 0; g < UG; ++g) butterflies_x<T, NB, 0>(v[g], 0);
#pragma unroll
    for (int g = 0; g < UG; ++g)
#pragma unroll
      for (int e = 0; e < E; ++e) scr[rw[g][e & 3] + ((e >> 2) << (LO + 2)) * W8] = v[g][e];
  }
}

// Last pass-1 round with every slot needed: the butterflies' results go from
// registers straight to Z (8-byte lanes, 64-byte row segments per 8 lanes),
// skipping the scratch write-back and the copy-out pass.
template <typename T, int BT, int W8, int NB, int NB0, int LO, int NT>
__device__ __forceinline__ void pipe_round_emit(const typename Lane8<T>::V* scr, int tid, T* zb, int64_t sstride,
                                                int64_t col0, int64_t d) {
  using V = typename Lane8<T>::V;
  constexpr int E = 1 << NB;
  constexpr int UNITS = BT * W8 / E;
  constexpr int HI = LO + NB;
  constexpr int CPL = 8 / (int)sizeof(T);  // columns per 8-byte lane
  static_assert(UNITS % NT == 0, "emit units");
#pragma unroll 1
  for (int u = tid; u < UNITS; u += NT) {
    const int c = u % W8, q = u / W8;
    int P[4];
    const int base = prow(q, 0, LO, HI);
    unit_bases<NB0, LO, E>(base, P);
    V v[E];
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = scr[(P[e & 3] + ((e >> 2) << (LO + 2))) * W8 + c];
    butterflies_x<T, NB, 0>(v, 0);
    if (col0 + c * CPL < d) {
      T* z = zb + (int64_t)base * sstride + c * CPL;
      const int64_t step = sstride << LO;
#pragma unroll
      for (int e = 0; e < E; ++e) *reinterpret_cast<V*>(z + e * step) = v[e];
    }
  }
}

template <typename T, int LOG, int LOGT, int SEGB, int MODE>
__global__ void __launch_bounds__(kThreads, 1) k_fwht_pipe(const __grid_constant__ CUtensorMap smap, PipeArgs a) {
  using S = PipeShape<LOG, LOGT, SEGB, T, MODE>;
  using L = Lane8<T>;
  using V = typename L::V;
  constexpr int W = S::W, BT = S::BT, STAGES = S::STAGES, NB0 = S::NB0, E0 = S::E0, QB = S::QB;
  constexpr int W8 = SEGB / 8;             // 8-byte lanes per tile row
  constexpr int CH = SEGB / 16;            // 16-byte chunks per tile row
  constexpr int CE = 16 / (int)sizeof(T);  // elements per chunk
  constexpr int NT = kNW * 32;
  extern __shared__ __align__(128) unsigned char psm[];
  V* scr = reinterpret_cast<V*>(psm + S::OFF_SCR);
  int* mapx = reinterpret_cast<int*>(psm + S::OFF_MAP);
  uint64_t* full = reinterpret_cast<uint64_t*>(psm + S::OFF_BAR);
  uint64_t* empty = full + STAGES;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t npanels = a.npanels, n_items = a.n_items;

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kNW);
    }
    fence_barrier_init();
  }
  if constexpr (MODE == P1) {
    // slot -> row of the block (slots are numbered in ascending row order)
    for (int i = tid; i < (1 << LOG); i += blockDim.x) {
      const int sl = a.lo2slot ? a.lo2slot[i] : i;
      if (sl >= 0) mapx[sl] = i;
    }
  }
  __syncthreads();

  if (warp == kNW) {  // ---------------- producer
    if (lane == 0) {
      umma::tma_prefetch_map(&smap);
      const uint64_t pol = policy_evict_first();
      int it = 0;
      for (int64_t i = blockIdx.x; i < n_items; i += gridDim.x, ++it) {
        const int s = it % STAGES;
        const uint32_t ph = (uint32_t)((it / STAGES) & 1);
        if (it >= STAGES) mbar_wait(&empty[s], ph ^ 1);
        const int64_t ti = i / npanels, p = i - ti * npanels;
        const int64_t row0 = ti * BT;
        unsigned char* stg = psm + s * S::STAGE;
        const bool withmap = MODE == P2 ? a.map2 != nullptr : (a.sgn != nullptr && row0 < a.n_valid);
        mbar_arrive_expect_tx(&full[s], (uint32_t)(S::TILE + (withmap ? S::MAPB : 0)));
        // box {W columns, QB units, E0 rows}: lands as [e][q][column]
        tma_load_3d(stg, &smap, (int32_t)(p * W), (int32_t)(row0 / E0), 0, &full[s]);
        if (withmap) {
          if constexpr (MODE == P2)
            bulk_g2s_evict_first(stg + S::TILE, a.map2 + row0, (uint32_t)S::MAPB, &full[s], pol);
          else  // the tile's sign words (the sign buffer is padded to n_pad bits)
            bulk_g2s(stg + S::TILE, a.sgn + (row0 >> 5), (uint32_t)S::MAPB, &full[s]);
        }
      }
    }
    return;
  }

  // ---------------- consumers
#ifdef ADASK_PIPE_TRACE
  long long tw = 0, t0c = 0, t1c = 0, tcc = 0, tb = 0;
#define TR_MARK(var) do { long long _n = clock64(); var += _n - _tl; _tl = _n; } while (0)
#else
#define TR_MARK(var) do {} while (0)
#endif
  int it = 0;
#pragma unroll 1
  for (int64_t i = blockIdx.x; i < n_items; i += gridDim.x, ++it) {
#ifdef ADASK_PIPE_TRACE
    long long _tl = clock64();
#endif
    const int s = it % STAGES;
    const uint32_t ph = (uint32_t)((it / STAGES) & 1);
    const int64_t ti = i / npanels, p = i - ti * npanels;
    const int64_t row0 = ti * BT, col0 = p * W;
    const unsigned char* stg = psm + s * S::STAGE;
    const V* tile = reinterpret_cast<const V*>(stg);
    mbar_wait(&full[s], ph);
    TR_MARK(tw);
    named_bar_sync(1, NT);  // the previous tile's copy-out is done with scr / mapx
    TR_MARK(tb);

    // ---- round 0: stage ([e][q] layout) -> sign flip -> bits [0, NB0) -> scratch
    {
      constexpr int UNITS = QB * W8;
#pragma unroll 1
      for (int u = tid; u < UNITS; u += NT) {
        const int c = u % W8, q = u / W8;
        V v[E0];
#pragma unroll
        for (int e = 0; e < E0; ++e) v[e] = tile[(e * QB + q) * W8 + c];
        if (MODE == P1 && a.sgn) {
          // diag(signs) A: exact negation where the sign bit is 0 (E0 <= 32
          // consecutive aligned rows: one sign word)
          const int64_t gr = row0 + q * E0;
          const uint32_t* sw = reinterpret_cast<const uint32_t*>(stg + S::TILE);
          const uint32_t bits = gr < a.n_valid ? sw[(q * E0) >> 5] >> ((q * E0) & 31) : 0xffffffffu;
#pragma unroll
          for (int e = 0; e < E0; ++e) v[e] = L::neg_if(v[e], !((bits >> e) & 1u));
        }
        butterflies_x<T, NB0, 0>(v, 0);
        int P[4];
        unit_bases<NB0, 0, E0>(q * E0, P);
        V* col = scr + c;
#pragma unroll
        for (int e = 0; e < E0; ++e) col[(P[e & 3] + ((e >> 2) << 2)) * W8] = v[e];
      }
      if constexpr (MODE == P2) {
        if (a.map2) {
          const int* mp = reinterpret_cast<const int*>(stg + S::TILE);
          for (int r = tid; r < BT; r += NT) mapx[r] = mp[r];
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);  // stage free for the next TMA load
    }
    TR_MARK(t0c);
    static_assert(S::ROUNDS <= 3, "at most three rounds (LOG <= 15)");
    if constexpr (S::ROUNDS == 3) {
      named_bar_sync(1, NT);
      pipe_round<T, BT, W8, 5, NB0, 5, NT>(scr, tid);
    }
    // pass 1 with every slot needed (m >= 2^10 rows selected): direct emit
    const bool direct = MODE == P1 && S::ROUNDS == 2 && a.nslots == (1 << LOG);
    if constexpr (S::ROUNDS > 1) {
      constexpr int LO = 5 * (S::ROUNDS - 1);
      named_bar_sync(1, NT);
      if (direct)
        pipe_round_emit<T, BT, W8, LOG - LO, NB0, LO, NT>(scr, tid, reinterpret_cast<T*>(a.Z) + ti * a.ldz + col0,
                                                         a.G * a.ldz, col0, a.d);
      else
        pipe_round<T, BT, W8, LOG - LO, NB0, LO, NT>(scr, tid);
    }
    TR_MARK(t1c);
    if (direct) continue;
    named_bar_sync(1, NT);
    TR_MARK(tb);

    // ---- copy-out: the needed rows of the tile, 16-byte chunks
    const unsigned char* sb = reinterpret_cast<const unsigned char*>(scr);
    constexpr int PER0 = BT * CH / NT;
    static_assert(BT * CH % NT == 0, "copy-out split");
    if constexpr (MODE == P1) {
      // Z rows of the needed slots: chunk u = (slot u / CH, 16-byte chunk
      // u % CH); batches of 8 with every shared-memory read before the stores
      static_assert(LOGT == LOG, "pass-1 tiles are one row block");
      static_assert(NT % CH == 0, "chunk lane");
      const int total = a.nslots * CH;
      const int ch = tid % CH;
      const bool colok = col0 + ch * CE < a.d;
      T* zb = reinterpret_cast<T*>(a.Z) + ti * a.ldz + col0 + ch * CE;
      const int64_t sstride = a.G * a.ldz;
#pragma unroll 1
      for (int u0 = tid; u0 < total; u0 += 8 * NT) {
        uint4 q4[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int u = u0 + j * NT;
          if (u < total) {
            const int r = mapx[u / CH];
            q4[j] = *reinterpret_cast<const uint4*>(sb + sphys<NB0>(r) * SEGB + ch * 16);
          }
        }
        if (colok) {
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int u = u0 + j * NT;
            if (u < total) *reinterpret_cast<uint4*>(zb + (int64_t)(u / CH) * sstride) = q4[j];
          }
        }
      }
    } else {
      // selected rows of SA: look the whole tile's map up first (bit mask of
      // this thread's chunks that carry an output row), then one scaled store
      // per selected chunk
      static_assert(PER0 <= 32, "copy-out mask");
      uint32_t sel = 0;
#pragma unroll
      for (int j = 0; j < PER0; ++j) {
        const int u = tid + j * NT;
        const int r = u / CH, ch = u - r * CH;
        const bool on = a.map2 ? mapx[r] >= 0 : true;
        if (on && col0 + ch * CE < a.d) sel |= 1u << j;
      }
#pragma unroll 1
      while (sel) {
        const int j = __ffs(sel) - 1;
        sel &= sel - 1;
        const int u = tid + j * NT;
        const int r = u / CH, ch = u - r * CH;
        const int64_t gr = row0 + r;
        const int64_t k = a.map2 ? (int64_t)mapx[r] : (((gr & ((1 << LOG) - 1)) << a.b1) | (gr >> LOG));
        const int64_t col = col0 + ch * CE;
        const uint4 q4 = *reinterpret_cast<const uint4*>(sb + sphys<NB0>(r) * SEGB + ch * 16);
        T x[CE];
        memcpy(x, &q4, 16);
        T* o = reinterpret_cast<T*>(a.out) + k * a.ldo + col;
        if (a.vec_out && col + CE <= a.d) {
          T y[CE];
          if (a.accumulate) {
            const uint4 o4 = *reinterpret_cast<const uint4*>(o);
            memcpy(y, &o4, 16);
          }
#pragma unroll
          for (int t = 0; t < CE; ++t) {
            const T yv = pipe_scale<T>(x[t], a.c1, a.c2);
            y[t] = a.accumulate ? (T)(y[t] + yv) : yv;
          }
          uint4 w4;
          memcpy(&w4, y, 16);
          *reinterpret_cast<uint4*>(o) = w4;
        } else {
#pragma unroll 1
          for (int t = 0; t < CE && col + t < a.d; ++t) {
            const T yv = pipe_scale<T>(x[t], a.c1, a.c2);
            o[t] = a.accumulate ? (T)(o[t] + yv) : yv;
          }
        }
      }
    }
#ifdef ADASK_PIPE_TRACE
    TR_MARK(tcc);
#endif
  }
#ifdef ADASK_PIPE_TRACE
  if (lane == 0 && (blockIdx.x == 0 || blockIdx.x == 77) && (warp == 0 || warp == 5))
    printf("pipe trace L%d M%d cta %d warp %d items %d: wait %lld r0 %lld r1 %lld bar %lld copy %lld cycles/item\n",
           LOG, MODE, blockIdx.x, warp, it, tw / it, t0c / it, t1c / it, tb / it, tcc / it);
#endif
}

template <typename T, int LOG, int LOGT, int SEGB, int MODE>
int launch_pipe(adask_ctx* ctx, int dtype, const void* src, int64_t rows, int64_t tile_rows, int64_t ld,
                const PipeArgs& a0, cudaStream_t st) {
  using S = PipeShape<LOG, LOGT, SEGB, T, MODE>;
  CUtensorMap map;
  ADASK_TRY(tensor_map_rows3d(&map, dtype, src, rows, a0.d, ld, (uint32_t)S::W, (uint32_t)S::QB, (uint32_t)S::E0));
  PipeArgs a = a0;
  a.npanels = cdiv(a.d, S::W);
  a.n_items = cdiv(tile_rows, S::BT) * a.npanels;
  auto kern = k_fwht_pipe<T, LOG, LOGT, SEGB, MODE>;
  ADASK_TRY(ensure_smem_attr((const void*)kern, (int)S::SMEM));
  const int grid = (int)std::min<int64_t>(a.n_items, kNumSMs);
  kern<<<grid, kThreads, S::SMEM, st>>>(map, a);
  ADASK_LAUNCHED(ctx);
  return ADASK_OK;
}

// segment bytes and tile rows for a pass of LOG bits: 64-byte rows up to
// 2^10-row transforms, 32-byte rows for 2^11; tiles of 64 KB (several
// transforms per tile when LOG is small)
template <typename T, int MODE>
int dispatch_pipe(adask_ctx* ctx, int dtype, int log, const void* src, int64_t rows, int64_t tile_rows,
                  int64_t ld, const PipeArgs& a, cudaStream_t st) {
  if constexpr (MODE == P1) {
    if (log != 10) return fail(ADASK_E_ARG, "fwht pipe: pass 1 of %d bits unsupported", log);
    return launch_pipe<T, 10, 10, 64, MODE>(ctx, dtype, src, rows, tile_rows, ld, a, st);
  } else {
  switch (log) {
#define C64(L) \
  case L:      \
    return launch_pipe<T, L, 10, 64, MODE>(ctx, dtype, src, rows, tile_rows, ld, a, st);
    C64(2) C64(3) C64(4) C64(5) C64(6) C64(7) C64(8) C64(9) C64(10)
#undef C64
    default:
      return fail(ADASK_E_ARG, "fwht pipe: pass of %d bits unsupported", log);
  }
  }
}

}  // namespace

__global__ void k_map2_fill(int32_t* map2, int64_t rows) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < rows; i += (int64_t)gridDim.x * blockDim.x)
    map2[i] = -1;
}
__global__ void k_map2_scatter(const int32_t* __restrict__ pos, int64_t m, int32_t* __restrict__ map2) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < m; k += (int64_t)gridDim.x * blockDim.x)
    map2[pos[k]] = (int32_t)k;
}

int fwht_build_map2(adask_ctx* ctx, const int32_t* pos, int64_t m, int32_t* map2, int64_t rows, cudaStream_t st) {
  k_map2_fill<<<(unsigned)std::min<int64_t>(cdiv(rows, 256), 4 * kNumSMs), 256, 0, st>>>(map2, rows);
  ADASK_LAUNCHED(ctx);
  k_map2_scatter<<<(unsigned)std::min<int64_t>(cdiv(m, 256), 4 * kNumSMs), 256, 0, st>>>(pos, m, map2);
  ADASK_LAUNCHED(ctx);
  return ADASK_OK;
}

// 11-bit pass 2 = a 10-bit pass over each half of the slot's 2048 rows plus
// the last butterfly stage.  Outputs sharing (slot, low 10 bits) share the
// half results: the representative output w (any one of them) names the pair
// of rows w (half 0) and m + w (half 1) of U.
__global__ void k_map2_scatter_lo(const int32_t* __restrict__ pos, int64_t m, int32_t* __restrict__ map2) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < m; k += (int64_t)gridDim.x * blockDim.x)
    map2[pos[k] & ~1024] = (int32_t)k;
}
__global__ void k_map2_scatter_hi(const int32_t* __restrict__ pos, int64_t m, int32_t* __restrict__ map2,
                                  int32_t* __restrict__ rep) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < m; k += (int64_t)gridDim.x * blockDim.x) {
    const int32_t p0 = pos[k] & ~1024;
    const int32_t w = map2[p0];
    map2[p0 | 1024] = (int32_t)(w + m);
    rep[k] = w;
  }
}

int fwht_build_map2_comb(adask_ctx* ctx, const int32_t* pos, int64_t m, int32_t* map2, int64_t rows, int32_t* rep,
                         cudaStream_t st) {
  const unsigned gm = (unsigned)std::min<int64_t>(cdiv(m, 256), 4 * kNumSMs);
  k_map2_fill<<<(unsigned)std::min<int64_t>(cdiv(rows, 256), 4 * kNumSMs), 256, 0, st>>>(map2, rows);
  ADASK_LAUNCHED(ctx);
  k_map2_scatter_lo<<<gm, 256, 0, st>>>(pos, m, map2);
  ADASK_LAUNCHED(ctx);
  k_map2_scatter_hi<<<gm, 256, 0, st>>>(pos, m, map2, rep);
  ADASK_LAUNCHED(ctx);
  return ADASK_OK;
}

// last stage (bit L-1) and the reference's two scalings:
// SA[k] (+)= ((U[w] +/- U[m + w]) / c1) * c2, '+' for outputs in the lower half
template <typename T>
__global__ void k_srht_combine(const T* __restrict__ U, int64_t ldu, const int32_t* __restrict__ rep,
                               const int32_t* __restrict__ pos, int64_t m, int64_t d, T* __restrict__ out,
                               int64_t ldo, double c1, double c2, int accumulate) {
  const int64_t total = m * d;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = e / d, c = e - k * d;
    const int64_t w = rep[k];
    const T lo = U[w * ldu + c], hi = U[(m + w) * ldu + c];
    const T v = (pos[k] & 1024) ? (T)(lo - hi) : (T)(lo + hi);
    const T y = pipe_scale<T>(v, c1, c2);
    T* o = out + k * ldo + c;
    *o = accumulate ? (T)(*o + y) : y;
  }
}

namespace {
static int ilog2p(int64_t n) {
  int l = 0;
  while ((1ll << l) < n) ++l;
  return l;
}

}  // namespace

// 0 = not eligible (caller uses the tile kernels), 1 = eligible.
int fwht_pipe_eligible(int dtype, const void* A, int64_t n, int64_t n_pad, int64_t lda, int64_t m, bool selected) {
  int force = -1;
  if (const char* e = getenv("ADASK_FWHT_PIPE")) {
    if (atoi(e) == 0) return 0;
    if (atoi(e) == 2) m = 0;      // force the pipelined passes (tests)
    if (atoi(e) == 3) force = 2;  // force the hybrid (tests)
  }
  const int L = ilog2p(n_pad);
  const size_t esz = dtype == ADASK_F64 ? 8 : 4;
  if (L < 12 || L > 21) return 0;
  if (L == 21 && !selected) return 0;  // full 2^21-point transforms keep the tile kernels
  if (((uintptr_t)A & 15) || ((size_t)lda * esz) % 16) return 0;
  if (n % 32) return 0;  // the [e][q] tensor-map view of A needs whole 32-row groups
  // fp64 with many selected rows: the tile kernels' pass 2 is faster on the
  // short (2^(L-10)-point) transforms (measured at 2^16 x 1024, m = 1024-4096):
  // pipelined pass 1 + tile pass 2 (2), or all tile kernels (0) past 2^20 rows
  if (force == 2) return (selected && L <= 20) ? 2 : 0;
  if (dtype == ADASK_F64 && m >= 512) return (selected && L <= 20) ? 2 : 0;
  return 1;
}

int fwht_pipe_group(adask_ctx* ctx, int dtype, const void* A, int64_t n, int64_t d, int64_t lda, const uint32_t* sgn,
                    int64_t n_pad, int64_t m, void* out, int64_t ldo, double c1, double c2, int accumulate,
                    cudaStream_t st, int hybrid, bool selected, bool comb, int64_t nslots, int64_t zrows, int64_t B,
                    int64_t G, int b1, int L2, int L2p, const int32_t* d_plan, const int32_t* d_map2,
                    const int32_t* d_rep, void* zw, int64_t ldz, void* uw);

int fwht_select_pipe(adask_ctx* ctx, int dtype, const void* A, int64_t n, int64_t d, int64_t lda,
                     const uint32_t* sgn, int64_t n_pad, const int64_t* idx, int64_t m, void* out, int64_t ldo,
                     double c1, double c2, int accumulate, cudaStream_t st, int hybrid) {
  const int L = ilog2p(n_pad);
  const int b1 = 10;  // pass-1 tiles are 2^10-row blocks
  const int L2 = L - b1;
  const bool comb = L2 == 11;  // 10-bit pass 2 per half + the last stage (64-byte rows throughout)
  const int L2p = comb ? 10 : L2;
  const int64_t B = 1ll << b1, G = n_pad >> b1;
  const size_t esz = dtype == ADASK_F64 ? 8 : 4;
  const int64_t BT2 = 1024;  // pass-2 tile rows (dispatch_pipe: 64-byte rows, 2^10-row tiles)
  if (comb && !idx) return fail(ADASK_E_ARG, "fwht pipe: full transform with an 11-bit pass 2");

  // ---- host plan: lo -> slot (B entries) and, per selected row, its
  // position slot*G + hi in Z (m entries); the dense map is built on device
  std::vector<int32_t> plan;
  int64_t nslots = B;
  if (idx) {
    std::vector<int32_t> lo2slot((size_t)B, -1);
    nslots = 0;
    for (int64_t k = 0; k < m; ++k) lo2slot[(size_t)(idx[k] & (B - 1))] = 0;
    for (int64_t lo = 0; lo < B; ++lo)
      if (lo2slot[(size_t)lo] == 0) lo2slot[(size_t)lo] = (int32_t)nslots++;
    // nearly every slot needed: keep all of them (identity slots) so that
    // pass 1 emits Z straight from registers (the few unused rows are free)
    if (nslots * 16 >= B * 15) {
      for (int64_t lo = 0; lo < B; ++lo) lo2slot[(size_t)lo] = (int32_t)lo;
      nslots = B;
    }
    plan.resize((size_t)(B + m));
    std::copy(lo2slot.begin(), lo2slot.end(), plan.begin());
    for (int64_t k = 0; k < m; ++k)
      plan[(size_t)(B + k)] = (int32_t)(lo2slot[(size_t)(idx[k] & (B - 1))] * G + (idx[k] >> b1));
  }
  const int64_t zrows = nslots * G;
  const int64_t map_rows = cdiv(zrows, BT2) * BT2;
  int32_t* d_plan = nullptr;
  int32_t* d_map2 = nullptr;
  int32_t* d_rep = nullptr;
  const int64_t ldz_h = (int64_t)align_up((size_t)d, 16 / esz);
  hybrid = hybrid && idx && !comb && ldz_h == d;
  std::vector<int32_t> old_plan;  // hybrid: slot_start [nslots + 1] | ent_hi [m] | ent_k [m]
  if (hybrid) {
    old_plan.assign((size_t)(nslots + 1 + 2 * m), 0);
    int32_t* ss = old_plan.data();
    int32_t* eh = ss + nslots + 1;
    int32_t* ek = eh + m;
    for (int64_t k = 0; k < m; ++k) ss[plan[(size_t)(idx[k] & (B - 1))] + 1]++;
    for (int64_t q = 0; q < nslots; ++q) ss[q + 1] += ss[q];
    std::vector<int32_t> fill(ss, ss + nslots);
    for (int64_t k = 0; k < m; ++k) {
      const int32_t q = plan[(size_t)(idx[k] & (B - 1))];
      const int32_t pos = fill[(size_t)q]++;
      eh[pos] = (int32_t)(idx[k] >> b1);
      ek[pos] = (int32_t)k;
    }
  }
  if (idx) {
    void* pw = nullptr;
    ADASK_TRY(ctx->ws[WS_PLAN].get((plan.size() + (size_t)map_rows + (size_t)m + old_plan.size()) * 4 + 256, st,
                                   &pw));
    d_plan = (int32_t*)pw;
    d_map2 = d_plan + align_up(plan.size(), 16);
    d_rep = d_map2 + align_up((size_t)map_rows, 16);
    ADASK_TRY(upload_async(ctx, d_plan, plan.data(), plan.size() * 4, st));
    if (hybrid) {
      int32_t* d_old = d_rep + align_up((size_t)m, 16);
      ADASK_TRY(upload_async(ctx, d_old, old_plan.data(), old_plan.size() * 4, st));
      d_map2 = d_old;  // reused below as the old plan's base
    } else if (comb)
      ADASK_TRY(fwht_build_map2_comb(ctx, d_plan + B, m, d_map2, map_rows, d_rep, st));
    else
      ADASK_TRY(fwht_build_map2(ctx, d_plan + B, m, d_map2, map_rows, st));
  }
  // Column groups: when the intermediate Z of all d columns would exceed the
  // L2 budget, the two passes run group by group over column panels so that
  // a group's Z (nslots * G rows x its columns) is written by pass 1 and read
  // back by pass 2 while it is still L2-resident, instead of a round trip
  // through HBM (config 1 at m >= 512: Z is as large as A).  Every column is
  // transformed independently, so the result is bitwise the one-group result.
  // Off by default: measured at 2^16 x 1024 fp64 (tools/srht_bench.py), 2-16
  // groups of separate launches cost more in per-launch setup and wave tails
  // than the HBM round trip of Z they save (m = 4096: 357 us in one group,
  // 391-617 us in groups) -- the L2-resident schedule needs both passes in
  // one persistent kernel.
  static const int64_t zbudget =
      getenv("ADASK_SRHT_ZBUDGET_MB") ? (atoll(getenv("ADASK_SRHT_ZBUDGET_MB")) << 20) : INT64_MAX;
  const int64_t panel = 64 / (int64_t)esz;  // columns per 64-byte tile row
  int64_t gw = d;
  if ((int64_t)zrows * (int64_t)align_up((size_t)d, 16 / esz) * (int64_t)esz > zbudget) {
    gw = std::max<int64_t>(panel, zbudget / ((int64_t)zrows * (int64_t)esz) / panel * panel);
    gw = std::min<int64_t>(gw, d);
  }
  void* zw = nullptr;
  const int64_t ldz = (int64_t)align_up((size_t)gw, 16 / esz);
  ADASK_TRY(ctx->ws[WS_SRHT].get((size_t)zrows * ldz * esz, st, &zw));
  void* uw = nullptr;
  if (comb) ADASK_TRY(ctx->ws[WS_SRHT_U].get((size_t)2 * m * ldz * esz, st, &uw));
  for (int64_t c0 = 0; c0 < d; c0 += gw) {
    const int64_t w = std::min<int64_t>(gw, d - c0);
    ADASK_TRY(fwht_pipe_group(ctx, dtype, (const char*)A + c0 * esz, n, w, lda, sgn, n_pad, m, (char*)out + c0 * esz,
                              ldo, c1, c2, accumulate, st, hybrid, idx != nullptr, comb, nslots, zrows, B, G, b1, L2,
                              L2p, d_plan, d_map2, d_rep, zw, (int64_t)align_up((size_t)w, 16 / esz), uw));
  }
  return ADASK_OK;
}

// one column group of fwht_select_pipe: pass 1 over A's columns [c0, c0 + d)
// into Z (row pitch ldz), pass 2 from Z into the same columns of out
int fwht_pipe_group(adask_ctx* ctx, int dtype, const void* A, int64_t n, int64_t d, int64_t lda, const uint32_t* sgn,
                    int64_t n_pad, int64_t m, void* out, int64_t ldo, double c1, double c2, int accumulate,
                    cudaStream_t st, int hybrid, bool selected, bool comb, int64_t nslots, int64_t zrows, int64_t B,
                    int64_t G, int b1, int L2, int L2p, const int32_t* d_plan, const int32_t* d_map2,
                    const int32_t* d_rep, void* zw, int64_t ldz, void* uw) {
  (void)B;
  (void)selected;
  const size_t esz = dtype == ADASK_F64 ? 8 : 4;
  PipeArgs a{};
  a.d = d;
  a.nslots = (int)nslots;
  a.n_valid = n;
  a.sgn = sgn;
  a.lo2slot = d_plan;  // null when idx is null (identity)
  a.Z = zw;
  a.ldz = ldz;
  a.G = G;
  a.map2 = d_map2;
  a.b1 = b1;
  // pass 2 writes SA directly, or (comb) the half transforms into U
  a.out = comb ? uw : out;
  a.ldo = comb ? ldz : ldo;
  a.c1 = comb ? 0.0 : c1;
  a.c2 = comb ? 0.0 : c2;
  a.accumulate = comb ? 0 : accumulate;
  a.vec_out = ((uintptr_t)a.out % 16 == 0) && ((size_t)a.ldo * esz) % 16 == 0;
  // pass 1 reads rows [0, n) of A; rows [n, n_pad) are TMA out-of-bounds zeros
  if (hybrid) {
    a.map2 = nullptr;
    if (dtype == ADASK_F64)
      ADASK_TRY((dispatch_pipe<double, P1>(ctx, dtype, b1, A, n, n_pad, lda, a, st)));
    else
      ADASK_TRY((dispatch_pipe<float, P1>(ctx, dtype, b1, A, n, n_pad, lda, a, st)));
    const int32_t* ss = d_map2;
    return fwht_tile_pass2(ctx, dtype, L2, zw, G, d, nslots, ss, ss + nslots + 1, ss + nslots + 1 + m, out, ldo, c1,
                           c2, accumulate, st);
  }
  if (dtype == ADASK_F64) {
    ADASK_TRY((dispatch_pipe<double, P1>(ctx, dtype, b1, A, n, n_pad, lda, a, st)));
    ADASK_TRY((dispatch_pipe<double, P2>(ctx, dtype, L2p, zw, zrows, zrows, ldz, a, st)));
  } else {
    ADASK_TRY((dispatch_pipe<float, P1>(ctx, dtype, b1, A, n, n_pad, lda, a, st)));
    ADASK_TRY((dispatch_pipe<float, P2>(ctx, dtype, L2p, zw, zrows, zrows, ldz, a, st)));
  }
  if (comb) {
    const unsigned blocks = (unsigned)std::min<int64_t>(cdiv(m * d, 256), 8 * kNumSMs);
    if (dtype == ADASK_F64)
      k_srht_combine<double><<<blocks, 256, 0, st>>>((const double*)uw, ldz, d_rep, d_plan + B, m, d, (double*)out,
                                                     ldo, c1, c2, accumulate);
    else
      k_srht_combine<float><<<blocks, 256, 0, st>>>((const float*)uw, ldz, d_rep, d_plan + B, m, d, (float*)out, ldo,
                                                    c1, c2, accumulate);
    ADASK_LAUNCHED(ctx);
  }
  return ADASK_OK;
}

}  // namespace adask
