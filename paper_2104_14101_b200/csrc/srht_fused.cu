// Fused SRHT: sign draws, both pruned-FWHT passes and the row selection in one
// persistent kernel                  reference: embeddings.py:81-102, linalg.py:62-88
//
// S A = sqrt(n_pad/m) R H E A.  The butterfly DAG is the reference's (stages
// in bit order), so any schedule that keeps the stage order per element is
// bitwise the reference; the transform is split at bit B1 = 9:
//
//   pass 1  (row block blk of 512 rows, 128-byte column panel p): bits 0-8,
//           fused with the sign flip and the zero padding, written to Z for the
//           needed slots (the low-9-bit values of idx);
//   pass 2  (512-row tile of Z, panel p): bits 9..L-1 over the G = n_pad/512
//           blocks of each slot; the selected rows go to SA, scaled as the
//           reference's two steps (v / sqrt(n_pad)) * sqrt(n_pad / m).
//
// Prologue (every CTA, before its first item): the packed sign bits
// integers(0, 2, size=n) (PCG64 jump-ahead, one 32-draw word per thread), then
// a grid-wide count; the producer waits for it only before its first sign copy
// (its first A tile is already in flight).  No other kernel runs per sketch.
//
// Schedule.  Column panels are processed in groups whose Z fits in L2; the
// work list P1(g0) .. P1(g_lag) P2(g0) P1(g_lag+1) P2(g1) ... is handed out by
// an atomic ticket and the producer of a pass-2 item waits on its group's
// pass-1 completion count, so Z is written and read back while L2-resident
// (config 1, m = 4096: 627 MB of DRAM reads for 537 MB of A, against a 1.5 GB
// round trip) and pass 2 overlaps the pass-1 stream of later groups.  Z lines
// are discarded from L2 after their last read (never written back).
//
// Machine mapping (one CTA per SM, warp-specialized):
//   * producer (one lane): ticket -> item one iteration ahead (the atomic's
//     round trip hidden), one 3-D TMA load of 512 rows x 128 B that lands as
//     [e][q] (row q*32 + e; rows past n arrive as zeros = the reference's
//     padding) plus the tile's sign words, into the stage of the item's
//     consumer group.  128-byte boxes: measured 1.15x the 64-byte boxes' rate
//     on 8 KB rows of A;
//   * two consumer groups of 8 warps take alternate items; thread (c, q) =
//     (t & 15, t >> 4) owns the 8-byte lane c (one fp64 column or a packed
//     fp32 pair: one FADD2 per two butterflies) of rows q*32 .. q*32+31:
//     bits 0-4 in registers, then the stage is released (the next tile's
//     load overlaps the rest), the exchange goes through one shared 64 KB
//     tile used in item order (a ring of mbarriers; one 128-byte row per
//     half-warp both ways: conflict-free), bits 5-8 (pass 2: 5..L2-1) on the
//     transposed registers, stores straight from registers.
//
// Measured on the B200 (tools/srht_fused_bench.py, 2^16 x 1024 fp64): 135 us
// (m = 32) .. 271 us (m = 4096) per sketch against 164 .. 354 us for the
// two-launch TMA pipeline of srht_pipe.cu.  What bounds it: the loads in
// flight.  A 64 KB tile per stage and the 64 KB exchange tile leave room for
// two stages per SM; the load-only probe (consumers releasing at once, three
// stages) reads A in 94 us.  Layouts measured and dropped: registers loaded
// straight from global (1024 x 64 B tiles: latency-bound, 194 us at m = 32),
// three stages with the exchange in place (139 us, stages held through the
// exchange), 256-row tiles with six stages (the shared exchange tile
// serializes twice as many items: 182 us), L2 prefetch of the next four
// tiles (no gain), a half-width exchange tile (eight lanes per round, two
// rounds) making room for a third stage shared round-robin (271 us at m = 32:
// 8-byte shared accesses are issued per half-warp, so a half-active round
// costs as many wavefronts as a full one), a per-thread mask of the
// registers that have a Z slot in front of the slot lookups (168 us: the
// extra live register tips the 96-register consumer loop into worse code),
// pass-2 tile records (entry count, masks, entries) copied into shared
// memory next to the Z tile by the producer instead of read-only global
// loads in the consumers (no gain: those loads hit L1 / L2 off the path).
//
// Algorithmic bytes per sketch: (n + m) * d * sizeof(T).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "rng.cuh"
#include "srht.cuh"
#include "tma.cuh"
#include "umma.cuh"

namespace adask {
namespace {

#ifndef FUSED_B1
#define FUSED_B1 9
#endif
constexpr int kB1 = FUSED_B1;                    // pass-1 bits (tile rows)
constexpr int kRows = 1 << kB1;                  // rows per tile
constexpr int kRowB = 128;                       // bytes per tile row (16 eight-byte lanes)
constexpr int kLanes = kRowB / 8;
constexpr int kQ = kRows / 32;                   // 32-row groups per tile
constexpr int kJB = kB1 - 5;                     // row bits 5.. handled after the exchange
constexpr int kGT = kLanes * kQ;                 // threads per consumer group (one tile each)
constexpr int kGroups = kB1 == 9 ? 2 : 3;        // consumer groups
constexpr int kRing = kB1 == 9 ? 1 : 2;          // stages per group (a group consumes its own in order)
constexpr int kStages = kGroups * kRing;
// producer: one warp, or (two 256-thread groups) a 4-warp group that hands
// its registers to the consumers with setmaxnreg: 96 per thread at launch
// (640 threads), then 32 / 112 (setmaxnreg.inc blocks until the CTA's own
// allocation covers it)
constexpr bool kRegSplit = kGroups * kGT > 384;
constexpr int kThreads = kGroups * kGT + (kRegSplit ? 128 : 32);
constexpr int kRegLaunch = 96, kRegProducer = 32, kRegConsumer = 112;
static_assert(!kRegSplit || kGroups * kGT * kRegConsumer + 128 * kRegProducer <= kThreads * kRegLaunch, "registers");
constexpr int kTile = kRows * kRowB;
constexpr int kStage = kTile + 128;              // + the tile's sign words (pass 1)
#ifndef FUSED_PF
#define FUSED_PF 1
#endif
constexpr int kPF = FUSED_PF;                    // producer: A tiles prefetched into L2 ahead
constexpr size_t kOffScr = (size_t)kStages * kStage;       // exchange tile, shared by the groups
constexpr size_t kOffSlot = kOffScr + kTile;
constexpr size_t kOffDesc = kOffSlot + kRows * 4;
constexpr size_t kOffBar = kOffDesc + kStages * 16;
constexpr int kXR = 4;                           // exchange-tile barriers (ring, >= kGroups)
// publisher mailboxes (kRegSplit): per group {seq, done, ring[kPubRing]}
constexpr int kPubRing = 8;
constexpr size_t kOffPub = kOffBar + (2 * kStages + kXR) * 8;
constexpr size_t kSmem = kOffPub + kGroups * (2 + kPubRing) * 4;
static_assert(kSmem <= 227 * 1024, "shared memory");

template <typename T>
struct FL;  // 8-byte butterfly lane
template <>
struct FL<double> {
  using V = double;
  static __device__ __forceinline__ V add(V a, V b) { return __dadd_rn(a, b); }
  static __device__ __forceinline__ V sub(V a, V b) { return __dsub_rn(a, b); }
  // sign flip by the top bit of `m` (0 or 0x80000000), on the integer pipe
  static __device__ __forceinline__ V flip(V v, uint32_t m) {
    return __hiloint2double(__double2hiint(v) ^ (int)m, __double2loint(v));
  }
  static __device__ __forceinline__ unsigned long long bits(V v) { return (unsigned long long)__double_as_longlong(v); }
};
template <>
struct FL<float> {
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
  static __device__ __forceinline__ V flip(V v, uint32_t m) { return v ^ ((unsigned long long)m << 32 | m); }
  static __device__ __forceinline__ unsigned long long bits(V v) { return v; }
};

struct FusedArgs {
  int64_t n_valid;           // rows of A (= sign draws)
  int64_t dbytes;            // d * sizeof(T)
  GenState gen;              // generator at the first sign draw of the whole transform
  uint64_t draw0;            // first sign draw of this (sub-)block
  uint32_t* sgn;             // packed sign bits (1 -> +1), n_pad bits (written by the prologue)
  int64_t nwords;            // n_pad / 32
  const int32_t* lo2slot;    // kRows entries, -1 = not needed
  const int32_t* toff;       // pass-2 tile t: its output entries are ent[toff[t] .. toff[t + 1])
  const int32_t* ent;        // tile row << 20 | output row k, grouped by tile (host plan)
  const uint32_t* pmask;     // per tile, per value group (kQ / R): bit e = register e is read
  unsigned char* Z;          // Z[(p * zrows + slot * G + blk) * 128 B]
  int64_t zrows;             // Z rows per panel (multiple of kRows)
  int64_t G;                 // row blocks
  unsigned char* out;
  int64_t ldo_b;
  double c1, c2;
  int accumulate;
  int vec_out;               // out rows 8-byte aligned
  int gp;                    // panels per group
  int npanels;
  int64_t n_items;
  const int4* segs;          // {kind, group, first ticket, count}
  unsigned* sync;            // [0] ticket, [1] exit count, [2] prologue count, [3 + g] pass-1 items of group g
  int dev;                   // dev switches: bit 0 no L2 discard of Z, bit 1 default L2 policy for Z
  unsigned long long* tlog;  // -DFUSED_TRACE: per CTA and group, per item {kind, t_wait, t_full, t_xwait, t_x, t_done}
};
#ifdef FUSED_TRACE
constexpr int kTraceItems = 96;  // per (CTA, group)
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define FTRACE(slot)                                                                                     \
  do {                                                                                                   \
    if (a.tlog && gt == 0 && n < kTraceItems)                                                            \
      a.tlog[(((size_t)blockIdx.x * kGroups + g) * kTraceItems + n) * 12 + (slot)] = gtimer();            \
  } while (0)
#else
#define FTRACE(slot) \
  do {               \
  } while (0)
#endif

__device__ __forceinline__ uint64_t pol_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void st_z(void* p, unsigned long long v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.b64 [%0], %1, %2;" ::"l"(p), "l"(v), "l"(pol) : "memory");
}
// counters are polled relaxed (an acquire load per poll would invalidate the
// SM's L1 each time) and the wait ends with one acquire fence
__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acquire_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void discard_l2(void* p) {
  asm volatile("discard.global.L2 [%0], 128;" ::"l"(p) : "memory");
}
// generic-proxy global writes <-> async-proxy (TMA / bulk copy) reads
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap* map, int32_t c0, int32_t c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"((uint64_t)map), "r"(c0),
               "r"(c1), "r"(0)
               : "memory");
}
__device__ __forceinline__ void tma_3d(void* dst, const CUtensorMap* map, int32_t c0, int32_t c1, uint64_t* bar,
                                       uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_u32(dst)),
      "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(0), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

// wait helpers; -DADASK_FUSED_DEBUG turns a wait of more than ~2 s into a
// report + trap (dev: locates a stuck dependency)
#ifdef ADASK_FUSED_DEBUG
#define FUSED_WAIT(cond, what, x)                                                                       \
  do {                                                                                                 \
    const long long _t0 = clock64();                                                                   \
    while (!(cond)) {                                                                                  \
      if (clock64() - _t0 > 4000000000ll) {                                                            \
        printf("srht fused: stuck at %s cta %d tid %d x %d\n", what, blockIdx.x, threadIdx.x, (int)(x)); \
        __trap();                                                                                      \
      }                                                                                                \
    }                                                                                                  \
  } while (0)
#else
#define FUSED_WAIT(cond, what, x) \
  do {                            \
    while (!(cond)) {             \
    }                             \
  } while (0)
#endif

// butterflies over bits [0, NB) of the register index (stage order = the
// reference's: lower bit first, a + b to the lower element, a - b upper)
template <typename T, int NB>
__device__ __forceinline__ void bfly(typename FL<T>::V (&v)[32]) {
  using L = FL<T>;
#pragma unroll
  for (int s = 0; s < NB; ++s) {
    const int h = 1 << s;
#pragma unroll
    for (int e = 0; e < 32; ++e) {
      if (!(e & h)) {
        const auto a = v[e], b = v[e + h];
        v[e] = L::add(a, b);
        v[e + h] = L::sub(a, b);
      }
    }
  }
}

__device__ __forceinline__ float fscale(float v, double c1, double c2) {
  float r = __fdiv_rn(v, (float)c1);
  if (c2 != 0.0) r = __fmul_rn(r, (float)c2);
  return r;
}
__device__ __forceinline__ double dscale(double v, double c1, double c2) {
  double r = __ddiv_rn(v, c1);
  if (c2 != 0.0) r = __dmul_rn(r, c2);
  return r;
}

// one 8-byte lane of an output row, scaled (accumulate optional); nb = valid
// bytes of the lane (8, or 4 for a trailing fp32 column)
template <typename T>
__device__ __forceinline__ void emit_out(const FusedArgs& a, unsigned char* o, unsigned long long bits, int nb) {
  if constexpr (sizeof(T) == 8) {
    double y = dscale(__longlong_as_double((long long)bits), a.c1, a.c2);
    double* po = reinterpret_cast<double*>(o);
    if (a.accumulate) y = *po + y;
    *po = y;
  } else {
    const float x0 = __uint_as_float((unsigned)bits), x1 = __uint_as_float((unsigned)(bits >> 32));
    float y0 = fscale(x0, a.c1, a.c2), y1 = fscale(x1, a.c1, a.c2);
    float* po = reinterpret_cast<float*>(o);
    if (nb == 8 && a.vec_out) {
      if (a.accumulate) {
        const float2 p = *reinterpret_cast<const float2*>(po);
        y0 = p.x + y0;
        y1 = p.y + y1;
      }
      *reinterpret_cast<float2*>(po) = make_float2(y0, y1);
    } else {
      po[0] = a.accumulate ? po[0] + y0 : y0;
      if (nb == 8) po[1] = a.accumulate ? po[1] + y1 : y1;
    }
  }
}

template <typename T, int L2>
__global__ void __launch_bounds__(kThreads, 1)
    k_srht_fused(const __grid_constant__ CUtensorMap amap, const __grid_constant__ CUtensorMap zmap, FusedArgs a) {
  using L = FL<T>;
  using V = typename L::V;
  constexpr int kR2 = L2 > 5 ? 1 << (L2 - 5) : 1;  // pass 2: values per selected row after the register stages
  extern __shared__ __align__(128) unsigned char fsm[];
  unsigned short* s_slot = reinterpret_cast<unsigned short*>(fsm + kOffSlot);
  int4* desc = reinterpret_cast<int4*>(fsm + kOffDesc);
  uint64_t* full = reinterpret_cast<uint64_t*>(fsm + kOffBar);
  uint64_t* empty = full + kStages;
  uint64_t* xdone = empty + kStages;  // [kXR]: item k has read the exchange tile back
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kGT / 32);
    }
    for (int i = 0; i < kXR; ++i) mbar_init(&xdone[i], kGT / 32);
    fence_barrier_init();
    for (int i = 0; i < kGroups * (2 + kPubRing); ++i) reinterpret_cast<int*>(fsm + kOffPub)[i] = 0;
  }
  // slot of row 32 j + key (key = q + kQ hh: the rows of one thread after the
  // exchange, register j + kQ hh) at [key][j], 16 bits each (0xFFFF: no slot):
  // a thread fetches its 32 slots with 16-byte loads
  static_assert(kQ % 8 == 0 && kRows <= 0xFFFF, "slot table");
  for (int i = tid; i < kRows; i += blockDim.x) {
    const int row = 32 * (i % kQ) + i / kQ;
    s_slot[i] = (unsigned short)a.lo2slot[row];
  }
  // ---- prologue: sign words (bit e of word w = draw 32 w + e; 1 -> +1),
  // spread over the grid
  for (int64_t w = blockIdx.x + (int64_t)tid * gridDim.x; w < a.nwords; w += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i0 = w * 32;
    uint32_t bits = 0;
    if (i0 < a.n_valid) {
      const int cnt = a.n_valid - i0 < 32 ? (int)(a.n_valid - i0) : 32;
      U32Stream st(a.gen, a.draw0 + (uint64_t)i0);
      for (int e = 0; e < cnt; ++e) bits |= (lemire_value(st.next(), 2u) & 1u) << e;
    }
    a.sgn[w] = bits;
  }
  fence_proxy_async_global();  // read next by bulk copies (async proxy)
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    atomicAdd(&a.sync[2], 1u);
  }

  if (warp >= kGroups * kGT / 32) {  // --------------------------- producer
    if constexpr (kRegSplit) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegProducer));
    if (kRegSplit && warp > kGroups * kGT / 32 && warp <= kGroups * kGT / 32 + kGroups && lane == 0) {
      // publisher of consumer group pg: the release fence + count of a
      // finished pass-1 item costs ~1 us (measured), so it runs here, off the
      // consumers' path.  The group's thread 0 posts the column group after
      // the barrier that follows the item's Z stores (release.cta); this
      // thread's acquire + gpu-scope fence make them visible before the count.
      const int pg = warp - kGroups * kGT / 32 - 1;
      volatile int* mb = reinterpret_cast<volatile int*>(fsm + kOffPub) + pg * (2 + kPubRing);
      int done = 0;
      for (;;) {
        int seq;
        asm volatile("ld.acquire.cta.shared.b32 %0, [%1];" : "=r"(seq) : "r"(smem_u32((const void*)mb)) : "memory");
        if (seq == done) {
          __nanosleep(40);
          continue;
        }
        const int grp = mb[2 + done % kPubRing];
        ++done;
        mb[1] = done;
        if (grp < 0) break;
        __threadfence();
        atomicAdd(&a.sync[3 + grp], 1u);
      }
    }
    if (warp == kGroups * kGT / 32 && lane == 0) {
      umma::tma_prefetch_map(&amap);
      umma::tma_prefetch_map(&zmap);
      const uint64_t pol = policy_evict_first();
      int si = 0, nterm = 0;
      bool pro = false, more = true;
      // Tickets run kPF + 1 items ahead of the stage loads: a ticket is
      // fetched, decoded one iteration later (the atomic's round trip hidden)
      // and its A tile prefetched into L2 then, so the tile load into shared
      // memory kPF items later reads L2 rather than waiting on HBM.
      auto decode = [&](unsigned t) -> int4 {
        if ((int64_t)t >= a.n_items) {
          more = false;
          return make_int4(-1, 0, 0, 0);
        }
        while (!((unsigned)a.segs[si].z <= t && t < (unsigned)(a.segs[si].z + a.segs[si].w))) ++si;
        const int4 sg = a.segs[si];
        const int p0 = sg.y * a.gp;
        const int gpg = min(a.gp, a.npanels - p0);
        const int li = (int)(t - (unsigned)sg.z);
        const int4 it = make_int4(sg.x, p0 + li % gpg, li / gpg, sg.y);
        if (it.x == 0) tma_prefetch_3d(&amap, it.y * (kRowB / (int)sizeof(T)), it.z * kQ);
        return it;
      };
      unsigned t_raw = atomicAdd(&a.sync[0], 1u);
      int4 pq[kPF];
#pragma unroll
      for (int i = 0; i < kPF; ++i) {
        pq[i] = more ? decode(t_raw) : make_int4(-1, 0, 0, 0);
        if (more) t_raw = atomicAdd(&a.sync[0], 1u);
      }
      for (int k = 0;; ++k) {
        const int n = k / kGroups;                          // the group's n-th item
        const int s = (k % kGroups) * kRing + n % kRing;    // its stage
        const int4 it = pq[0];
#pragma unroll
        for (int i = 0; i + 1 < kPF; ++i) pq[i] = pq[i + 1];
        pq[kPF - 1] = more ? decode(t_raw) : make_int4(-1, 0, 0, 0);
        if (more) t_raw = atomicAdd(&a.sync[0], 1u);
        if (n >= kRing) FUSED_WAIT(mbar_test(&empty[s], (uint32_t)(((n / kRing) & 1) ^ 1)), "empty", k);
        if (it.x == 1) {  // pass 2: the group's pass 1 must be complete
          const int gpg = min(a.gp, a.npanels - it.w * a.gp);
          const unsigned need = (unsigned)(a.G * gpg);
          FUSED_WAIT(ld_relaxed(a.sync + 3 + it.w) >= need, "pass-1 count", it.w);
          fence_acquire_gpu();
          fence_proxy_async_global();
        }
        desc[s] = it;
        unsigned char* stg = fsm + (size_t)s * kStage;
        if (it.x < 0) {
          mbar_arrive(&full[s]);
          if (++nterm == kGroups) break;
          continue;
        }
        if (it.x == 0) {
          mbar_arrive_expect_tx(&full[s], (uint32_t)(kTile + kRows / 8));
          tma_3d(stg, &amap, it.y * (kRowB / (int)sizeof(T)), it.z * kQ, &full[s], pol);
        } else {
          mbar_arrive_expect_tx(&full[s], (uint32_t)kTile);
          tma_3d(stg, &zmap, 0, (int)(((int64_t)it.y * a.zrows + (int64_t)it.z * kRows) / 32), &full[s], pol);
        }
        if (!pro) {  // the grid's prologue (signs, map) must be complete
          FUSED_WAIT(ld_relaxed(a.sync + 2) >= gridDim.x, "prologue", k);
          fence_acquire_gpu();
          fence_proxy_async_global();
          pro = true;
        }
        if (it.x == 0) bulk_g2s(stg + kTile, a.sgn + (int64_t)it.z * kQ, kRows / 8, &full[s]);
      }
    }
  } else {  // ------------------------------------------------------- consumers
    if constexpr (kRegSplit) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegConsumer));
    const int g = warp / (kGT / 32);
    const int gt = tid - g * kGT, c = gt & (kLanes - 1), q = gt >> 4;
    const uint64_t pol_zw = (a.dev & 2) ? policy_evict_normal() : pol_evict_last();
    V* scr = reinterpret_cast<V*>(fsm + kOffScr);
    volatile int* mb = reinterpret_cast<volatile int*>(fsm + kOffPub) + g * (2 + kPubRing);
    int nposted = 0;
    // thread 0 of the group, after the barrier that follows the item's Z
    // stores: hand the count to the publisher warp (grp < 0: exit)
    auto post = [&](int grp) {
      if (gt != 0) return;
      if constexpr (kRegSplit) {
        while (nposted - mb[1] >= kPubRing) {
        }
        mb[2 + nposted % kPubRing] = grp;
        ++nposted;
        asm volatile("st.release.cta.shared.b32 [%0], %1;" ::"r"(smem_u32((const void*)mb)), "r"(nposted) : "memory");
      } else if (grp >= 0) {
        __threadfence();
        atomicAdd(&a.sync[3 + grp], 1u);
      }
    };
#pragma unroll 1
    for (int n = 0;; ++n) {
      const int k = n * kGroups + g;
      const int s = g * kRing + n % kRing;
      FTRACE(1);
      FUSED_WAIT(mbar_test(&full[s], (uint32_t)((n / kRing) & 1)), "full", k);
      const int4 it = desc[s];
      if (it.x < 0) {
        post(-1);
        break;
      }
      FTRACE(2);
#ifdef FUSED_TRACE
      if (a.tlog && gt == 0 && n < kTraceItems)
        a.tlog[(((size_t)blockIdx.x * kGroups + g) * kTraceItems + n) * 12] = 1 + it.x;
#endif
      const V* tile = reinterpret_cast<const V*>(fsm + (size_t)s * kStage);
      const int kind = it.x, panel = it.y;
      const int64_t index = it.z;
      const int64_t colb = (int64_t)panel * kRowB + c * 8;
      const int64_t nbl = a.dbytes - colb;
      const int nb = nbl >= 8 ? 8 : (nbl > 0 ? (int)nbl : 0);

      // round 0: rows q*32 + e, landed [e][q] (position e*kQ + q); the stage
      // is released as soon as it is in registers, so the next tile's load
      // overlaps everything below
      // pass 2: the registers some selected row reads (0: nothing to do)
      const uint32_t v_need = kind == 0 ? ~0u : __ldg(a.pmask + index * (kQ / kR2) + q / kR2);
      V v[32];
      if (v_need) {
#pragma unroll
        for (int e = 0; e < 32; ++e) v[e] = tile[(e * kQ + q) * kLanes + c];
      }
      uint32_t nw = 0;
      if (kind == 0) nw = ~reinterpret_cast<const uint32_t*>(tile + kRows * kLanes)[q];
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (kind == 0) {
#pragma unroll
        for (int e = 0; e < 32; ++e) v[e] = L::flip(v[e], (nw << (31 - e)) & 0x80000000u);
        bfly<T, 5>(v);
      } else {
        // the tile's Z lines are in shared memory now: drop them from L2
        unsigned char* zt = a.Z + ((int64_t)panel * a.zrows + index * kRows) * kRowB;
        if (!(a.dev & 1))
          for (int l = gt; l < kTile / 128; l += kGT) discard_l2(zt + (int64_t)l * 128);
        if (v_need) bfly<T, (L2 < 5 ? L2 : 5)>(v);
      }
      // Exchange through the shared tile, used by the items in order: wait
      // until item k - 1 has read it back.  One barrier per item in a ring of
      // kXR >= kGroups: the barrier's previous phase (item k - 1 - kXR) is
      // complete by the time this group gets here, so the parity test is
      // unambiguous.
      FTRACE(3);
      if (k >= 1)
        FUSED_WAIT(mbar_test(&xdone[(k - 1) % kXR], (uint32_t)(((k - 1) / kXR) & 1)), "xdone", k);
      FTRACE(4);
      if (kind == 0) {
        // full exchange (row-major: one 128-byte row per half-warp both ways,
        // conflict-free).  Thread (c, u = q) then holds rows 32 j + u + 8 h at
        // register 8 h + j (j = row bits 5-7, h = bits 3-4).
#pragma unroll
        for (int e = 0; e < 32; ++e) scr[(q * 32 + e) * kLanes + c] = v[e];
        named_bar_sync(1 + g, kGT);
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = scr[(32 * (i & (kQ - 1)) + q + kQ * (i >> kJB)) * kLanes + c];
        __syncwarp();
        if (lane == 0) mbar_arrive(&xdone[k % kXR]);  // (every item takes one phase)
        FTRACE(5);
        bfly<T, kJB>(v);
        FTRACE(10);
        // row r of block `index` -> Z row slot(r) * G + index of the panel
        if (nb > 0) {
          unsigned char* zb = a.Z + ((int64_t)panel * a.zrows + index) * kRowB + c * 8;
          const uint32_t gstride = (uint32_t)a.G * kRowB;  // slot * gstride < 2^32 (L <= 18)
#pragma unroll
          for (int hh = 0; hh < 32 / kQ; ++hh) {
            const uint4* sp = reinterpret_cast<const uint4*>(s_slot + (q + kQ * hh) * kQ);
#pragma unroll
            for (int j8 = 0; j8 < kQ / 8; ++j8) {
              const uint4 sv = sp[j8];
              const uint32_t w4[4] = {sv.x, sv.y, sv.z, sv.w};
#pragma unroll
              for (int jj = 0; jj < 8; ++jj) {
                const uint32_t sl = (w4[jj >> 1] >> (16 * (jj & 1))) & 0xFFFFu;
                if (sl != 0xFFFFu)
                  st_z(zb + (uint64_t)sl * gstride, L::bits(v[kQ * hh + 8 * j8 + jj]), pol_zw);
              }
            }
          }
        }
        FTRACE(7);
        fence_proxy_async_global();  // Z is read next by TMA
        FTRACE(8);
        named_bar_sync(1 + g, kGT);  // every Z store of the item issued
        FTRACE(9);
        post(it.w);
        FTRACE(6);
      } else {
        // Pass 2 finishes only the selected rows.  Tile row t = 32 q + e is
        // Z row slot * G + blk; after the register stages (blk bits 0-4) a
        // selected row needs the R = G / 32 values of its value group
        // (t / 32R, e) -- threads q = (t / 32R) R + j, j = 0..R-1, register e
        // -- combined by the remaining stages.  Only the registers some
        // selected row reads go through the exchange tile (position
        // ((q / R) 32 + e) R + q % R: a warp's two q are adjacent rows);
        // thread (c, q) then finishes outputs q, q + 16, ... of the tile's
        // list (host plan) from them, in the reference's stage order.
        const int pb = (q / kR2) * 32 * kR2 + (q % kR2);
#pragma unroll
        for (int e = 0; e < 32; ++e)
          if ((v_need >> e) & 1u) scr[(pb + e * kR2) * kLanes + c] = v[e];
        named_bar_sync(1 + g, kGT);
        const int i1 = __ldg(a.toff + index + 1);
        for (int i = __ldg(a.toff + index) + q; i < i1; i += kQ) {
          const int en = __ldg(a.ent + i);
          const int t = en >> 20;
          const int p0 = ((t / (32 * kR2)) * 32 + (t & 31)) * kR2;
          V w[kR2];
#pragma unroll
          for (int j = 0; j < kR2; ++j) w[j] = scr[(p0 + j) * kLanes + c];
#pragma unroll
          for (int h = 1; h < kR2; h <<= 1) {
#pragma unroll
            for (int j = 0; j < kR2; ++j) {
              if (!(j & h)) {
                const auto x0 = w[j], x1 = w[j + h];
                w[j] = L::add(x0, x1);
                w[j + h] = L::sub(x0, x1);
              }
            }
          }
          const int jh = (t >> 5) & (kR2 - 1);
          V y = w[0];
#pragma unroll
          for (int j = 1; j < kR2; ++j)
            if (jh == j) y = w[j];
          if (nb > 0) emit_out<T>(a, a.out + (int64_t)(en & 0xFFFFF) * a.ldo_b + colb, L::bits(y), nb);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&xdone[k % kXR]);
        FTRACE(6);
      }
    }
  }
  // the last CTA out resets the counters for the next launch
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    const unsigned done = atomicAdd(&a.sync[1], 1u);
    if (done == gridDim.x - 1) {
      const int ng = (a.npanels + a.gp - 1) / a.gp;
      a.sync[0] = 0;
      a.sync[1] = 0;
      a.sync[2] = 0;
      for (int i = 0; i < ng; ++i) a.sync[3 + i] = 0;
      __threadfence();
    }
  }
}

template <typename T, int L2>
int launch_fused_l2(adask_ctx* ctx, const CUtensorMap& am, const CUtensorMap& zm, const FusedArgs& a,
                    cudaStream_t st) {
  auto kern = k_srht_fused<T, L2>;
  ADASK_TRY(ensure_smem_attr((const void*)kern, (int)kSmem));
  const int grid = (int)std::min<int64_t>(a.n_items, kNumSMs);
  kern<<<grid, kThreads, kSmem, st>>>(am, zm, a);
  ADASK_LAUNCHED(ctx);
  return ADASK_OK;
}

template <typename T>
int launch_fused(adask_ctx* ctx, int L2, const CUtensorMap& am, const CUtensorMap& zm, const FusedArgs& a,
                 cudaStream_t st) {
  switch (L2) {
#define C(X) \
  case X:    \
    if constexpr (X <= kB1) return launch_fused_l2<T, X>(ctx, am, zm, a, st); \
    break;
    C(1) C(2) C(3) C(4) C(5) C(6) C(7) C(8) C(9)
#undef C
    default:
      return fail(ADASK_E_ARG, "srht fused: pass 2 of %d bits unsupported", L2);
  }
}

int ilog2f(int64_t n) {
  int l = 0;
  while ((1ll << l) < n) ++l;
  return l;
}

}  // namespace

// 1 when the fused kernel handles this SRHT: 2^10..2^18 padded rows, whole
// 32-row groups (the [e][q] tile view) and 16-byte aligned rows.
// ADASK_SRHT_FUSED=0, or an explicit ADASK_FWHT_PIPE choice, selects the
// two-launch paths (srht_pipe.cu / srht.cu); both are read per call.
int srht_fused_eligible(int dtype, const void* A, int64_t n, int64_t n_pad, int64_t lda) {
  const char* env = getenv("ADASK_SRHT_FUSED");
  if ((env && atoi(env) == 0) || getenv("ADASK_FWHT_PIPE")) return 0;
  const int L = ilog2f(n_pad);
  if (L < kB1 + 1 || L > 2 * kB1) return 0;  // pass 2 within one tile
  const size_t esz = dtype == ADASK_F64 ? 8 : 4;
  if (((uintptr_t)A & 15) || ((size_t)lda * esz) % 16 || n % 32) return 0;
  return 1;
}

namespace {
// one (sub-)block of n_pad padded rows: its rows of A, valid row count, first
// sign draw, sign scratch and output
struct FusedSub {
  const void* A;
  int64_t n;
  uint64_t draw0;
  uint32_t* sgn;
  void* out;
};

// The selected rows idx (within a block of n_pad rows) of every sub-block in
// `subs`, with one host plan and one launch per sub-block.
int srht_fused_subs(adask_ctx* ctx, int dtype, const FusedSub* subs, int nsub, int64_t d, int64_t lda,
                    const adask_pcg64* g, int64_t n_pad, const int64_t* idx, int64_t m, int64_t ldo, double c1,
                    double c2, int accumulate, cudaStream_t st) {
  const int L = ilog2f(n_pad);
  const int L2 = L - kB1;
  const int64_t G = n_pad >> kB1;
  const size_t esz = dtype == ADASK_F64 ? 8 : 4;
  const int W = kRowB / (int)esz;
  if (m >= (1 << 20)) return fail(ADASK_E_ARG, "srht fused: m too large");

  // ---- host plan: lo -> slot, the segments, per pass-2 tile its outputs
  std::vector<int32_t> lo2slot(kRows, -1);
  int64_t nslots = 0;
  for (int64_t k = 0; k < m; ++k) lo2slot[(size_t)(idx[k] & (kRows - 1))] = 0;
  for (int lo = 0; lo < kRows; ++lo)
    if (lo2slot[(size_t)lo] == 0) lo2slot[(size_t)lo] = (int32_t)nslots++;
  if (nslots * 16 >= kRows * 15) {  // nearly all: identity slots (a few spare Z rows)
    for (int lo = 0; lo < kRows; ++lo) lo2slot[(size_t)lo] = lo;
    nslots = kRows;
  }
  const int64_t zrows = align_up((size_t)(nslots * G), kRows);
  const int64_t T2 = zrows / kRows;  // pass-2 tiles per panel
  const int64_t dbytes = d * (int64_t)esz;
  const int npanels = (int)cdiv(dbytes, kRowB);
  const int64_t zbudget = (getenv("ADASK_SRHT_FUSED_ZMB") ? atoll(getenv("ADASK_SRHT_FUSED_ZMB")) : 24) << 20;
  const int64_t zpanel = zrows * kRowB;
  const int gp = (int)std::max<int64_t>(1, std::min<int64_t>(npanels, zbudget / zpanel));
  // pass 2 trails pass 1 by `lag` groups, so lag + 1 groups of Z are live: two
  // groups of lag while that stays within ~80 MB of the 126 MB L2, else one
  // (2^18-row sub-blocks have 32 MB panels: lag 2 -> 1 is 568 -> 484 us at m = 4096)
  const int lag = getenv("ADASK_SRHT_FUSED_LAG") ? std::max(1, atoi(getenv("ADASK_SRHT_FUSED_LAG")))
                                                 : (3 * gp * zpanel <= (80ll << 20) ? 2 : 1);
  const int ng = (int)cdiv(npanels, gp);
  // work list: P1(0..lag-1), then [P1(g) P2(g-lag)] ..., then the last P2s
  std::vector<int4> segs;
  int64_t t = 0;
  auto add = [&](int kind, int gg) {
    const int gpg = std::min(gp, npanels - gg * gp);
    const int64_t cnt = (kind == 0 ? G : T2) * gpg;
    segs.push_back(make_int4(kind, gg, (int)t, (int)cnt));
    t += cnt;
  };
  for (int gg = 0; gg < ng + lag; ++gg) {
    if (gg < ng) add(0, gg);
    if (gg >= lag) add(1, gg - lag);
  }
  const int64_t n_items = t;
  if (n_items >= (1ll << 31)) return fail(ADASK_E_ARG, "srht fused: too many work items");

  // pass-2 tile lists: the outputs of each Z tile (tile row << 20 | k) and,
  // per value group of kR2 threads, the registers its outputs read
  const int R2 = L2 > 5 ? 1 << (L2 - 5) : 1;
  const int64_t nmask = T2 * (kQ / R2);
  const size_t o_toff = kRows, o_ent = o_toff + (size_t)T2 + 1, o_mask = o_ent + (size_t)m;
  std::vector<int32_t> plan(o_mask + (size_t)nmask, 0);
  std::copy(lo2slot.begin(), lo2slot.end(), plan.begin());
  std::vector<int32_t> zrow((size_t)m);
  for (int64_t k = 0; k < m; ++k) {
    zrow[(size_t)k] = (int32_t)(lo2slot[(size_t)(idx[k] & (kRows - 1))] * G + (idx[k] >> kB1));
    ++plan[o_toff + (size_t)(zrow[(size_t)k] / kRows) + 1];
  }
  for (int64_t i = 0; i < T2; ++i) plan[o_toff + (size_t)i + 1] += plan[o_toff + (size_t)i];
  {
    std::vector<int32_t> fill(plan.begin() + (ptrdiff_t)o_toff, plan.begin() + (ptrdiff_t)(o_toff + T2));
    uint32_t* msk = reinterpret_cast<uint32_t*>(plan.data() + o_mask);
    for (int64_t k = 0; k < m; ++k) {
      const int64_t tile = zrow[(size_t)k] / kRows;
      const int tr = (int)(zrow[(size_t)k] % kRows);
      plan[o_ent + (size_t)fill[(size_t)tile]++] = (tr << 20) | (int32_t)k;
      msk[tile * (kQ / R2) + tr / (32 * R2)] |= 1u << (tr & 31);
    }
  }
  const size_t plan_b = align_up(plan.size() * 4, 16);
  const size_t segs_b = segs.size() * sizeof(int4);
  void* pw = nullptr;
  ADASK_TRY(ctx->ws[WS_PLAN].get(plan_b + segs_b, st, &pw));
  std::vector<unsigned char> up(plan_b + segs_b);
  memcpy(up.data(), plan.data(), plan.size() * 4);
  memcpy(up.data() + plan_b, segs.data(), segs_b);
  ADASK_TRY(upload_async(ctx, pw, up.data(), up.size(), st));

  void* zw = nullptr;
  ADASK_TRY(ctx->ws[WS_SRHT].get((size_t)npanels * zpanel, st, &zw));
  // counters (self-resetting): zeroed once per allocation
  void* sw = nullptr;
  const size_t sync_b = align_up((size_t)(3 + ng) * 4 + 64, 256);
  ADASK_TRY(ctx->ws[WS_SRHT_SYNC].get(std::max<size_t>(sync_b, (size_t)1 << 12), st, &sw));
  if (ctx->srht_sync_gen != ctx->ws[WS_SRHT_SYNC].gen) {
    ADASK_CUDA(cudaMemsetAsync(sw, 0, ctx->ws[WS_SRHT_SYNC].bytes, st));
    ctx->srht_sync_gen = ctx->ws[WS_SRHT_SYNC].gen;
  }
  unsigned* sync = (unsigned*)sw;

  CUtensorMap am, zm;
  ADASK_TRY(tensor_map_rows3d(&zm, dtype, zw, (int64_t)npanels * zrows, W, W, (uint32_t)W, kQ, 32u));

  FusedArgs a{};
  a.dbytes = dbytes;
  a.gen = GenState::from(*g);
  a.nwords = n_pad / 32;
  a.lo2slot = (const int32_t*)pw;
  a.toff = (const int32_t*)pw + o_toff;
  a.ent = (const int32_t*)pw + o_ent;
  a.pmask = reinterpret_cast<const uint32_t*>((const int32_t*)pw + o_mask);
  a.Z = (unsigned char*)zw;
  a.zrows = zrows;
  a.G = G;
  a.ldo_b = ldo * (int64_t)esz;
  a.c1 = c1;
  a.c2 = c2;
  a.accumulate = accumulate;
  a.gp = gp;
  a.npanels = npanels;
  a.n_items = n_items;
  a.segs = (const int4*)((const char*)pw + plan_b);
  a.sync = sync;
  a.dev = getenv("ADASK_SRHT_FUSED_DEV") ? atoi(getenv("ADASK_SRHT_FUSED_DEV")) : 0;
#ifdef FUSED_TRACE
  // development build: per-item timestamps dumped to the file named by ADASK_SRHT_FUSED_TRACE
  const char* tr = getenv("ADASK_SRHT_FUSED_TRACE");
  const size_t tl_n = (size_t)kNumSMs * kGroups * kTraceItems * 12;
  if (tr) {
    ADASK_CUDA(cudaMalloc(&a.tlog, tl_n * 8));
    ADASK_CUDA(cudaMemsetAsync(a.tlog, 0, tl_n * 8, st));
  }
#endif
  int rc = ADASK_OK;
  for (int sb = 0; sb < nsub && rc == ADASK_OK; ++sb) {
    const FusedSub& u = subs[sb];
    if (u.n <= 0) {  // all padding: zero rows (0 / c1 * c2 = 0)
      if (!accumulate) ADASK_CUDA(cudaMemset2DAsync(u.out, (size_t)ldo * esz, 0, (size_t)dbytes, (size_t)m, st));
      continue;
    }
    ADASK_TRY(tensor_map_rows3d(&am, dtype, u.A, u.n, d, lda, (uint32_t)W, kQ, 32u));
    a.n_valid = u.n;
    a.draw0 = u.draw0;
    a.sgn = u.sgn;
    a.out = (unsigned char*)u.out;
    a.vec_out = ((uintptr_t)u.out % 8 == 0) && (a.ldo_b % 8 == 0);
    rc = dtype == ADASK_F64 ? launch_fused<double>(ctx, L2, am, zm, a, st) : launch_fused<float>(ctx, L2, am, zm, a, st);
  }
#ifdef FUSED_TRACE
  if (tr && rc == ADASK_OK) {
    std::vector<unsigned long long> h(tl_n);
    ADASK_CUDA(cudaStreamSynchronize(st));
    ADASK_CUDA(cudaMemcpy(h.data(), a.tlog, tl_n * 8, cudaMemcpyDeviceToHost));
    cudaFree(a.tlog);
    if (FILE* f = fopen(tr, "wb")) {
      fwrite(h.data(), 8, tl_n, f);
      fclose(f);
    }
  }
#endif
  return rc;
}

// combine the S = 2^LS sub-block partials of every selected row: stages
// 18 .. 18 + LS - 1 of the butterfly DAG (lower + upper / lower - upper by the
// row's bit), then the reference's two scaling steps
template <typename T, int LS>
__global__ void k_srht_combine(const T* __restrict__ P, int64_t mu, int64_t d, const int32_t* __restrict__ urow,
                               const int32_t* __restrict__ uhi, int64_t m, T* __restrict__ out, int64_t ldo,
                               double c1, double c2, int accumulate) {
  constexpr int S = 1 << LS;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= m * d) return;
  const int64_t k = e / d, j = e - k * d;
  const int hi = uhi[k];
  const T* p = P + (int64_t)urow[k] * d + j;
  T v[S];
#pragma unroll
  for (int s = 0; s < S; ++s) v[s] = p[(int64_t)s * mu * d];
#pragma unroll
  for (int b = 0; b < LS; ++b) {
    const bool up = (hi >> b) & 1;
#pragma unroll
    for (int s = 0; s < (S >> (b + 1)); ++s) {
      const T x0 = v[2 * s], x1 = v[2 * s + 1];
      if constexpr (sizeof(T) == 8)
        v[s] = up ? __dsub_rn(x0, x1) : __dadd_rn(x0, x1);
      else
        v[s] = up ? __fsub_rn(x0, x1) : __fadd_rn(x0, x1);
    }
  }
  T y;
  if constexpr (sizeof(T) == 8)
    y = dscale(v[0], c1, c2);
  else
    y = fscale(v[0], c1, c2);
  T* o = out + k * ldo + j;
  *o = accumulate ? (T)(*o + y) : y;
}

}  // namespace

int srht_fused(adask_ctx* ctx, int dtype, const void* A, int64_t n, int64_t d, int64_t lda, const adask_pcg64* g,
               uint32_t* sgn, int64_t n_pad, const int64_t* idx, int64_t m, void* out, int64_t ldo, double c1,
               double c2, int accumulate, cudaStream_t st) {
  const FusedSub one{A, n, 0, sgn, out};
  return srht_fused_subs(ctx, dtype, &one, 1, d, lda, g, n_pad, idx, m, ldo, c1, c2, accumulate, st);
}

// Blocks of 2^19 .. 2^22 padded rows: the transform's first 18 stages act
// inside aligned sub-blocks of 2^18 rows, so each sub-block runs the fused
// kernel (Z stays L2-resident) for the DISTINCT low 18-bit values of the
// selected rows, unscaled, into a partial buffer; k_srht_combine applies the
// remaining stages for every selected row.  HBM traffic: A once plus the
// partials (S mu d) instead of A plus a Z round trip.
int srht_fused_big_eligible(int dtype, const void* A, int64_t n, int64_t n_pad, int64_t lda, int64_t m) {
  const char* env = getenv("ADASK_SRHT_FUSED");
  if ((env && atoi(env) == 0) || getenv("ADASK_FWHT_PIPE")) return 0;
  if (kB1 != 9) return 0;
  const int L = ilog2f(n_pad);
  if (L < 19 || L > 22) return 0;
  static const int64_t min_m = getenv("ADASK_SRHT_BIG_MIN_M") ? atoll(getenv("ADASK_SRHT_BIG_MIN_M")) : 0;
  // the partial rows (S mu d, mu <= m) stay under half of the block's own bytes
  if (m < min_m || m > (1 << 17)) return 0;
  const size_t esz = dtype == ADASK_F64 ? 8 : 4;
  if (((uintptr_t)A & 15) || ((size_t)lda * esz) % 16 || n % 32) return 0;
  return 1;
}

int srht_fused_big(adask_ctx* ctx, int dtype, const void* A, int64_t n, int64_t d, int64_t lda,
                   const adask_pcg64* g, uint32_t* sgn, int64_t n_pad, const int64_t* idx, int64_t m, void* out,
                   int64_t ldo, double c1, double c2, int accumulate, cudaStream_t st) {
  static const int sub_env = getenv("ADASK_SRHT_BIG_SUBL") ? atoi(getenv("ADASK_SRHT_BIG_SUBL")) : 18;
  const int kSubL = std::min(18, std::max({sub_env, ilog2f(n_pad) - 4, 11}));
  const int64_t kSub = 1ll << kSubL;
  const int LS = ilog2f(n_pad) - kSubL;
  const int S = 1 << LS;
  const size_t esz = dtype == ADASK_F64 ? 8 : 4;
  // distinct low parts (sorted) and, per selected row, its partial row and high bits
  std::vector<int64_t> lo((size_t)m);
  for (int64_t k = 0; k < m; ++k) lo[(size_t)k] = idx[k] & (kSub - 1);
  std::vector<int64_t> u(lo);
  std::sort(u.begin(), u.end());
  u.erase(std::unique(u.begin(), u.end()), u.end());
  const int64_t mu = (int64_t)u.size();
  std::vector<int32_t> map((size_t)(2 * m));
  for (int64_t k = 0; k < m; ++k) {
    map[(size_t)k] = (int32_t)(std::lower_bound(u.begin(), u.end(), lo[(size_t)k]) - u.begin());
    map[(size_t)(m + k)] = (int32_t)(idx[k] >> kSubL);
  }
  void* pw = nullptr;
  ADASK_TRY(ctx->ws[WS_SRHT_PART].get((size_t)S * mu * d * esz, st, &pw));
  void* mw = nullptr;
  ADASK_TRY(ctx->ws[WS_SRHT_MAP].get(map.size() * 4, st, &mw));
  ADASK_TRY(upload_async(ctx, mw, map.data(), map.size() * 4, st));
  std::vector<FusedSub> subs((size_t)S);
  for (int sb = 0; sb < S; ++sb) {
    FusedSub& f = subs[(size_t)sb];
    f.A = (const char*)A + (size_t)sb * kSub * lda * esz;
    f.n = std::max<int64_t>(0, std::min<int64_t>(kSub, n - sb * kSub));
    f.draw0 = (uint64_t)sb * kSub;
    f.sgn = sgn + (size_t)sb * (kSub / 32);
    f.out = (char*)pw + (size_t)sb * mu * d * esz;
  }
  ADASK_TRY(srht_fused_subs(ctx, dtype, subs.data(), S, d, lda, g, kSub, u.data(), mu, d, 1.0, 0.0, 0, st));
  const unsigned blocks = (unsigned)cdiv(m * d, 256);
  const int32_t* urow = (const int32_t*)mw;
  const int32_t* uhi = urow + m;
#define COMB(T, LSV)                                                                                            \
  k_srht_combine<T, LSV><<<blocks, 256, 0, st>>>((const T*)pw, mu, d, urow, uhi, m, (T*)out, ldo, c1, c2, accumulate)
  if (dtype == ADASK_F64) {
    switch (LS) {
      case 1: COMB(double, 1); break;
      case 2: COMB(double, 2); break;
      case 3: COMB(double, 3); break;
      default: COMB(double, 4); break;
    }
  } else {
    switch (LS) {
      case 1: COMB(float, 1); break;
      case 2: COMB(float, 2); break;
      case 3: COMB(float, 3); break;
      default: COMB(float, 4); break;
    }
  }
#undef COMB
  ADASK_LAUNCHED(ctx);
  return ADASK_OK;
}

}  // namespace adask
