// SJLT bucket accumulation, streamed by bulk copies  reference: embeddings.py:105-129
//
// Same arithmetic as k_bucket_accumulate (sjlt.cu): every bucket b sums
// sign_i * A[i, :] over its entries in ascending entry order, in fp64, with
// no floating-point atomics -- bitwise the reference's csr_matvecs.  Different
// machine schedule:
//   * persistent CTAs (one per SM); items = (bucket, column panel), the panel
//     as wide as the whole row when there are enough buckets (16 KB rows of
//     2^20 x 2048 fp64 are gathered as whole rows, not 2 KB column slices);
//   * a producer warp loads the bucket's entry indices and signs 32 at a
//     time and streams each row segment into a STAGES-deep shared-memory ring
//     with cp.async.bulk (mbarrier completion, L2 evict-first): the bytes in
//     flight per SM are set by the ring (~190 KB), not by registers/occupancy;
//   * 8 consumer warps own 16-byte column chunks of the panel and accumulate
//     the ring rows in order; the bucket's row of SA is written at item end.
// Bytes: (n + m) * d * sizeof(T) (algorithmic; the gather reads each row once).
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "sjlt.cuh"
#include "tma.cuh"

namespace adask {
namespace {

constexpr int kNW = 8;
constexpr int kThreads = (kNW + 1) * 32;
constexpr int kRingBytes = 196 * 1024;
constexpr int kMaxChunks = 4;  // 16-byte chunks per consumer thread (panel <= 16 KB)

struct SjltPipeArgs {
  const void* A;
  int64_t lda, d;
  const int32_t* order;  // sorted entry indices
  const int32_t* start;  // bucket offsets [m + 1]
  const int32_t* sgn;    // sign draw per entry (1 -> +1)
  int32_t s;             // nonzeros per column (entry e is row e / s)
  int64_t m;
  int64_t pw;            // panel width in elements (multiple of 16 bytes)
  int64_t npanels;
  int stages;
  int stage_bytes;
  double scale;          // 1 / sqrt(s)
  int use_scale;
  void* SA;
  int64_t ldsa;
  int accumulate;
};

template <typename T>
__global__ void __launch_bounds__(kThreads, 1) k_sjlt_pipe(SjltPipeArgs a) {
  constexpr int CE = 16 / (int)sizeof(T);  // elements per 16-byte chunk
  constexpr int NT = kNW * 32;
  extern __shared__ __align__(128) unsigned char ssm[];
  const int STAGES = a.stages, SB = a.stage_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(ssm + (size_t)STAGES * SB);
  uint64_t* empty = full + STAGES;
  int* meta = reinterpret_cast<int*>(empty + STAGES);  // sign per stage
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t n_items = a.m * a.npanels;

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kNW);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == kNW) {  // ---------------- producer
    const uint64_t pol = policy_evict_first();
    const char* A = reinterpret_cast<const char*>(a.A);
    const size_t esz = sizeof(T);
    int st = 0;          // ring position (no integer division per row)
    uint32_t ph = 0;
    bool wrapped = false;
    const int64_t lda_b = a.lda * (int64_t)esz;
    for (int64_t it = blockIdx.x; it < n_items; it += gridDim.x) {
      const int64_t b = it / a.npanels, p = it - b * a.npanels;
      const int32_t p0 = a.start[b], p1 = a.start[b + 1];
      const int64_t c0 = p * a.pw;
      const uint32_t bytes = (uint32_t)(std::min<int64_t>(a.pw, a.d - c0) * esz);
      const char* Ab = A + c0 * (int64_t)esz;
      for (int32_t g = p0; g < p1; g += 32) {
        const int32_t e = g + lane < p1 ? __ldg(a.order + g + lane) : 0;
        const int32_t sg = g + lane < p1 ? __ldg(a.sgn + e) : 0;
        const int32_t rw = a.s == 1 ? e : e / a.s;
        const int cnt = min(32, p1 - g);
        for (int j = 0; j < cnt; ++j) {
          const int32_t rj = __shfl_sync(0xffffffffu, rw, j);
          const int32_t sj = __shfl_sync(0xffffffffu, sg, j);
          if (lane == 0) {
            if (wrapped) mbar_wait(&empty[st], ph ^ 1);
            meta[st] = sj;
            mbar_arrive_expect_tx(&full[st], bytes);
            bulk_g2s_evict_first(ssm + (size_t)st * SB, Ab + (int64_t)rj * lda_b, bytes, &full[st], pol);
          }
          if (++st == STAGES) {
            st = 0;
            ph ^= 1;
            wrapped = true;
          }
        }
      }
    }
    return;
  }

  // ---------------- consumers: thread owns chunks tid, tid + NT, ... of the panel
  int st = 0;
  uint32_t ph = 0;
  for (int64_t it = blockIdx.x; it < n_items; it += gridDim.x) {
    const int64_t b = it / a.npanels, p = it - b * a.npanels;
    const int32_t p0 = a.start[b], p1 = a.start[b + 1];
    const int64_t c0 = p * a.pw;
    const int64_t width = std::min<int64_t>(a.pw, a.d - c0);
    const int nch = (int)((width + CE - 1) / CE);
    double acc[kMaxChunks][CE];
#pragma unroll
    for (int k = 0; k < kMaxChunks; ++k)
#pragma unroll
      for (int v = 0; v < CE; ++v) acc[k][v] = 0.0;
    for (int32_t i = p0; i < p1; ++i) {
      mbar_wait(&full[st], ph);
      const int sg = meta[st];
      const unsigned char* row = ssm + (size_t)st * SB;
      uint4 q[kMaxChunks];
#pragma unroll
      for (int k = 0; k < kMaxChunks; ++k) {
        const int ch = tid + k * NT;
        if (ch < nch) q[k] = *reinterpret_cast<const uint4*>(row + ch * 16);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
      if (++st == STAGES) {
        st = 0;
        ph ^= 1;
      }
#pragma unroll
      for (int k = 0; k < kMaxChunks; ++k) {
        const int ch = tid + k * NT;
        if (ch < nch) {
          T x[CE];
          memcpy(x, &q[k], 16);
#pragma unroll
          for (int v = 0; v < CE; ++v) {
            const double xv = (double)x[v];
            if (a.use_scale)  // s > 1: y += (sign / sqrt(s)) * x, product then sum
              acc[k][v] = __dadd_rn(acc[k][v], __dmul_rn(sg ? a.scale : -a.scale, xv));
            else
              acc[k][v] = __dadd_rn(acc[k][v], sg ? xv : -xv);  // exact +-x
          }
        }
      }
    }
    T* dst = reinterpret_cast<T*>(a.SA) + b * a.ldsa + c0;
#pragma unroll
    for (int k = 0; k < kMaxChunks; ++k) {
      const int ch = tid + k * NT;
      if (ch < nch) {
#pragma unroll
        for (int v = 0; v < CE; ++v) {
          const int64_t c = (int64_t)ch * CE + v;
          if (c < width) {
            double r = acc[k][v];
            if (a.accumulate) r = (double)dst[c] + r;
            dst[c] = (T)r;
          }
        }
      }
    }
  }
}

}  // namespace

// 1 = launched; 0 = not eligible (the caller uses k_bucket_accumulate).
int sjlt_accumulate_pipe(adask_ctx* ctx, int dtype, const void* A, int64_t d, int64_t lda, const int32_t* order,
                         const int32_t* start, const int32_t* sgn, int32_t s, int64_t m, void* SA, int64_t ldsa,
                         int accumulate, cudaStream_t st, int* launched) {
  *launched = 0;
  int mode = 1;
  if (const char* e = getenv("ADASK_SJLT_PIPE")) mode = atoi(e);
  if (mode == 0) return ADASK_OK;
  const size_t esz = dtype == ADASK_F64 ? 8 : 4;
  if (((uintptr_t)A % 16) || ((size_t)lda * esz) % 16 || ((size_t)d * esz) % 16) return ADASK_OK;
  // panel: the whole row up to 16 KB; narrower (>= 4 KB) until there are
  // >= 2 items per SM
  const int64_t row_bytes = (int64_t)d * esz;
  // Whole 16 KB rows stream fastest (measured at 2^20 x 2048 fp64, m = 128:
  // 2.66 ms with 16 KB pieces, 3.46 with 8 KB, 5.1 with 4 KB: the DRAM sees
  // short random pieces) and a partly filled second wave costs little (the
  // active CTAs get the idle ones' bandwidth; m = 256: 2.81 ms with 256 items
  // against 3.53 with 512 half-row items), so the panel is halved only while
  // fewer than ~2/3 of the SMs would have an item.
  int64_t pb = std::min<int64_t>(row_bytes, (int64_t)kMaxChunks * kNW * 32 * 16);
  const int64_t min_pb = getenv("ADASK_SJLT_MINPB") ? atoll(getenv("ADASK_SJLT_MINPB")) : 2048;
  while (pb > min_pb && m * cdiv(row_bytes, pb) < 96) pb /= 2;
  pb = std::max<int64_t>(16, pb / 16 * 16);
  // very few buckets: the register kernel's narrow mode (ADASK_SJLT_PIPE=2 forces this one)
  static const int64_t pipe_min_m = getenv("ADASK_SJLT_PIPE_MIN_M") ? atoll(getenv("ADASK_SJLT_PIPE_MIN_M")) : 16;
  if (mode == 1 && m < pipe_min_m) return ADASK_OK;
  SjltPipeArgs a{};
  a.A = A;
  a.lda = lda;
  a.d = d;
  a.order = order;
  a.start = start;
  a.sgn = sgn;
  a.s = s;
  a.m = m;
  a.pw = pb / (int64_t)esz;
  a.npanels = cdiv(d, a.pw);
  a.stage_bytes = (int)align_up((size_t)pb, 128);
  a.stages = std::min<int>(32, kRingBytes / a.stage_bytes);
  a.scale = 1.0 / sqrt((double)s);
  a.use_scale = s > 1;
  a.SA = SA;
  a.ldsa = ldsa;
  a.accumulate = accumulate;
  const size_t smem = (size_t)a.stages * a.stage_bytes + (size_t)a.stages * (16 + 4) + 64;
  const int grid = (int)std::min<int64_t>(m * a.npanels, kNumSMs);
  if (dtype == ADASK_F64) {
    ADASK_TRY(ensure_smem_attr((const void*)k_sjlt_pipe<double>, (int)smem));
    k_sjlt_pipe<double><<<grid, kThreads, smem, st>>>(a);
  } else {
    ADASK_TRY(ensure_smem_attr((const void*)k_sjlt_pipe<float>, (int)smem));
    k_sjlt_pipe<float><<<grid, kThreads, smem, st>>>(a);
  }
  ADASK_LAUNCHED(ctx);
  *launched = 1;
  return ADASK_OK;
}

}  // namespace adask
