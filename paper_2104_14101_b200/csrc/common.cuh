// Shared plumbing for libadask: status handling, the device context and its
// grow-only workspaces, launch accounting, small device helpers.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <string>
#include <utility>
#include <vector>

#include "../../include/adask.h"

namespace adask {

constexpr int kNumSMs = 148;  // B200: 2 dies x 74 SMs

void set_error(const char* fmt, ...);
int fail(int status, const char* fmt, ...);

#define ADASK_CUDA(expr)                                                              \
  do {                                                                                \
    cudaError_t _e = (expr);                                                          \
    if (_e != cudaSuccess)                                                            \
      return ::adask::fail(ADASK_E_CUDA, "%s failed: %s (%s:%d)", #expr,              \
                           cudaGetErrorString(_e), __FILE__, __LINE__);               \
  } while (0)

#define ADASK_TRY(expr)          \
  do {                           \
    int _s = (expr);             \
    if (_s != ADASK_OK) return _s; \
  } while (0)

#define ADASK_LAUNCHED(ctx)                                                            \
  do {                                                                                 \
    cudaError_t _e = cudaGetLastError();                                               \
    if (_e != cudaSuccess)                                                             \
      return ::adask::fail(ADASK_E_CUDA, "kernel launch failed: %s (%s:%d)",           \
                           cudaGetErrorString(_e), __FILE__, __LINE__);                \
    (ctx)->launches++;                                                                 \
  } while (0)

// Grow-only device scratch buffer.  Growth synchronises the stream first so a
// buffer still in use by queued kernels is never freed under them.
struct Workspace {
  void* ptr = nullptr;
  size_t bytes = 0;
  // incremented on every (re)allocation: cudaMalloc may hand back the address
  // just freed, so a changed pointer does not detect a new (uninitialized) buffer
  unsigned gen = 0;
  int get(size_t need, cudaStream_t st, void** out) {
    if (need > bytes) {
      ++gen;
      if (ptr) {
        cudaError_t e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) return fail(ADASK_E_CUDA, "sync: %s", cudaGetErrorString(e));
        cudaFree(ptr);
        ptr = nullptr;
        bytes = 0;
      }
      size_t nb = need + need / 4 + 4096;
      cudaError_t e = cudaMalloc(&ptr, nb);
      if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(ADASK_E_NOMEM, "cudaMalloc(%zu) failed: %s", nb, cudaGetErrorString(e));
      }
      bytes = nb;
    }
    *out = ptr;
    return ADASK_OK;
  }
  void release() {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    bytes = 0;
  }
};

enum WsSlot {
  WS_HESS = 0,   // hess_mult per-CTA partial d-vectors
  WS_RNG,        // sign / bucket streams, rejection lists
  WS_SORT,       // SJLT counting-sort keys / values / CUB temp
  WS_SRHT,       // pruned FWHT intermediate
  WS_GAUSS,      // Gaussian S tiles
  WS_CHOL,       // factorization scratch
  WS_VEC,        // iteration-body scratch (scalars, temporaries)
  WS_SMALL,      // small host-visible-by-copy scalars
  WS_SIGNS,      // SRHT sign stream
  WS_PLAN,       // SRHT slot / entry plan
  WS_GEMM,       // split-K partials of gemm_impl
  WS_GEMV,       // partials of column GEMVs (precond apply)
  WS_GRAM,       // Gram / capacitance matrix being factored
  WS_APPLY,      // temporaries of the dense preconditioner apply
  WS_SA0,        // native driver: the current sketch SA (referenced by the live preconditioner)
  WS_SA1,        // native driver: the next sketch
  WS_SRHT_U,     // pipelined SRHT: the two half transforms of an 11-bit pass 2
  WS_GRAM_PACK,  // Gram: 16-byte aligned copy of an odd-shaped operand
  WS_GRAM_RL,    // Gram: 1/lam (Woodbury scaling), zero padded
  WS_CHOL_FLAGS, // dataflow Cholesky: ticket counter + per-tile flags
  WS_CHOL_ITEMS, // dataflow Cholesky: helper item list (per nblk)
  WS_PAIR,       // sharded PCG proposal: the partial pair [A^T A p | A^T A x]
  WS_SA_ROWS,    // sharded build: this rank's reduce-scattered rows of SA
  WS_SRHT_SYNC,  // fused SRHT: work ticket + per-group pass-1 counters (self-resetting)
  WS_CHECK,      // problem validation verdict flags
  WS_SRHT_PART,  // big-block SRHT: per-sub-block partial rows
  WS_SRHT_MAP,   // big-block SRHT: selected row -> partial row, high bits
  WS_COUNT
};

// Live per-unit timing (CUDA events on the launching stream), enabled by
// adask_prof_enable; used by bench.py for the roofline of the dominant unit.
enum ProfKind {
  PK_HESS = 0,   // fused A^T A pass (hess_mult)
  PK_SRHT,       // whole SRHT sketch
  PK_SJLT,       // whole SJLT sketch
  PK_GAUSS,      // whole Gaussian sketch
  PK_BUILD,      // preconditioner build (Gram + Cholesky + inverse)
  PK_APPLY,      // preconditioner apply
  PK_GRAM,       // build: the Gram / capacitance (inside PK_BUILD)
  PK_CHOL,       // build: Cholesky factor + triangular inverse (inside PK_BUILD)
  PK_COUNT
};

}  // namespace adask

struct adask_prof_rec {
  cudaEvent_t a, b;
  double bytes;
  double flops;
};

namespace adask {
// NCCL communicator of a row-sharded solve (comm.cu); nccl is an ncclComm_t
struct CommState {
  void* nccl = nullptr;
  int rank = 0, world = 1;
  bool owned = false;
};
}  // namespace adask

struct adask_ctx {
  int device = 0;
  adask::CommState comm;
  // dataflow Cholesky (chol_df.cu): flag block identity, epoch, ticket base
  unsigned chol_flags_gen = 0;  // Workspace::gen of the flag block last cleared
  int chol_epoch = 0;
  unsigned chol_ticket = 0;
  // dataflow Cholesky helper item lists, built and uploaded once per tile
  // count for the context's lifetime (the adaptive solves cycle through the
  // same sizes every solve): nblk -> {device list, items}
  std::vector<std::pair<void*, int>> chol_items;
  int64_t launches = 0;
  // fused SRHT counters: zeroed once per allocation, reset by each launch's last CTA
  unsigned srht_sync_gen = 0;   // Workspace::gen of the counter / map block last cleared
  int srht_epoch = 0;
  adask::Workspace ws[adask::WS_COUNT];
  double* pinned = nullptr;  // pinned host scalars for synchronous readbacks
  int* pinned_flags = nullptr;
  int prof = 0;
  std::vector<adask_prof_rec> prof_recs[adask::PK_COUNT];
  std::vector<cudaEvent_t> event_pool;
  // native driver: the Cholesky's pivot check is read at the driver's next
  // stream synchronization instead of a sync of its own (pinned_flags[1])
  bool defer_spd = false;
  // pinned staging ring for host -> device plan uploads (adask::upload_async)
  struct Stage {
    void* p = nullptr;
    size_t bytes = 0;
    cudaEvent_t ev = nullptr;
    bool pending = false;
  } stage[4];
  int stage_next = 0;
  // host-mapped mailbox of the iteration decrements: the last kernel of each
  // body writes delta_tilde / flags / a sequence number into pinned memory,
  // the host spins on the sequence number (no copy-engine D2H, no stream sync)
  void* mail = nullptr;
  uint32_t mail_seq = 0;
  // profiled pass only: pinned gate word [0] = released sequence, [1] = timeouts
  // (adask::prof_gate_hold; ADASK_PROF_GATE=0 turns the gate off)
  uint32_t* gate = nullptr;
  uint32_t gate_seq = 0;
};

namespace adask {
// Programmatic dependent launch: a kernel launched with launch_pdl may start
// (block scheduling, prologue) while its predecessor in the stream drains;
// pdl_wait() blocks until the predecessor has completed and its writes are
// visible.  Kernels that call pdl_wait() first are safe under either launch.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
bool pdl_enabled();
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args... args) {
  if (!pdl_enabled()) {
    kern<<<grid, block, smem, st>>>(args...);
    return cudaGetLastError();
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, (KArgs)args...);
}
// Host -> device copy through a ring of pinned staging buffers: stream
// ordered and asynchronous (a cudaMemcpyAsync from pageable memory first
// synchronizes the stream, so the host could not prepare the next block's
// plan while the GPU works on this one).
int upload_async(adask_ctx* ctx, void* dst, const void* src, size_t bytes, cudaStream_t st);
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device):
// the driver call costs microseconds of host time, and on the per-iteration
// path the GPU idles while the host issues the next kernel.
int ensure_smem_attr(const void* fn, int bytes);
// RAII timing scope for one unit; no-op unless profiling is enabled.
// Gate for a unit whose host side plans between its launches: a one-warp
// kernel holds the stream until the unit is fully enqueued (host release, or
// a 20 ms timeout), so the unit's event window holds its device work only,
// not host enqueue gaps after a decision sync left the stream empty.
int prof_gate_hold(adask_ctx* ctx, cudaStream_t st);
bool prof_gate_enabled();

struct ProfScope {
  adask_ctx* ctx;
  int kind;
  cudaStream_t st;
  adask_prof_rec rec{};
  bool on;
  bool gated = false;
  ProfScope(adask_ctx* c, int k, cudaStream_t s, double bytes, double flops = 0.0, bool gate = false)
      : ctx(c), kind(k), st(s), on(c && c->prof) {
    if (!on) return;
    rec.a = take();
    rec.b = take();
    rec.bytes = bytes;
    rec.flops = flops;
    if (gate && prof_gate_enabled()) gated = prof_gate_hold(ctx, st) == 0;
    cudaEventRecord(rec.a, st);
  }
  ~ProfScope() {
    if (!on) return;
    cudaEventRecord(rec.b, st);
    ctx->prof_recs[kind].push_back(rec);
    if (gated) __atomic_store_n(&ctx->gate[0], ctx->gate_seq, __ATOMIC_RELEASE);
  }
  cudaEvent_t take() {
    cudaEvent_t e;
    if (!ctx->event_pool.empty()) {
      e = ctx->event_pool.back();
      ctx->event_pool.pop_back();
    } else {
      cudaEventCreate(&e);
    }
    return e;
  }
};
}  // namespace adask

namespace adask {

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }
inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }
__host__ __device__ inline size_t align_up_dev(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Activate ctx's device for the calling thread.
int use_device(adask_ctx* ctx);

// ---------------------------------------------------------------- device utils
template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Reduce R (power of two <= 32) per-lane values across the warp with a
// recursive-halving exchange: R - 1 + 5 - log2(R) shuffles instead of 5R.
// Returns the warp total of row `r`, where r = warp_multi_row<R>(lane); every
// lane with (lane & (32/R - 1)) == 0 holds a distinct row.  Fixed order.
template <int R>
__device__ __forceinline__ int warp_multi_row(int lane) {
  int r = 0, bitpos = 4;
#pragma unroll
  for (int h = R; h > 1; h >>= 1) {
    r = (r << 1) | ((lane >> bitpos) & 1);
    --bitpos;
  }
  return r;
}
template <int R>
__device__ __forceinline__ double warp_multi_sum(double (&v)[R]) {
  const int lane = threadIdx.x & 31;
  int off = 16;
#pragma unroll
  for (int h = R; h > 1; h >>= 1) {
    const bool up = (lane & off) != 0;
#pragma unroll
    for (int j = 0; j < h / 2; ++j) {
      const double send = up ? v[j] : v[j + h / 2];
      const double keep = up ? v[j + h / 2] : v[j];
      v[j] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
    off >>= 1;
  }
  double t = v[0];
  for (; off > 0; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
  return t;
}

// Deterministic block reduction of one double (fixed tree, any blockDim that is
// a multiple of 32, <= 1024).  All threads get the result.
__device__ __forceinline__ double block_sum(double v, double* sh /*[32]*/) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double t = (lane < nw) ? sh[lane] : 0.0;
  t = warp_sum(t);
  return t;
}

}  // namespace adask
