#include <map>
#include <mutex>
// Host side of libadask: error state, device context, and the numpy-exact
// seeding / PCG64 / bounded-integer / choice bookkeeping that decides which
// rows a sketch touches.  None of this is floating-point compute: it is the
// integer bookkeeping the reference delegates to numpy's Generator
// (embeddings.py:56-58 SeedSequence, :95-100 integers + choice, :117-124).
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "comm.cuh"
#include "gemm.cuh"
#include "pcg64.cuh"

namespace adask {

static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int fail(int status, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return status;
}

int use_device(adask_ctx* ctx) {
  if (!ctx) return fail(ADASK_E_ARG, "null context");
  int cur = -1;
  cudaError_t e = cudaGetDevice(&cur);
  if (e != cudaSuccess) return fail(ADASK_E_CUDA, "cudaGetDevice: %s", cudaGetErrorString(e));
  if (cur != ctx->device) ADASK_CUDA(cudaSetDevice(ctx->device));
  return ADASK_OK;
}

// ------------------------------------------------------------ SeedSequence
// numpy.random.SeedSequence (bit_generator.pyx): pool of 4 uint32 words,
// hashmix / mix of the entropy, then generate_state.
namespace ss {
constexpr uint32_t INIT_A = 0x43b0d7e5u, MULT_A = 0x931e8875u;
constexpr uint32_t INIT_B = 0x8b51f9ddu, MULT_B = 0x58f38dedu;
constexpr uint32_t MIX_MULT_L = 0xca01f9ddu, MIX_MULT_R = 0x4973f715u;
constexpr int POOL = 4;

static inline uint32_t hashmix(uint32_t v, uint32_t& hc) {
  v ^= hc;
  hc *= MULT_A;
  v *= hc;
  v ^= v >> 16;
  return v;
}
static inline uint32_t mix(uint32_t x, uint32_t y) {
  uint32_t r = MIX_MULT_L * x - MIX_MULT_R * y;
  r ^= r >> 16;
  return r;
}
static void pool_from_entropy(const uint32_t* ent, int64_t n, uint32_t pool[POOL]) {
  uint32_t hc = INIT_A;
  for (int i = 0; i < POOL; ++i) pool[i] = hashmix(i < n ? ent[i] : 0u, hc);
  for (int s = 0; s < POOL; ++s)
    for (int d = 0; d < POOL; ++d)
      if (s != d) pool[d] = mix(pool[d], hashmix(pool[s], hc));
  for (int64_t s = POOL; s < n; ++s)
    for (int d = 0; d < POOL; ++d) pool[d] = mix(pool[d], hashmix(ent[s], hc));
}
static void generate(const uint32_t pool[POOL], uint32_t* out, int64_t n_words) {
  uint32_t hc = INIT_B;
  for (int64_t i = 0; i < n_words; ++i) {
    uint32_t v = pool[i % POOL];
    v ^= hc;
    hc *= MULT_B;
    v *= hc;
    v ^= v >> 16;
    out[i] = v;
  }
}
}  // namespace ss

static inline int push_words(uint64_t v, uint32_t* w) {
  // numpy _int_to_uint32_array: little-endian 32-bit words, at least one.
  int n = 0;
  do {
    w[n++] = (uint32_t)v;
    v >>= 32;
  } while (v);
  return n;
}

// Host generator with numpy's next_uint32 buffering.
struct HostGen {
  u128 st, inc;
  bool has;
  uint32_t buf;
  uint64_t draws = 0;  // 32-bit draws consumed (next32 calls)
  explicit HostGen(const adask_pcg64& g)
      : st{g.state_hi, g.state_lo}, inc{g.inc_hi, g.inc_lo}, has(g.has_uint32 != 0), buf(g.uinteger) {}
  void store(adask_pcg64* g) const {
    g->state_hi = st.hi;
    g->state_lo = st.lo;
    g->inc_hi = inc.hi;
    g->inc_lo = inc.lo;
    g->has_uint32 = has ? 1 : 0;
    g->uinteger = buf;
  }
  uint64_t next64() {
    st = pcg_step(st, inc);
    return pcg_output(st);
  }
  uint32_t next32() {
    ++draws;
    if (has) {
      has = false;
      return buf;
    }
    uint64_t v = next64();
    has = true;
    buf = (uint32_t)(v >> 32);
    return (uint32_t)v;
  }
  // random_bounded_uint64(.., off=0, rng, mask=0, use_masked=false) for rng < 2^32-1
  uint32_t bounded(uint32_t rng) {
    if (rng == 0) return 0;
    if (rng == 0xFFFFFFFFu) return next32();
    const uint32_t ex = rng + 1;
    uint64_t m = (uint64_t)next32() * ex;
    uint32_t left = (uint32_t)m;
    if (left < ex) {
      const uint32_t thr = (uint32_t)(0u - ex) % ex;
      while (left < thr) {
        m = (uint64_t)next32() * ex;
        left = (uint32_t)m;
      }
    }
    return (uint32_t)(m >> 32);
  }
};

}  // namespace adask

using namespace adask;

extern "C" {

const char* adask_last_error(void) { return g_err; }
int adask_version(void) { return 1; }

int adask_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int adask_seedseq_generate(const uint32_t* entropy, int64_t n_entropy, uint32_t* out_words,
                           int64_t n_words) {
  if ((n_entropy > 0 && !entropy) || n_entropy < 0 || n_words < 0 || (n_words > 0 && !out_words))
    return fail(ADASK_E_ARG, "seedseq_generate: bad arguments");
  uint32_t pool[ss::POOL];
  ss::pool_from_entropy(entropy, n_entropy, pool);
  ss::generate(pool, out_words, n_words);
  return ADASK_OK;
}

uint64_t adask_derive_seed(uint64_t base, uint64_t k) {
  uint32_t ent[4];
  int n = push_words(base, ent);
  n += push_words(k, ent + n);
  uint32_t out[2];
  adask_seedseq_generate(ent, n, out, 2);
  return (uint64_t)out[0] | ((uint64_t)out[1] << 32);
}

int adask_pcg64_seed(const uint32_t* entropy, int64_t n_entropy, adask_pcg64* g) {
  if (!g) return fail(ADASK_E_ARG, "pcg64_seed: null generator");
  // PCG64._seed_seq: generate_state(4, uint64) -> seed = (v0 << 64) | v1,
  // inc = (v2 << 64) | v3; pcg64_srandom_r: inc = (inc << 1) | 1, state = 0,
  // step, state += seed, step.
  uint32_t w[8];
  ADASK_TRY(adask_seedseq_generate(entropy, n_entropy, w, 8));
  uint64_t v[4];
  for (int i = 0; i < 4; ++i) v[i] = (uint64_t)w[2 * i] | ((uint64_t)w[2 * i + 1] << 32);
  u128 seed{v[0], v[1]}, inc{v[2], v[3]};
  inc = u128{(inc.hi << 1) | (inc.lo >> 63), (inc.lo << 1) | 1u};
  u128 st{0, 0};
  st = pcg_step(st, inc);
  st = add128(st, seed);
  st = pcg_step(st, inc);
  g->state_hi = st.hi;
  g->state_lo = st.lo;
  g->inc_hi = inc.hi;
  g->inc_lo = inc.lo;
  g->has_uint32 = 0;
  g->uinteger = 0;
  return ADASK_OK;
}

int adask_pcg64_advance(adask_pcg64* g, uint64_t n_u64) {
  if (!g) return fail(ADASK_E_ARG, "null generator");
  u128 st{g->state_hi, g->state_lo}, inc{g->inc_hi, g->inc_lo};
  st = pcg_jump(st, inc, n_u64);
  g->state_hi = st.hi;
  g->state_lo = st.lo;
  return ADASK_OK;
}

int adask_pcg64_skip_u32(adask_pcg64* g, uint64_t n) {
  if (!g) return fail(ADASK_E_ARG, "null generator");
  if (n == 0) return ADASK_OK;
  if (g->has_uint32) {
    g->has_uint32 = 0;
    --n;
  }
  adask_pcg64_advance(g, n / 2);
  if (n & 1) {
    HostGen h(*g);
    uint64_t r = h.next64();
    h.has = true;
    h.buf = (uint32_t)(r >> 32);
    h.store(g);
  }
  return ADASK_OK;
}

uint64_t adask_pcg64_next_u64(adask_pcg64* g) {
  HostGen h(*g);
  uint64_t v = h.next64();
  h.store(g);
  return v;
}

uint32_t adask_pcg64_next_u32(adask_pcg64* g) {
  HostGen h(*g);
  uint32_t v = h.next32();
  h.store(g);
  return v;
}

uint32_t adask_pcg64_bounded_u32(adask_pcg64* g, uint32_t rng) {
  HostGen h(*g);
  uint32_t v = h.bounded(rng);
  h.store(g);
  return v;
}

int adask_pcg64_integers_host(adask_pcg64* g, uint32_t m, int64_t count, int64_t* out) {
  if (!g || m == 0 || count < 0 || (count > 0 && !out))
    return fail(ADASK_E_ARG, "integers_host: bad arguments");
  HostGen h(*g);
  for (int64_t i = 0; i < count; ++i) out[i] = (int64_t)h.bounded(m - 1);
  h.store(g);
  return ADASK_OK;
}

// Generator.choice(N, m, replace=False, shuffle=True) for N < 2^32
// (numpy _generator.pyx): tail shuffle when N > 10000 and m > N // 50,
// otherwise Floyd's algorithm with a linear-probe hash set followed by a
// Fisher-Yates shuffle of the m picks.
static void choice_impl(HostGen& h, int64_t N, int64_t m, int64_t* out) {
  if (m == 0) return;
  if (N > 10000 && m > N / 50) {
    std::vector<int64_t> a((size_t)N);
    for (int64_t i = 0; i < N; ++i) a[(size_t)i] = i;
    int64_t first = N - m > 1 ? N - m : 1;
    for (int64_t i = N - 1; i >= first; --i) {
      int64_t j = (int64_t)h.bounded((uint32_t)i);
      int64_t t = a[(size_t)j];
      a[(size_t)j] = a[(size_t)i];
      a[(size_t)i] = t;
    }
    std::memcpy(out, a.data() + (N - m), (size_t)m * sizeof(int64_t));
  } else {
    uint64_t mask = (uint64_t)(1.2 * (double)m);
    // _gen_mask: smallest all-ones mask >= max
    mask |= mask >> 1;
    mask |= mask >> 2;
    mask |= mask >> 4;
    mask |= mask >> 8;
    mask |= mask >> 16;
    mask |= mask >> 32;
    const uint64_t EMPTY = ~0ull;
    std::vector<uint64_t> hs((size_t)(mask + 1), EMPTY);
    for (int64_t j = N - m; j < N; ++j) {
      uint64_t val = h.bounded((uint32_t)j);
      uint64_t loc = val & mask;
      while (hs[loc] != EMPTY && hs[loc] != val) loc = (loc + 1) & mask;
      if (hs[loc] == EMPTY) {
        hs[loc] = val;
        out[j - N + m] = (int64_t)val;
      } else {
        loc = (uint64_t)j & mask;
        while (hs[loc] != EMPTY) loc = (loc + 1) & mask;
        hs[loc] = (uint64_t)j;
        out[j - N + m] = j;
      }
    }
    for (int64_t i = m - 1; i >= 1; --i) {
      int64_t j = (int64_t)h.bounded((uint32_t)i);
      int64_t t = out[j];
      out[j] = out[i];
      out[i] = t;
    }
  }
}

int adask_choice_noreplace(adask_pcg64* g, int64_t N, int64_t m, int64_t* out) {
  if (!g || N < 0 || m < 0 || m > N || (m > 0 && !out))
    return fail(ADASK_E_ARG, "choice: need 0 <= m <= N");
  if (N > 0xFFFFFFFFll) return fail(ADASK_E_ARG, "choice: population >= 2^32 unsupported");
  HostGen h(*g);
  choice_impl(h, N, m, out);
  h.store(g);
  return ADASK_OK;
}

// SJLT row picks for s > 1 (embeddings.py:121-123): rows[j*s:(j+1)*s] =
// choice(m, s, replace=False) for j = 0..n-1; *draws = 32-bit draws consumed.
int adask_sjlt_rows(adask_pcg64* g, int64_t n, int64_t m, int64_t s, int64_t* rows, uint64_t* draws) {
  if (!g || n < 0 || s < 1 || s > m || (n > 0 && !rows)) return fail(ADASK_E_ARG, "sjlt_rows: bad arguments");
  if (m > 0xFFFFFFFFll) return fail(ADASK_E_ARG, "sjlt_rows: m >= 2^32 unsupported");
  HostGen h(*g);
  for (int64_t j = 0; j < n; ++j) choice_impl(h, m, s, rows + j * s);
  h.store(g);
  if (draws) *draws = h.draws;
  return ADASK_OK;
}

int adask_ctx_create(int device, adask_ctx** out) {
  if (!out) return fail(ADASK_E_ARG, "null out");
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    cudaGetLastError();
    return fail(ADASK_E_CUDA, "no CUDA device available (%s)", cudaGetErrorString(e));
  }
  if (device < 0 || device >= n) return fail(ADASK_E_ARG, "device %d out of range", device);
  ADASK_CUDA(cudaSetDevice(device));
  // Keep freed stream-ordered allocations in the device's default pool (the
  // solver allocates and frees preconditioners / sketches every resketch).
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t thr = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  cudaGetLastError();
  adask_ctx* c = new adask_ctx();
  c->device = device;
  e = cudaMallocHost(&c->pinned, 64 * sizeof(double));
  if (e != cudaSuccess) {
    delete c;
    return fail(ADASK_E_CUDA, "cudaMallocHost: %s", cudaGetErrorString(e));
  }
  e = cudaMallocHost(&c->pinned_flags, 64 * sizeof(int));
  if (e != cudaSuccess) {
    cudaFreeHost(c->pinned);
    delete c;
    return fail(ADASK_E_CUDA, "cudaMallocHost: %s", cudaGetErrorString(e));
  }
  *out = c;
  return ADASK_OK;
}

int adask_ctx_destroy(adask_ctx* ctx) {
  if (!ctx) return ADASK_OK;
  cudaSetDevice(ctx->device);
  cudaDeviceSynchronize();
  for (auto& w : ctx->ws) w.release();
  for (auto& it : ctx->chol_items)
    if (it.first) cudaFree(it.first);
  adask::comm_release(ctx);
  if (ctx->pinned) cudaFreeHost(ctx->pinned);
  if (ctx->pinned_flags) cudaFreeHost(ctx->pinned_flags);
  if (ctx->mail) cudaFreeHost(ctx->mail);
  if (ctx->gate) cudaFreeHost(ctx->gate);
  for (auto& b : ctx->stage) {
    if (b.ev) {
      cudaEventSynchronize(b.ev);
      cudaEventDestroy(b.ev);
    }
    if (b.p) cudaFreeHost(b.p);
  }
  delete ctx;
  return ADASK_OK;
}

int64_t adask_ctx_launches(const adask_ctx* ctx) { return ctx ? ctx->launches : -1; }

}  // extern "C"

namespace adask {
int upload_async(adask_ctx* ctx, void* dst, const void* src, size_t bytes, cudaStream_t st) {
  if (bytes == 0) return ADASK_OK;
  adask_ctx::Stage& b = ctx->stage[ctx->stage_next];
  ctx->stage_next = (ctx->stage_next + 1) % 4;
  if (b.pending) {
    ADASK_CUDA(cudaEventSynchronize(b.ev));  // its previous copy has been consumed
    b.pending = false;
  }
  if (b.bytes < bytes) {
    if (b.p) cudaFreeHost(b.p);
    b.p = nullptr;
    b.bytes = 0;
    const size_t nb = std::max<size_t>(bytes + bytes / 4, 64 * 1024);
    ADASK_CUDA(cudaMallocHost(&b.p, nb));
    b.bytes = nb;
  }
  if (!b.ev) ADASK_CUDA(cudaEventCreateWithFlags(&b.ev, cudaEventDisableTiming));
  memcpy(b.p, src, bytes);
  ADASK_CUDA(cudaMemcpyAsync(dst, b.p, bytes, cudaMemcpyHostToDevice, st));
  ADASK_CUDA(cudaEventRecord(b.ev, st));
  b.pending = true;
  return ADASK_OK;
}

__global__ void k_prof_gate(volatile uint32_t* g, uint32_t seq, unsigned long long timeout_ns) {
  if (threadIdx.x != 0) return;
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
  while ((int32_t)(g[0] - seq) < 0) {
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    if (t - t0 > timeout_ns) {
      g[1] = g[1] + 1;
      break;
    }
    __nanosleep(256);
  }
}

bool prof_gate_enabled() {
  static const bool on = !(getenv("ADASK_PROF_GATE") && atoi(getenv("ADASK_PROF_GATE")) == 0);
  return on;
}

int prof_gate_hold(adask_ctx* ctx, cudaStream_t st) {
  if (!ctx->gate) {
    void* p = nullptr;
    if (cudaMallocHost(&p, 64) != cudaSuccess) {
      cudaGetLastError();
      return ADASK_E_CUDA;
    }
    memset(p, 0, 64);
    ctx->gate = (uint32_t*)p;
    ctx->gate_seq = 0;
  }
  ++ctx->gate_seq;
  k_prof_gate<<<1, 32, 0, st>>>(ctx->gate, ctx->gate_seq, 20000000ull);
  if (cudaGetLastError() != cudaSuccess) {
    __atomic_store_n(&ctx->gate[0], ctx->gate_seq, __ATOMIC_RELEASE);
    return ADASK_E_CUDA;
  }
  return ADASK_OK;
}

bool pdl_enabled() {
  static const bool on = getenv("ADASK_NO_PDL") == nullptr;
  return on;
}
int ensure_smem_attr(const void* fn, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  int& have = done[{fn, dev}];
  if (have >= bytes) return ADASK_OK;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) return fail(ADASK_E_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
  have = bytes;
  return ADASK_OK;
}
}  // namespace adask

extern "C" int adask_prof_enable(adask_ctx* ctx, int on) {
  if (!ctx) return fail(ADASK_E_ARG, "null context");
  ctx->prof = on ? 1 : 0;
  if (on) {
    // create the timing events up front: a cudaEventCreate inside a timed
    // region costs microseconds of host time per unit
    cudaSetDevice(ctx->device);
    size_t live = 0;
    for (auto& v : ctx->prof_recs) live += 2 * v.size();
    while (ctx->event_pool.size() + live < 8192) {
      cudaEvent_t e;
      if (cudaEventCreate(&e) != cudaSuccess) {
        cudaGetLastError();
        break;
      }
      ctx->event_pool.push_back(e);
    }
  }
  return ADASK_OK;
}

extern "C" int adask_prof_reset(adask_ctx* ctx) {
  if (!ctx) return fail(ADASK_E_ARG, "null context");
  cudaSetDevice(ctx->device);
  for (auto& v : ctx->prof_recs) {
    for (auto& r : v) {
      ctx->event_pool.push_back(r.a);
      ctx->event_pool.push_back(r.b);
    }
    v.clear();
  }
  return ADASK_OK;
}

// Totals for one unit kind since the last reset (synchronises the device).
extern "C" int adask_prof_query(adask_ctx* ctx, int kind, int64_t* count, double* total_ms,
                                double* total_bytes, double* total_flops) {
  if (!ctx || kind < 0 || kind >= PK_COUNT) return fail(ADASK_E_ARG, "prof_query: bad arguments");
  ADASK_CUDA(cudaSetDevice(ctx->device));
  ADASK_CUDA(cudaDeviceSynchronize());
  double ms = 0, by = 0, fl = 0;
  for (auto& r : ctx->prof_recs[kind]) {
    float t = 0;
    ADASK_CUDA(cudaEventElapsedTime(&t, r.a, r.b));
    ms += t;
    by += r.bytes;
    fl += r.flops;
  }
  if (count) *count = (int64_t)ctx->prof_recs[kind].size();
  if (total_ms) *total_ms = ms;
  if (total_bytes) *total_bytes = by;
  if (total_flops) *total_flops = fl;
  return ADASK_OK;
}
