// Native adaptive driver: adaptive_run (solvers.py:585-659) in C++.
//
// The accept / reject control flow, the thresholds c(alpha, rho) phi^ell
// (pow on doubles, as Python's float ** int), the converged floor, the cap and
// capped-retry rules and the derive_seed(seed, K) redraw chain follow the
// reference statement by statement; the Python implementation in solvers.py
// is the same logic and the tests compare both traces.  Running the loop
// natively removes the Python/ctypes round trips around every loop pass: what
// remains per pass is the device work plus one 64-byte readback of the new
// decrement.  Sketches (all families, row-sharded with global randomness),
// the preconditioner build and the fused iteration bodies are the libadask
// kernels; sharded problems all-reduce SA and A^T A x through the problem's
// allreduce hook.
#include <chrono>
#include <cmath>
#include <future>
#include <vector>

#include "common.cuh"
#include "comm.cuh"
#include "hessmult.cuh"

#include "precond.cuh"
#include "rng.cuh"
#include "sjlt.cuh"
#include "srht.cuh"

namespace adask {
int problem_hess(adask_ctx* ctx, const adask_problem* pb, const double* X, const double* B, double* out,
                 cudaStream_t st);
int pcg_propose_impl(adask_ctx* ctx, const adask_problem* pb, const adask_precond* P, const double* x,
                     const double* r, const double* p, const double* dt_col, double* Hp, double* x_new,
                     double* r_new, double* rt_new, double* dt_new, double* delta_tilde_host, double* hx_mb,
                     int* hx_ok, cudaStream_t st);
int pcg_restart_impl(adask_ctx* ctx, const adask_problem* pb, const adask_precond* P, const double* x,
                     double* r, double* rt, double* p, double* dt_col, double* delta_tilde_host,
                     const double* hx_mb, cudaStream_t st);
int ihs_restart_impl(adask_ctx* ctx, const adask_problem* pb, const adask_precond* P, const double* x, double* g,
                     double* v, double* delta_tilde_host, bool have_g, cudaStream_t st);

__global__ void k_sub(int64_t n, const double* a, const double* b, double* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = a[i] - b[i];
}

static void seed_words(uint64_t v, std::vector<uint32_t>& w) {
  w.clear();
  do {
    w.push_back((uint32_t)v);
    v >>= 32;
  } while (v);
}

static int gen_from_seed(uint64_t seed, adask_pcg64* g) {
  std::vector<uint32_t> w;
  seed_words(seed, w);
  return adask_pcg64_seed(w.data(), (int64_t)w.size(), g);
}

struct DevBuf {
  void* p = nullptr;
  cudaStream_t st = nullptr;
  int alloc(size_t bytes, cudaStream_t s) {
    st = s;
    ADASK_CUDA(cudaMallocAsync(&p, bytes ? bytes : 16, s));
    return ADASK_OK;
  }
  ~DevBuf() {
    if (p) cudaFreeAsync(p, st);
  }
};

// The SRHT's host index draw for the next potential resketch, computed on a
// worker thread while the device runs the current iterations (its inputs --
// the next size and seed -- are fixed in advance by the doubling rule).
struct IdxAhead {
  int64_t m = -1;
  uint64_t seed = 0;
  std::future<std::vector<int64_t>> fut;
  void start(uint64_t s, int64_t n, int64_t mm) {
    m = mm;
    seed = s;
    fut = std::async(std::launch::async, [s, n, mm]() {
      std::vector<int64_t> idx;
      adask_pcg64 g;
      if (gen_from_seed(s, &g) != ADASK_OK || srht_draw_idx(&g, n, mm, &idx) != ADASK_OK) idx.clear();
      return idx;
    });
  }
  // the precomputed draw if it matches (m, seed), else empty
  std::vector<int64_t> take(uint64_t s, int64_t mm) {
    std::vector<int64_t> r;
    if (fut.valid()) {
      r = fut.get();
      if (m != mm || seed != s) r.clear();
    }
    m = -1;
    return r;
  }
};

// SA (m x d, dtype) for the configured family at sketch seed `seed`.
static int make_sketch(adask_ctx* ctx, const adask_problem* pb, const adask_adaptive_cfg* cfg, int64_t m,
                       uint64_t seed, void* SA, cudaStream_t st, IdxAhead* ahead = nullptr) {
  const int64_t d = pb->d;
  const size_t esz = pb->dtype == ADASK_F64 ? 8 : 4;
  switch (cfg->family) {
    case ADASK_GAUSSIAN:
      ADASK_TRY(adask_sketch_gaussian(ctx, pb->dtype, pb->A, pb->n, d, pb->lda, cfg->row0, m, seed, SA, d,
                                      cfg->flags & ADASK_TF32, (void*)st));
      break;
    case ADASK_SRHT: {
      if (cfg->n_total != pb->n) return fail(ADASK_E_ARG, "the global SRHT does not shard (use block SRHT)");
      adask_pcg64 g;
      ADASK_TRY(gen_from_seed(seed, &g));
      std::vector<int64_t> pre;
      if (ahead) pre = ahead->take(seed, m);
      ADASK_TRY(sketch_srht_impl(ctx, pb->dtype, pb->A, pb->n, d, pb->lda, &g, m, SA, d, nullptr, 0, st,
                                 pre.empty() ? nullptr : &pre));
      break;
    }
    case ADASK_SRHT_BLOCK: {
      const int64_t B = cfg->block;
      if (B < 1 || cfg->row0 % B) return fail(ADASK_E_ARG, "block SRHT: shard must start on a block boundary");
      ADASK_CUDA(cudaMemsetAsync(SA, 0, (size_t)m * d * esz, st));
      for (int64_t r0 = 0; r0 < pb->n; r0 += B) {
        const int64_t rows = std::min<int64_t>(B, pb->n - r0);
        adask_pcg64 g;
        ADASK_TRY(gen_from_seed(adask_derive_seed(seed, (uint64_t)((cfg->row0 + r0) / B)), &g));
        const void* Ab = (const char*)pb->A + (size_t)r0 * pb->lda * esz;
        ADASK_TRY(sketch_srht_impl(ctx, pb->dtype, Ab, rows, d, pb->lda, &g, m, SA, d, nullptr,
                                   ADASK_ACCUMULATE, st));
      }
      break;
    }
    case ADASK_SJLT: {
      adask_pcg64 g;
      ADASK_TRY(gen_from_seed(seed, &g));
      std::vector<int64_t> rows;
      uint64_t sign_first = 0;
      if (cfg->s > 1) {
        if (cfg->row0 != 0 || cfg->n_total != pb->n)
          return fail(ADASK_E_ARG, "row-sharded SJLT with s > 1 is not supported");
        rows.resize((size_t)(pb->n * cfg->s));
        adask_pcg64 h = g;
        ADASK_TRY(adask_sjlt_rows(&h, pb->n, m, cfg->s, rows.data(), &sign_first));
      }
      ADASK_TRY(sketch_sjlt_impl(ctx, pb->dtype, pb->A, pb->n, d, pb->lda, cfg->row0, cfg->n_total, m,
                                 cfg->s, &g, rows.empty() ? nullptr : rows.data(), sign_first, SA, d, 0, st));
      break;
    }
    default:
      return fail(ADASK_E_ARG, "unknown sketch family %d", cfg->family);
  }
  return ADASK_OK;  // row-sharded: the partial S_g A_g (combined by build_precond)
}

// Preconditioner from a sketch.  One GPU: build(SA).  Row-sharded, dense path
// (m >= d) with m divisible by the world size: reduce-scatter the partial
// S_g A_g, Gram of this rank's m/G rows, all-reduce of the d x d Gram, then
// nu^2 Lam and the (replicated) factor.  Otherwise (Woodbury path: its apply
// reads all of SA; or SA already summed) all-reduce SA and build.
static int build_precond(adask_ctx* ctx, const adask_problem* pb, void* SA, int64_t m, bool sa_summed,
                         adask_precond** P, int64_t* info, cudaStream_t st) {
  const int64_t d = pb->d;
  const double nu = std::sqrt(pb->nu2);
  if (!problem_sharded(ctx, pb))
    return precond_build_impl(ctx, pb->dtype, SA, m, m, d, d, nu, pb->lam, nullptr, P, info, st);
  const int G = comm_world(ctx, pb);
  if (!sa_summed && m >= d && m % G == 0 && getenv("ADASK_SHARD_SA_ALLREDUCE") == nullptr) {
    const size_t esz = pb->dtype == ADASK_F64 ? 8 : 4;
    const int64_t mr = m / G;
    void* scratch = nullptr;
    ADASK_TRY(ctx->ws[WS_SA_ROWS].get((size_t)mr * d * esz, st, &scratch));
    void* rows = nullptr;
    ADASK_TRY(problem_reduce_scatter(ctx, pb, SA, scratch, mr * d, pb->dtype, &rows, st));
    GramReduce red = [&](void* M, int64_t count, int dt) { return problem_allreduce(ctx, pb, M, count, dt, st); };
    return precond_build_impl(ctx, pb->dtype, rows, mr, m, d, d, nu, pb->lam, &red, P, info, st);
  }
  if (!sa_summed) ADASK_TRY(problem_allreduce(ctx, pb, SA, m * d, pb->dtype, st));
  return precond_build_impl(ctx, pb->dtype, SA, m, m, d, d, nu, pb->lam, nullptr, P, info, st);
}

// ------------------------------------------------------------ incremental growth
// ADASK_INCREMENTAL: every sketch uses the seed of sketch 0 and the sketch
// grows instead of being redrawn when m doubles (north_star "incremental
// sketch growth"; not reference semantics, so the oracle has the same mode).
//   Gaussian: rows [0, m_old) are the previous SA rescaled by sqrt(m_old / m),
//             only rows [m_old, m) are generated and applied;
//   SRHT / block SRHT: the normalized transform Y = fwht(D A) / sqrt(n_pad)
//             of every block is computed once and kept; a sketch of any m is
//             the gather Y[perm[:m]] * sqrt(n_pad / m) (nested uniform subsets);
//   SJLT: redrawn as in the reference mode.
template <typename T>
__global__ void k_rescale_rows(const T* __restrict__ src, int64_t n, double s, T* __restrict__ dst) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = (T)((double)src[i] * s);
}

struct Incremental {
  bool on = false;
  // transforms of all blocks and draw orders: stream-ordered pool blocks
  // (not context workspaces) -- as large as A, released when the solve ends
  DevBuf ybuf, pbuf;
  void* y = nullptr;
  void* perm = nullptr;
  std::vector<int64_t> npad;  // per block
  std::vector<size_t> yoff, poff;
  bool ready = false;
};

static int make_sketch_incr(adask_ctx* ctx, const adask_problem* pb, const adask_adaptive_cfg* cfg, Incremental& inc,
                            int64_t m, const void* SA_old, int64_t m_old, void* SA, cudaStream_t st) {
  const int64_t d = pb->d;
  const size_t esz = pb->dtype == ADASK_F64 ? 8 : 4;
  const uint64_t seed0 = adask_derive_seed(cfg->seed, 0);
  if (cfg->family == ADASK_GAUSSIAN) {
    if (!SA_old || m_old <= 0) {
      ADASK_TRY(adask_sketch_gaussian(ctx, pb->dtype, pb->A, pb->n, d, pb->lda, cfg->row0, m, seed0, SA, d,
                                      cfg->flags & ADASK_TF32, (void*)st));
      return problem_allreduce(ctx, pb, SA, m * d, pb->dtype, st);
    }
    if (m == m_old) {  // capped retry: the grown sketch is the same sketch
      ADASK_CUDA(cudaMemcpyAsync(SA, SA_old, (size_t)m * d * esz, cudaMemcpyDeviceToDevice, st));
      return ADASK_OK;
    }
    const double sc = std::sqrt((double)m_old / (double)m);
    const int64_t nold = m_old * d;
    if (pb->dtype == ADASK_F64)
      k_rescale_rows<double><<<(unsigned)cdiv(nold, 256), 256, 0, st>>>((const double*)SA_old, nold, sc, (double*)SA);
    else
      k_rescale_rows<float><<<(unsigned)cdiv(nold, 256), 256, 0, st>>>((const float*)SA_old, nold, sc, (float*)SA);
    ADASK_LAUNCHED(ctx);
    void* fresh = (char*)SA + (size_t)nold * esz;
    ADASK_TRY(adask_sketch_gaussian_rows(ctx, pb->dtype, pb->A, pb->n, d, pb->lda, cfg->row0, m, m_old, m - m_old,
                                         seed0, fresh, d, cfg->flags & ADASK_TF32, (void*)st));
    return problem_allreduce(ctx, pb, fresh, (m - m_old) * d, pb->dtype, st);
  }
  if (cfg->family == ADASK_SRHT || cfg->family == ADASK_SRHT_BLOCK) {
    const bool blocked = cfg->family == ADASK_SRHT_BLOCK;
    const int64_t B = blocked ? cfg->block : pb->n;
    if (!blocked && cfg->n_total != pb->n) return fail(ADASK_E_ARG, "the global SRHT does not shard (use block SRHT)");
    if (blocked && (B < 1 || cfg->row0 % B)) return fail(ADASK_E_ARG, "block SRHT: shard must start on a block boundary");
    if (!inc.ready) {
      size_t ybytes = 0, pcount = 0;
      for (int64_t r0 = 0; r0 < pb->n; r0 += B) {
        const int64_t rows = std::min<int64_t>(B, pb->n - r0);
        const int64_t np = (int64_t)1 << (int)std::ceil(std::log2((double)std::max<int64_t>(rows, 1)));
        inc.npad.push_back(np);
        inc.yoff.push_back(ybytes);
        inc.poff.push_back(pcount);
        ybytes += (size_t)np * d * esz;
        pcount += (size_t)np;
      }
      ADASK_TRY(inc.ybuf.alloc(ybytes, st));
      ADASK_TRY(inc.pbuf.alloc(pcount * sizeof(int64_t), st));
      inc.y = inc.ybuf.p;
      inc.perm = inc.pbuf.p;
      std::vector<int64_t> perm;
      size_t bi = 0;
      for (int64_t r0 = 0; r0 < pb->n; r0 += B, ++bi) {
        const int64_t rows = std::min<int64_t>(B, pb->n - r0);
        adask_pcg64 g;
        ADASK_TRY(gen_from_seed(blocked ? adask_derive_seed(seed0, (uint64_t)((cfg->row0 + r0) / B)) : seed0, &g));
        perm.assign((size_t)inc.npad[bi], 0);
        const void* Ab = (const char*)pb->A + (size_t)r0 * pb->lda * esz;
        ADASK_TRY(srht_transform_impl(ctx, pb->dtype, Ab, rows, d, pb->lda, &g, (char*)inc.y + inc.yoff[bi],
                                      perm.data(), st));
        ADASK_CUDA(cudaMemcpyAsync((int64_t*)inc.perm + inc.poff[bi], perm.data(), perm.size() * sizeof(int64_t),
                                   cudaMemcpyHostToDevice, st));
        ADASK_CUDA(cudaStreamSynchronize(st));  // perm (pageable host) is reused by the next block
      }
      inc.ready = true;
    }
    for (size_t bi = 0; bi < inc.npad.size(); ++bi)
      ADASK_TRY(srht_gather_impl(ctx, pb->dtype, (char*)inc.y + inc.yoff[bi], inc.npad[bi], d,
                                 (const int64_t*)inc.perm + inc.poff[bi], m, SA, d, bi > 0 ? 1 : 0, st));
    return problem_allreduce(ctx, pb, SA, m * d, pb->dtype, st);
  }
  ADASK_TRY(make_sketch(ctx, pb, cfg, m, seed0, SA, st));  // SJLT: no growth rule, redraw
  return problem_allreduce(ctx, pb, SA, m * d, pb->dtype, st);
}

static int exact_err(adask_ctx* ctx, const adask_problem* pb, const double* x, const double* xstar,
                     double* diff, double* Hd, double* out, cudaStream_t st) {
  const int64_t n = pb->d * pb->c;
  k_sub<<<(unsigned)cdiv(n, 256), 256, 0, st>>>(n, x, xstar, diff);
  ADASK_LAUNCHED(ctx);
  ADASK_TRY(problem_hess(ctx, pb, diff, nullptr, Hd, st));
  return adask_dot(ctx, diff, Hd, pb->d, pb->c, pb->d, out, (void*)st);
}

}  // namespace adask

using namespace adask;

extern "C" int adask_adaptive_run(adask_ctx* ctx, const adask_problem* pb, const adask_adaptive_cfg* cfg,
                                  const double* x0, double* x_out, const double* xstar,
                                  adask_trace_rec* recs, int64_t max_recs, int64_t* n_recs, void* stream) {
  ADASK_TRY(use_device(ctx));
  if (!pb || !cfg || !x0 || !x_out || !recs || !n_recs) return fail(ADASK_E_ARG, "adaptive_run: null argument");
  if (!(cfg->rho > 0.0 && cfg->rho < 1.0)) return fail(ADASK_E_ARG, "rho must lie in (0, 1)");
  if (cfg->m_init < 1 || cfg->T < 0) return fail(ADASK_E_ARG, "bad m_init / T");
  cudaStream_t st = S(stream);
  const auto t_start = std::chrono::steady_clock::now();
  auto wall = [&]() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
  };
  const int64_t d = pb->d, c = pb->c, cd = c * d;
  const size_t esz = pb->dtype == ADASK_F64 ? 8 : 4;
  *n_recs = 0;
  // state buffers
  DevBuf vecs;
  ADASK_TRY(vecs.alloc((size_t)(13 * cd + 4 * c) * sizeof(double), st));
  double* base = (double*)vecs.p;
  double *x = base, *xn = base + cd, *a1 = base + 2 * cd, *a2 = base + 3 * cd, *a3 = base + 4 * cd;
  double *b1 = base + 5 * cd, *b2 = base + 6 * cd, *b3 = base + 7 * cd, *xp = base + 8 * cd;
  double *diff = base + 9 * cd, *Hd = base + 10 * cd, *Hp = base + 11 * cd;
  double *dtc = base + 12 * cd, *dtn = dtc + c;  // per-column r.rt (current / proposed)
  double* hxc = dtn + c;  // PCG: H x - B at the current iterate, from the proposal's fused pass
  ADASK_CUDA(cudaMemcpyAsync(x, x0, cd * sizeof(double), cudaMemcpyDeviceToDevice, st));

  const int64_t n_pad_total = (int64_t)1 << (int)std::ceil(std::log2((double)std::max<int64_t>(cfg->n_total, 1)));
  int64_t cap = cfg->family == ADASK_SRHT ? n_pad_total : cfg->n_total;
  if (cfg->family == ADASK_SRHT_BLOCK) {
    // each block sketch needs m <= padded block rows
    const int64_t b = std::min(cfg->block, cfg->n_total);
    const int64_t bpad = (int64_t)1 << (int)std::ceil(std::log2((double)std::max<int64_t>(b, 1)));
    cap = std::min(cap, bpad);
  }
  int64_t m = std::min(cfg->m_init, cap);
  int64_t K = 0;
  auto record = [&](int64_t t, int64_t mm, int64_t k, double dt, const double* xs, int ev) -> int {
    if (*n_recs >= max_recs) return fail(ADASK_E_ARG, "trace buffer too small");
    adask_trace_rec& r = recs[*n_recs];
    r.t = t;
    r.m = mm;
    r.k = k;
    r.delta_tilde = dt;
    r.delta_exact = NAN;
    r.has_exact = 0;
    if (xstar) {
      ADASK_TRY(exact_err(ctx, pb, xs, xstar, diff, Hd, &r.delta_exact, st));
      r.has_exact = 1;
    }
    r.wall_seconds = wall();
    r.event = ev;
    ++*n_recs;
    return ADASK_OK;
  };

  // Cholesky pivot checks are read after each restart's synchronization (the
  // reference raises NotPositiveDefinite from build; reported here before any
  // error the restart itself may raise from the unusable factor)
  struct DeferGuard {
    adask_ctx* c;
    bool old;
    ~DeferGuard() { c->defer_spd = old; }
  } dguard{ctx, ctx->defer_spd};
  ctx->defer_spd = getenv("ADASK_NO_DEFER_SPD") == nullptr;
  ctx->pinned_flags[1] = 0;
  auto spd_check = [&]() -> int {
    const int h = ctx->pinned_flags[1];
    if (h != 0) {
      ctx->pinned_flags[1] = 0;
      return fail(ADASK_E_NOT_SPD, "Matrix is not positive definite (leading minor %d)", h);
    }
    return ADASK_OK;
  };

  // sketch + build
  // SA buffers: two grow-only context workspaces (the live preconditioner
  // references the current one; the next sketch goes to the other), so
  // repeated solves allocate nothing once the largest sketch has been seen
  struct SaBuf {
    void* p = nullptr;
  } sa_buf;
  int sa_slot = WS_SA0;
  ADASK_TRY(ctx->ws[sa_slot].get((size_t)m * d * esz, st, &sa_buf.p));
  Incremental inc;
  inc.on = (cfg->flags & ADASK_INCREMENTAL) != 0;
  if (inc.on)
    ADASK_TRY(make_sketch_incr(ctx, pb, cfg, inc, m, nullptr, 0, sa_buf.p, st));
  else
    ADASK_TRY(make_sketch(ctx, pb, cfg, m, adask_derive_seed(cfg->seed, 0), sa_buf.p, st));
  IdxAhead ahead;
  const bool ahead_on = cfg->family == ADASK_SRHT && !inc.on && getenv("ADASK_NO_IDX_AHEAD") == nullptr;
  if (ahead_on) ahead.start(adask_derive_seed(cfg->seed, 1), pb->n, std::min(2 * m, cap));
  adask_precond* P = nullptr;
  int64_t info = 0;
  ADASK_TRY(build_precond(ctx, pb, sa_buf.p, m, inc.on, &P, &info, st));
  struct PGuard {
    adask_precond** p;
    ~PGuard() {
      if (*p) adask_precond_destroy(*p);
    }
  } pguard{&P};

  const bool pcg = cfg->method == ADASK_METHOD_PCG;
  const bool polyak = cfg->method == ADASK_METHOD_POLYAK;
  double mu = 1.0 - cfg->rho, beta = 0.0;
  if (polyak) {
    const double root = std::sqrt(1.0 - cfg->rho);
    mu = 2.0 * (1.0 - cfg->rho) / (1.0 + root);
    beta = (1.0 - root) / (1.0 + root);
  }
  // PCG: a1 = r, a2 = rt, a3 = p ; b1 = r_new, b2 = rt_new ; IHS: a1 = g, a2 = v, b1 = g_new, b2 = v_new
  double delta = 0.0;
  // Restarts after a resketch reuse H x - B at the unchanged iterate: IHS from
  // its gradient buffer, PCG from the proposal's two-column pass (hx_ok).
  // Both are the values the reference's recomputation gives, bit for bit.
  int hx_ok = 0;
  bool g_ok = false;
  const bool reuse = getenv("ADASK_NO_RESTART_REUSE") == nullptr;
  auto restart = [&]() -> int {
    if (pcg) return pcg_restart_impl(ctx, pb, P, x, a1, a2, a3, dtc, &delta, reuse && hx_ok ? hxc : nullptr, st);
    ADASK_TRY(ihs_restart_impl(ctx, pb, P, x, a1, a2, &delta, reuse && g_ok, st));
    g_ok = true;
    if (polyak) ADASK_CUDA(cudaMemcpyAsync(xp, x, cd * sizeof(double), cudaMemcpyDeviceToDevice, st));
    return ADASK_OK;
  };
  {
    const int rs = restart();
    ADASK_TRY(spd_check());
    ADASK_TRY(rs);
  }
  const double dt_first = delta;
  double dt_I = delta;
  int64_t t = 0, I = 0;
  bool capped_retry = false;
  ADASK_TRY(record(0, m, 0, delta, x, ADASK_EV_PLAIN));
  while (t < cfg->T) {
    double dnew = 0.0;
    if (pcg)
      ADASK_TRY(pcg_propose_impl(ctx, pb, P, x, a1, a3, dtc, Hp, xn, b1, b2, dtn, &dnew, reuse ? hxc : nullptr,
                                 &hx_ok, st));
    else
      ADASK_TRY(adask_ihs_propose(ctx, pb, P, x, a2, mu, polyak ? xp : nullptr, beta, xn, b1, b2, &dnew,
                                  (void*)st));
    const int64_t ell = t + 1 - I;
    const double threshold = cfg->c_alpha_rho * std::pow(cfg->phi_rho, (double)ell);
    const bool converged = dt_I <= 0.0 || dnew <= 1e-26 * dt_first;
    bool reject = (!converged) && dnew > threshold * dt_I;
    if (reject && capped_retry) reject = false;  // m already at cap and one redraw failed: accept
    if (reject) {
      K += 1;
      const bool at_cap = m >= cap;
      const int64_t m_old = m;
      m = std::min(2 * m, cap);
      capped_retry = at_cap;
      adask_precond_destroy(P);
      P = nullptr;
      const int nslot = sa_slot == WS_SA0 ? WS_SA1 : WS_SA0;
      SaBuf nsa;
      ADASK_TRY(ctx->ws[nslot].get((size_t)m * d * esz, st, &nsa.p));
      if (inc.on)
        ADASK_TRY(make_sketch_incr(ctx, pb, cfg, inc, m, sa_buf.p, m_old, nsa.p, st));
      else
        ADASK_TRY(make_sketch(ctx, pb, cfg, m, adask_derive_seed(cfg->seed, (uint64_t)K), nsa.p, st,
                              ahead_on ? &ahead : nullptr));
      if (ahead_on) ahead.start(adask_derive_seed(cfg->seed, (uint64_t)K + 1), pb->n, std::min(2 * m, cap));
      std::swap(sa_buf.p, nsa.p);
      sa_slot = nslot;
      ADASK_TRY(build_precond(ctx, pb, sa_buf.p, m, inc.on, &P, &info, st));
      {
        const int rs = restart();
        ADASK_TRY(spd_check());
        ADASK_TRY(rs);
      }
      dt_I = delta;
      I = t;
      ADASK_TRY(record(t, m, K, dt_I, x, ADASK_EV_RESKETCH));
    } else {
      if (pcg) {
        // commit: p = rt_new + p * (dt_new / dt_old), then rotate the buffers
        ADASK_TRY(adask_pcg_commit(ctx, d, c, b2, dtn, dtc, a3, (void*)st));
        std::swap(x, xn);
        std::swap(a1, b1);
        std::swap(a2, b2);
        std::swap(dtc, dtn);
      } else {
        if (polyak) {
          std::swap(xp, x);  // x_prev <- x
          std::swap(x, xn);  // x <- x_new (xn now holds the stale x_prev: scratch)
        } else {
          std::swap(x, xn);
        }
        std::swap(a1, b1);
        std::swap(a2, b2);
      }
      delta = dnew;
      t += 1;
      capped_retry = false;
      ADASK_TRY(record(t, m, K, delta, x, ADASK_EV_ACCEPTED));
    }
  }
  ADASK_CUDA(cudaMemcpyAsync(x_out, x, cd * sizeof(double), cudaMemcpyDeviceToDevice, st));
  ADASK_CUDA(cudaStreamSynchronize(st));
  return ADASK_OK;
}
