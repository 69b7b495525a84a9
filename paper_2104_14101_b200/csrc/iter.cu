// Fused iteration bodies of the sketched solvers.
// reference: solvers.py:227-282 (_PcgState), :522-571 (_IhsState, _PolyakState).
//
// Each body is: one fused A^T A pass (hessmult.cu), one single-CTA d-vector
// kernel (dots, step sizes, axpys, guards), one preconditioner apply, one
// single-CTA reduction kernel, and one 64-byte device->host readback of the
// decrement plus guard flags -- the single host synchronisation the adaptive
// accept/reject rule needs per loop pass.  All reductions are fixed-order
// (bitwise reproducible).
#include <atomic>
#include <chrono>
#include <cstring>

#include "common.cuh"
#include "comm.cuh"
#include "hessmult.cuh"
#include "precond.cuh"

namespace adask {

enum { FLAG_NEGATIVE = 1, FLAG_BREAKDOWN = 2 };

struct IterScalars {
  double delta_tilde;
  double pad[3];
  int flags;
  int pad2[7];
};

struct IterMail {
  double delta_tilde;
  int flags;
  uint32_t seq;
};

// thread 0, after writing sc: the host-visible copy, then the sequence number
__device__ __forceinline__ void publish(const IterScalars* sc, IterMail* mail, uint32_t seq) {
  if (!mail) return;
  mail->delta_tilde = sc->delta_tilde;
  mail->flags = sc->flags;
  __threadfence_system();
  *reinterpret_cast<volatile uint32_t*>(&mail->seq) = seq;
}

constexpr int kVecThreads = 1024;

// Fixed-order block sum (kVecThreads threads).
__device__ __forceinline__ double blk_sum(double v, double* sh) { return block_sum(v, sh); }

// PCG restart tail: r = -g (g = H x - B); p = rt; dt_col = max(colsum(r*rt),0)
// with the NegativeValue guard (solvers.py:245-255).
__global__ void __launch_bounds__(kVecThreads) k_pcg_restart_tail(int64_t d, int64_t c, const double* rt,
                                                                  double* r, double* p, double* dt_col,
                                                                  IterScalars* sc, IterMail* mail, uint32_t seq) {
  pdl_wait();
  __shared__ double sh[32];
  double tot = 0.0;
  int flags = 0;
  for (int64_t j = 0; j < c; ++j) {
    double s = 0.0, q = 0.0;
    for (int64_t i = threadIdx.x; i < d; i += blockDim.x) {
      double rv = r[j * d + i];
      double tv = rt[j * d + i];
      s = fma(rv, tv, s);
      q = fma(rv, rv, q);
      p[j * d + i] = tv;
    }
    s = blk_sum(s, sh);
    q = blk_sum(q, sh);
    if (s < -1e-12 * q) flags |= FLAG_NEGATIVE;
    double dt = s > 0.0 ? s : 0.0;
    if (threadIdx.x == 0) dt_col[j] = dt;
    tot += dt;
  }
  if (threadIdx.x == 0) {
    sc->delta_tilde = 0.5 * tot;
    sc->flags = flags;
    publish(sc, mail, seq);
  }
}

__global__ void k_negate(double* v, int64_t n) {
  pdl_wait();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = -v[i];
}

// PCG propose, first half (solvers.py:265-272)
__global__ void __launch_bounds__(kVecThreads) k_pcg_step(int64_t d, int64_t c, const double* x,
                                                          const double* r, const double* p,
                                                          const double* Hp, const double* dt_col,
                                                          double* x_new, double* r_new,
                                                          IterScalars* sc) {
  pdl_wait();
  __shared__ double sh[32];
  int flags = 0;
  for (int64_t j = 0; j < c; ++j) {
    double s = 0.0;
    for (int64_t i = threadIdx.x; i < d; i += blockDim.x) s = fma(p[j * d + i], Hp[j * d + i], s);
    const double pHp = blk_sum(s, sh);
    const bool active = dt_col[j] > 0.0;
    if (active && pHp <= 0.0) flags |= FLAG_BREAKDOWN;
    const double alpha = active ? dt_col[j] / (pHp > 0.0 ? pHp : 1.0) : 0.0;
    for (int64_t i = threadIdx.x; i < d; i += blockDim.x) {
      x_new[j * d + i] = x[j * d + i] + p[j * d + i] * alpha;
      r_new[j * d + i] = r[j * d + i] - Hp[j * d + i] * alpha;
    }
  }
  if (threadIdx.x == 0) sc->flags = flags;
}

// PCG propose, second half: dt_new = _scalars(r_new, rt_new)
__global__ void __launch_bounds__(kVecThreads) k_pcg_scalars(int64_t d, int64_t c, const double* r,
                                                             const double* rt, double* dt_new,
                                                             IterScalars* sc, IterMail* mail, uint32_t seq) {
  pdl_wait();
  __shared__ double sh[32];
  double tot = 0.0;
  int flags = 0;
  for (int64_t j = 0; j < c; ++j) {
    double s = 0.0, q = 0.0;
    for (int64_t i = threadIdx.x; i < d; i += blockDim.x) {
      double rv = r[j * d + i];
      s = fma(rv, rt[j * d + i], s);
      q = fma(rv, rv, q);
    }
    s = blk_sum(s, sh);
    q = blk_sum(q, sh);
    if (s < -1e-12 * q) flags |= FLAG_NEGATIVE;
    double dt = s > 0.0 ? s : 0.0;
    if (threadIdx.x == 0) dt_new[j] = dt;
    tot += dt;
  }
  if (threadIdx.x == 0) {
    sc->delta_tilde = 0.5 * tot;
    sc->flags |= flags;
    publish(sc, mail, seq);
  }
}

// commit: p = rt_new + p * ratio,  ratio = old > 0 ? dt_new / old : 0  (solvers.py:277-282)
__global__ void k_pcg_commit(int64_t d, int64_t c, const double* rt_new, const double* dt_new,
                             const double* dt_old, double* p) {
  pdl_wait();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= d * c) return;
  const int64_t j = i / d;
  const double old = dt_old[j];
  const double ratio = old > 0.0 ? dt_new[j] / old : 0.0;
  p[i] = rt_new[i] + p[i] * ratio;
}

// 0.5 * sum(a .* b)
__global__ void __launch_bounds__(kVecThreads) k_half_dot(int64_t d, int64_t c, int64_t ld,
                                                          const double* a, const double* b,
                                                          IterScalars* sc, IterMail* mail, uint32_t seq) {
  pdl_wait();
  __shared__ double sh[32];
  double tot = 0.0;
  for (int64_t j = 0; j < c; ++j) {
    double s = 0.0;
    for (int64_t i = threadIdx.x; i < d; i += blockDim.x) s = fma(a[j * ld + i], b[j * ld + i], s);
    tot += blk_sum(s, sh);
  }
  if (threadIdx.x == 0) {
    sc->delta_tilde = 0.5 * tot;
    sc->flags = 0;
    publish(sc, mail, seq);
  }
}

// IHS / heavy-ball step: x_new = x - mu v (+ beta (x - x_prev))   (solvers.py:538, 562)
__global__ void k_ihs_step(int64_t n, const double* x, const double* v, double mu,
                           const double* x_prev, double beta, double* x_new) {
  pdl_wait();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double t = x[i] - mu * v[i];
  if (x_prev) t = t + beta * (x[i] - x_prev[i]);
  x_new[i] = t;
}

static int get_scalars(adask_ctx* ctx, IterScalars** sc, cudaStream_t st) {
  void* wsp = nullptr;
  ADASK_TRY(ctx->ws[WS_SMALL].get(sizeof(IterScalars), st, &wsp));
  *sc = (IterScalars*)wsp;
  if (!ctx->mail && !getenv("ADASK_NO_MAILBOX")) {
    void* mp = nullptr;
    if (cudaMallocHost(&mp, sizeof(IterMail) + 64) == cudaSuccess) {
      memset(mp, 0, sizeof(IterMail) + 64);
      ctx->mail = mp;
    } else {
      cudaGetLastError();
    }
  }
  ++ctx->mail_seq;
  if (ctx->mail_seq == 0) ctx->mail_seq = 1;
  return ADASK_OK;
}

static IterMail* mail_of(adask_ctx* ctx) { return reinterpret_cast<IterMail*>(ctx->mail); }

// The decrement and guard flags of the body just enqueued: from the mailbox
// (spin on its sequence number; errors surface through a stream query every
// ~50 ms of waiting), or, without one, a D2H copy and a stream sync.
static int read_scalars(adask_ctx* ctx, IterScalars* sc, double* dt_host, int* flags,
                        cudaStream_t st) {
  IterMail* m = mail_of(ctx);
  if (m) {
    const uint32_t want = ctx->mail_seq;
    volatile uint32_t* seq = &m->seq;
    auto t0 = std::chrono::steady_clock::now();
    for (uint64_t spin = 0; *seq != want; ++spin) {
      if ((spin & 0xFFFF) == 0xFFFF) {
        const cudaError_t q = cudaStreamQuery(st);
        if (q != cudaSuccess && q != cudaErrorNotReady)
          return fail(ADASK_E_CUDA, "iteration body failed: %s", cudaGetErrorString(q));
        if (q == cudaSuccess && *seq != want)
          return fail(ADASK_E_CUDA, "iteration mailbox not written (sequence %u)", want);
        if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(600))
          return fail(ADASK_E_CUDA, "iteration mailbox wait timed out");
      }
    }
    std::atomic_thread_fence(std::memory_order_acquire);
    if (dt_host) *dt_host = ((volatile IterMail*)m)->delta_tilde;
    *flags = ((volatile IterMail*)m)->flags;
    return ADASK_OK;
  }
  ADASK_CUDA(cudaMemcpyAsync(ctx->pinned, sc, sizeof(IterScalars), cudaMemcpyDeviceToHost, st));
  ADASK_CUDA(cudaStreamSynchronize(st));
  const IterScalars* h = reinterpret_cast<const IterScalars*>(ctx->pinned);
  if (dt_host) *dt_host = h->delta_tilde;
  *flags = h->flags;
  return ADASK_OK;
}

// H X (- B) for the problem; row-sharded problems all-reduce the partial
// A_local^T A_local X before the regularizer / B epilogue.
int problem_hess(adask_ctx* ctx, const adask_problem* pb, const double* X, const double* B,
                        double* out, cudaStream_t st) {
  const int64_t d = pb->d, c = pb->c;
  if (!problem_sharded(ctx, pb))
    return hess_mult_impl(ctx, pb->dtype, pb->A, pb->n, d, pb->lda, X, c, d, pb->nu2, pb->lam, B, d, out,
                          d, 0, st);
  ADASK_TRY(hess_mult_impl(ctx, pb->dtype, pb->A, pb->n, d, pb->lda, X, c, d, pb->nu2, pb->lam, nullptr, d,
                           out, d, ADASK_PARTIAL, st));
  ADASK_TRY(problem_allreduce(ctx, pb, out, d * c, ADASK_F64, st));
  return vec_hess_finish_impl(ctx, out, d, c, d, X, pb->nu2, pb->lam, B, out, st);
}

static int check_problem(const adask_problem* pb) {
  if (!pb || (!pb->A && pb->n > 0) || pb->n < 0 || pb->d < 1 || pb->c < 1 || pb->lda < pb->d || !pb->lam)
    return fail(ADASK_E_ARG, "bad problem descriptor");
  return ADASK_OK;
}

__global__ void k_negate_copy(const double* __restrict__ a, double* __restrict__ out, int64_t n) {
  pdl_wait();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = -a[i];
}

// PCG proposal that also leaves H x - B (x = the current iterate) in hx_mb when
// the pass over A can serve both columns (*hx_ok = 1): a rejected proposal's
// restart then needs no second pass (pcg_restart_impl with hx_mb).  Every
// value is bitwise the one adask_pcg_propose / adask_pcg_restart compute.
int pcg_propose_impl(adask_ctx* ctx, const adask_problem* pb, const adask_precond* P, const double* x,
                     const double* r, const double* p, const double* dt_col, double* Hp, double* x_new,
                     double* r_new, double* rt_new, double* dt_new, double* delta_tilde_host, double* hx_mb,
                     int* hx_ok, cudaStream_t st) {
  ADASK_TRY(check_problem(pb));
  const int64_t d = pb->d, c = pb->c;
  *hx_ok = 0;
  if (hx_mb && c == 1) {
    if (!problem_sharded(ctx, pb)) {
      ADASK_TRY(hess_mult_pair_impl(ctx, pb->dtype, pb->A, pb->n, d, pb->lda, p, nullptr, Hp, x, pb->B, hx_mb,
                                    pb->nu2, pb->lam, st, hx_ok));
    } else {
      // row-sharded: the partial pair [A_g^T A_g p | A_g^T A_g x] in one 2d
      // buffer, ONE all-reduce, then the regularizer / B epilogues.  Every
      // rank takes this path (an empty or unaligned shard forms its partials
      // with the single-column pass, or as zeros), so the number and order
      // of the collectives never depends on per-rank state.
      void* wsp = nullptr;
      ADASK_TRY(ctx->ws[WS_PAIR].get((size_t)2 * d * sizeof(double), st, &wsp));
      double* pr = (double*)wsp;
      int fused = 0;
      if (pb->n > 0)
        ADASK_TRY(hess_mult_pair_impl(ctx, pb->dtype, pb->A, pb->n, d, pb->lda, p, nullptr, pr, x, nullptr, pr + d,
                                      pb->nu2, pb->lam, st, &fused, 1));
      if (!fused) {
        ADASK_TRY(hess_mult_impl(ctx, pb->dtype, pb->A, pb->n, d, pb->lda, p, 1, d, pb->nu2, pb->lam, nullptr, d,
                                 pr, d, ADASK_PARTIAL, st));
        ADASK_TRY(hess_mult_impl(ctx, pb->dtype, pb->A, pb->n, d, pb->lda, x, 1, d, pb->nu2, pb->lam, nullptr, d,
                                 pr + d, d, ADASK_PARTIAL, st));
      }
      ADASK_TRY(problem_allreduce(ctx, pb, pr, 2 * d, ADASK_F64, st));
      ADASK_TRY(vec_hess_finish_impl(ctx, pr, d, 1, d, p, pb->nu2, pb->lam, nullptr, Hp, st));
      ADASK_TRY(vec_hess_finish_impl(ctx, pr + d, d, 1, d, x, pb->nu2, pb->lam, pb->B, hx_mb, st));
      *hx_ok = 1;
    }
  }
  if (!*hx_ok) ADASK_TRY(problem_hess(ctx, pb, p, nullptr, Hp, st));
  IterScalars* sc = nullptr;
  ADASK_TRY(get_scalars(ctx, &sc, st));
  ADASK_CUDA(launch_pdl(k_pcg_step, dim3(1), dim3(kVecThreads), 0, st, d, c, x, r, p, (const double*)Hp, dt_col,
                        x_new, r_new, sc));
  ctx->launches++;
  ADASK_TRY(precond_apply_impl(ctx, P, r_new, c, d, rt_new, d, st));
  ADASK_CUDA(launch_pdl(k_pcg_scalars, dim3(1), dim3(kVecThreads), 0, st, d, c, (const double*)r_new,
                        (const double*)rt_new, dt_new, sc, mail_of(ctx), ctx->mail_seq));
  ctx->launches++;
  int flags = 0;
  ADASK_TRY(read_scalars(ctx, sc, delta_tilde_host, &flags, st));
  if (flags & FLAG_BREAKDOWN) return fail(ADASK_E_BREAKDOWN, "direction with nonpositive curvature");
  if (flags & FLAG_NEGATIVE) return fail(ADASK_E_NEGATIVE, "r.T H_S^-1 r went negative beyond roundoff");
  return ADASK_OK;
}

// PCG restart; hx_mb = H x - B from the proposal's fused pass, or null.
int pcg_restart_impl(adask_ctx* ctx, const adask_problem* pb, const adask_precond* P, const double* x,
                     double* r, double* rt, double* p, double* dt_col, double* delta_tilde_host,
                     const double* hx_mb, cudaStream_t st) {
  ADASK_TRY(check_problem(pb));
  const int64_t d = pb->d, c = pb->c;
  if (hx_mb) {
    ADASK_CUDA(launch_pdl(k_negate_copy, dim3((unsigned)cdiv(d * c, 256)), dim3(256), 0, st, hx_mb, r, d * c));
    ADASK_LAUNCHED(ctx);
  } else {
    // r = B - H x   (computed as -(H x - B), exact)
    ADASK_TRY(problem_hess(ctx, pb, x, pb->B, r, st));
    ADASK_CUDA(launch_pdl(k_negate, dim3((unsigned)cdiv(d * c, 256)), dim3(256), 0, st, r, d * c));
    ADASK_LAUNCHED(ctx);
  }
  ADASK_TRY(precond_apply_impl(ctx, P, r, c, d, rt, d, st));
  IterScalars* sc = nullptr;
  ADASK_TRY(get_scalars(ctx, &sc, st));
  ADASK_CUDA(launch_pdl(k_pcg_restart_tail, dim3(1), dim3(kVecThreads), 0, st, d, c, rt, r, p, dt_col, sc,
                        mail_of(ctx), ctx->mail_seq));
  ADASK_LAUNCHED(ctx);
  int flags = 0;
  ADASK_TRY(read_scalars(ctx, sc, delta_tilde_host, &flags, st));
  if (flags & FLAG_NEGATIVE) return fail(ADASK_E_NEGATIVE, "r.T H_S^-1 r went negative beyond roundoff");
  return ADASK_OK;
}

// IHS restart; have_g: g already holds grad f(x) = H x - B (computed by the
// proposal that produced x, or by the previous restart at the same x -- the
// same kernel on the same x, so the same bits the reference's recomputation
// would give), and the pass over A is skipped.
int ihs_restart_impl(adask_ctx* ctx, const adask_problem* pb, const adask_precond* P, const double* x, double* g,
                     double* v, double* delta_tilde_host, bool have_g, cudaStream_t st) {
  ADASK_TRY(check_problem(pb));
  const int64_t d = pb->d, c = pb->c;
  if (!have_g) ADASK_TRY(problem_hess(ctx, pb, x, pb->B, g, st));
  ADASK_TRY(precond_apply_impl(ctx, P, g, c, d, v, d, st));
  IterScalars* sc = nullptr;
  ADASK_TRY(get_scalars(ctx, &sc, st));
  ADASK_CUDA(launch_pdl(k_half_dot, dim3(1), dim3(kVecThreads), 0, st, d, c, d, g, v, sc, mail_of(ctx),
                        ctx->mail_seq));
  ADASK_LAUNCHED(ctx);
  int flags = 0;
  return read_scalars(ctx, sc, delta_tilde_host, &flags, st);
}

}  // namespace adask

using namespace adask;

extern "C" int adask_pcg_restart(adask_ctx* ctx, const adask_problem* pb, const adask_precond* P,
                                 const double* x, double* r, double* rt, double* p, double* dt_col,
                                 double* delta_tilde_host, void* stream) {
  ADASK_TRY(use_device(ctx));
  ADASK_TRY(check_problem(pb));
  cudaStream_t st = S(stream);
  const int64_t d = pb->d, c = pb->c;
  // r = B - H x   (computed as -(H x - B), exact)
  ADASK_TRY(problem_hess(ctx, pb, x, pb->B, r, st));
  ADASK_CUDA(launch_pdl(k_negate, dim3((unsigned)cdiv(d * c, 256)), dim3(256), 0, st, r, d * c));
  ADASK_LAUNCHED(ctx);
  ADASK_TRY(precond_apply_impl(ctx, P, r, c, d, rt, d, st));
  IterScalars* sc = nullptr;
  ADASK_TRY(get_scalars(ctx, &sc, st));
  ADASK_CUDA(launch_pdl(k_pcg_restart_tail, dim3(1), dim3(kVecThreads), 0, st, d, c, rt, r, p, dt_col, sc,
                        mail_of(ctx), ctx->mail_seq));
  ADASK_LAUNCHED(ctx);
  int flags = 0;
  ADASK_TRY(read_scalars(ctx, sc, delta_tilde_host, &flags, st));
  if (flags & FLAG_NEGATIVE) return fail(ADASK_E_NEGATIVE, "r.T H_S^-1 r went negative beyond roundoff");
  return ADASK_OK;
}

extern "C" int adask_pcg_propose(adask_ctx* ctx, const adask_problem* pb, const adask_precond* P,
                                 const double* x, const double* r, const double* p,
                                 const double* dt_col, double* Hp, double* x_new, double* r_new,
                                 double* rt_new, double* dt_new, double* delta_tilde_host,
                                 void* stream) {
  ADASK_TRY(use_device(ctx));
  ADASK_TRY(check_problem(pb));
  cudaStream_t st = S(stream);
  const int64_t d = pb->d, c = pb->c;
  ADASK_TRY(problem_hess(ctx, pb, p, nullptr, Hp, st));
  IterScalars* sc = nullptr;
  ADASK_TRY(get_scalars(ctx, &sc, st));
  k_pcg_step<<<1, kVecThreads, 0, st>>>(d, c, x, r, p, Hp, dt_col, x_new, r_new, sc);
  ADASK_LAUNCHED(ctx);
  ADASK_TRY(precond_apply_impl(ctx, P, r_new, c, d, rt_new, d, st));
  k_pcg_scalars<<<1, kVecThreads, 0, st>>>(d, c, r_new, rt_new, dt_new, sc, mail_of(ctx), ctx->mail_seq);
  ADASK_LAUNCHED(ctx);
  int flags = 0;
  ADASK_TRY(read_scalars(ctx, sc, delta_tilde_host, &flags, st));
  if (flags & FLAG_BREAKDOWN) return fail(ADASK_E_BREAKDOWN, "direction with nonpositive curvature");
  if (flags & FLAG_NEGATIVE) return fail(ADASK_E_NEGATIVE, "r.T H_S^-1 r went negative beyond roundoff");
  return ADASK_OK;
}

extern "C" int adask_pcg_commit(adask_ctx* ctx, int64_t d, int64_t c, const double* rt_new,
                                const double* dt_new, const double* dt_old, double* p, void* stream) {
  ADASK_TRY(use_device(ctx));
  cudaStream_t st = S(stream);
  ADASK_CUDA(launch_pdl(k_pcg_commit, dim3((unsigned)cdiv(d * c, 256)), dim3(256), 0, st, d, c, rt_new, dt_new, dt_old, p));
  ADASK_LAUNCHED(ctx);
  return ADASK_OK;
}

extern "C" int adask_ihs_restart(adask_ctx* ctx, const adask_problem* pb, const adask_precond* P,
                                 const double* x, double* g, double* v, double* delta_tilde_host,
                                 void* stream) {
  ADASK_TRY(use_device(ctx));
  ADASK_TRY(check_problem(pb));
  cudaStream_t st = S(stream);
  const int64_t d = pb->d, c = pb->c;
  ADASK_TRY(problem_hess(ctx, pb, x, pb->B, g, st));
  ADASK_TRY(precond_apply_impl(ctx, P, g, c, d, v, d, st));
  IterScalars* sc = nullptr;
  ADASK_TRY(get_scalars(ctx, &sc, st));
  ADASK_CUDA(launch_pdl(k_half_dot, dim3(1), dim3(kVecThreads), 0, st, d, c, d, g, v, sc, mail_of(ctx),
                        ctx->mail_seq));
  ADASK_LAUNCHED(ctx);
  int flags = 0;
  return read_scalars(ctx, sc, delta_tilde_host, &flags, st);
}

extern "C" int adask_ihs_propose(adask_ctx* ctx, const adask_problem* pb, const adask_precond* P,
                                 const double* x, const double* v, double mu, const double* x_prev,
                                 double beta, double* x_new, double* g_new, double* v_new,
                                 double* delta_tilde_host, void* stream) {
  ADASK_TRY(use_device(ctx));
  ADASK_TRY(check_problem(pb));
  cudaStream_t st = S(stream);
  const int64_t d = pb->d, c = pb->c;
  ADASK_CUDA(launch_pdl(k_ihs_step, dim3((unsigned)cdiv(d * c, 256)), dim3(256), 0, st, d * c, x, v, mu, x_prev, beta, x_new));
  ADASK_LAUNCHED(ctx);
  ADASK_TRY(problem_hess(ctx, pb, x_new, pb->B, g_new, st));
  ADASK_TRY(precond_apply_impl(ctx, P, g_new, c, d, v_new, d, st));
  IterScalars* sc = nullptr;
  ADASK_TRY(get_scalars(ctx, &sc, st));
  ADASK_CUDA(launch_pdl(k_half_dot, dim3(1), dim3(kVecThreads), 0, st, d, c, d, g_new, v_new, sc, mail_of(ctx),
                        ctx->mail_seq));
  ADASK_LAUNCHED(ctx);
  int flags = 0;
  return read_scalars(ctx, sc, delta_tilde_host, &flags, st);
}

extern "C" int adask_dot(adask_ctx* ctx, const double* a, const double* b, int64_t d, int64_t c,
                         int64_t ld, double* result_host, void* stream) {
  ADASK_TRY(use_device(ctx));
  cudaStream_t st = S(stream);
  IterScalars* sc = nullptr;
  ADASK_TRY(get_scalars(ctx, &sc, st));
  ADASK_CUDA(launch_pdl(k_half_dot, dim3(1), dim3(kVecThreads), 0, st, d, c, ld, a, b, sc, mail_of(ctx),
                        ctx->mail_seq));
  ADASK_LAUNCHED(ctx);
  int flags = 0;
  return read_scalars(ctx, sc, result_host, &flags, st);
}
