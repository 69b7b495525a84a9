/*
 * adask.h — C ABI of libadask, the B200 (sm_100a) hot path of the adaptive
 * sketch-and-precondition solvers (arXiv 2104.14101, reference package
 * `adasketch`, /root/reference/pkg/src/adasketch).
 *
 * The reference is pure Python/numpy and has no FFI layer; its boundary is the
 * Python API exported by adasketch/__init__.py:3-57.  Each entry point below
 * replaces the numpy/scipy work behind one reference function; the citation
 * names that function.  The Python package `paper_2104_14101_b200` binds these
 * with ctypes (INTEGRATION.md shows the binding a maintainer of the reference
 * would add).
 *
 * Conventions
 *   - Every matrix is row-major with an explicit leading dimension (elements).
 *   - Matrices (A, SA, factors) are `dtype` (ADASK_F64 or ADASK_F32); every
 *     d-vector and every scalar is double.
 *   - Multi-column right-hand sides (d x c in the reference) are passed as c
 *     contiguous columns: column j of X starts at X + j*ldx.
 *   - Device pointers unless the name ends in _host.  `stream` is a
 *     cudaStream_t passed as void*.  Work is stream-ordered; only calls that
 *     return host scalars synchronise the stream.
 *   - Return value is a status code (ADASK_OK == 0); adask_last_error() gives
 *     the message.  Status codes map one-to-one onto the reference's
 *     exception classes (adasketch/errors.py:4-61).
 *   - Deterministic: no floating-point atomics on any result path; repeated
 *     calls on the same inputs return bitwise-identical outputs.
 */
#ifndef ADASK_H
#define ADASK_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes -> reference exceptions (errors.py) ------------------- */
enum adask_status {
  ADASK_OK = 0,
  ADASK_E_DIM = 1,              /* DimensionMismatch      errors.py:8      */
  ADASK_E_NOT_SPD = 2,          /* NotPositiveDefinite    errors.py:12     */
  ADASK_E_NOT_POW2 = 3,         /* NotPowerOfTwo          errors.py:16     */
  ADASK_E_SKETCH_TOO_LARGE = 4, /* SketchTooLarge         errors.py:36     */
  ADASK_E_SPARSITY = 5,         /* InvalidSparsity        errors.py:40     */
  ADASK_E_NEGATIVE = 6,         /* NegativeValue          errors.py:48     */
  ADASK_E_BREAKDOWN = 7,        /* BreakdownDetected      errors.py:52     */
  ADASK_E_ARG = 8,              /* ValueError                              */
  ADASK_E_CUDA = 9,             /* RuntimeError (CUDA error string)        */
  ADASK_E_NOMEM = 10            /* MemoryError                             */
};

enum adask_dtype { ADASK_F64 = 0, ADASK_F32 = 1 };

/* flags */
#define ADASK_ACCUMULATE 0x1u /* sketch: SA += result instead of SA = result      */
#define ADASK_PARTIAL 0x2u    /* hess_mult: out = A^T A X only (no nu^2 Lam X - B) */
#define ADASK_TF32 0x4u       /* gaussian fp32: TF32 tensor-core GEMM             */
#define ADASK_INCREMENTAL 0x8u /* adaptive_run: grow the sketch instead of redrawing */

const char* adask_last_error(void);
int adask_version(void);
int adask_device_count(void);

/* ======================================================================== */
/* Host-side randomness bookkeeping (numpy 2.3.5 Generator compatible).     */
/* Pure host code: callable without a GPU.                                  */
/* ======================================================================== */

/* numpy.random.PCG64 state (bit_generator.state): 128-bit state and
 * increment, plus the buffered upper half used by next_uint32.            */
typedef struct adask_pcg64 {
  uint64_t state_hi, state_lo;
  uint64_t inc_hi, inc_lo;
  int32_t has_uint32;
  uint32_t uinteger;
} adask_pcg64;

/* SeedSequence(entropy).generate_state(n_words, uint32); entropy given as
 * little-endian uint32 words of the (concatenated) integers.
 * Replaces numpy SeedSequence used by derive_seed, embeddings.py:56-58.    */
int adask_seedseq_generate(const uint32_t* entropy, int64_t n_entropy,
                           uint32_t* out_words, int64_t n_words);

/* derive_seed(base, k) = SeedSequence((base, k)).generate_state(1, u64)[0]
 * for base, k < 2^64 (embeddings.py:56-58).                               */
uint64_t adask_derive_seed(uint64_t base, uint64_t k);

/* np.random.default_rng(seed).bit_generator: PCG64(SeedSequence(entropy)).
 * Replaces np.random.default_rng at embeddings.py:71, 95, 117.           */
int adask_pcg64_seed(const uint32_t* entropy, int64_t n_entropy, adask_pcg64* g);
/* Advance by n 64-bit outputs (PCG64.advance). */
int adask_pcg64_advance(adask_pcg64* g, uint64_t n_u64);
/* Skip n 32-bit draws, honouring the buffered half (next_uint32 semantics). */
int adask_pcg64_skip_u32(adask_pcg64* g, uint64_t n_u32);
uint64_t adask_pcg64_next_u64(adask_pcg64* g);
uint32_t adask_pcg64_next_u32(adask_pcg64* g);
/* Generator.integers(0, rng+1) single draw via Lemire on next_uint32 (rng < 2^32-1). */
uint32_t adask_pcg64_bounded_u32(adask_pcg64* g, uint32_t rng);
/* Generator.choice(N, m, replace=False): Floyd + shuffle, or tail shuffle.
 * Replaces rng.choice at embeddings.py:100 (SRHT row subsample).          */
int adask_choice_noreplace(adask_pcg64* g, int64_t N, int64_t m, int64_t* out_host);
/* SJLT row picks for s > 1 (embeddings.py:121-123): rows[j*s .. j*s+s) =
 * choice(m, s, replace=False) for every column j; *draws_out = 32-bit draws
 * consumed (the sign draws start there).                                   */
int adask_sjlt_rows(adask_pcg64* g, int64_t n, int64_t m, int64_t s, int64_t* rows_out,
                    uint64_t* draws_out);
/* Host restatement of Generator.integers(0, m, size=count) (buckets or
 * signs), used by tests to pin the device stream. kind: 0 = value, 1 = sign (+-1 as int8). */
int adask_pcg64_integers_host(adask_pcg64* g, uint32_t m, int64_t count, int64_t* out_host);

/* ======================================================================== */
/* Device context                                                           */
/* ======================================================================== */
typedef struct adask_ctx adask_ctx;
int adask_ctx_create(int device, adask_ctx** out);
int adask_ctx_destroy(adask_ctx* ctx);
/* Kernel launches issued through this ctx since creation (instrumentation). */
int64_t adask_ctx_launches(const adask_ctx* ctx);
/* Live timing of work units with CUDA events on the launching stream.
 * kind: 0 hess_mult, 1 SRHT sketch, 2 SJLT sketch, 3 Gaussian sketch,
 * 4 preconditioner build, 5 preconditioner apply.  Query synchronises and
 * returns the number of units, their summed device time and algorithmic
 * bytes / flops.                                          */
int adask_prof_enable(adask_ctx* ctx, int on);
int adask_prof_reset(adask_ctx* ctx);
int adask_prof_query(adask_ctx* ctx, int kind, int64_t* count, double* total_ms,
                     double* total_bytes, double* total_flops);

/* ======================================================================== */
/* Randomness on the device                                                 */
/* ======================================================================== */

/* Values of Generator.integers(0, m, size=count) drawn from a fresh
 * generator `g`, starting at 32-bit draw index u32_first (jump-ahead; item i
 * uses the i-th accepted draw at or after u32_first).  out: int32[count].
 * m == 2 gives the SRHT/SJLT sign bits (embeddings.py:96, 124).
 * On return *u32_next_host (if non-null) holds the draw index that follows
 * the last consumed one.                                                   */
int adask_pcg64_integers(adask_ctx* ctx, const adask_pcg64* g, uint64_t u32_first,
                         int64_t count, uint32_t m, int32_t* out,
                         uint64_t* u32_next_host, void* stream);

/* Gaussian sketch matrix entries, Philox4x32-10 + Box-Muller, N(0,1)/sqrt(m):
 * S[k, i] for k in [0, m), i in [col0, col0 + ncols), written row-major to
 * out with leading dimension ldo.  Counter = (pair index of global column i,
 * row k); key = 64-bit seed.  Deterministic and shard-invariant.          */
int adask_philox_gaussian(adask_ctx* ctx, int dtype, int64_t m, int64_t col0, int64_t ncols,
                          uint64_t key, void* out, int64_t ldo, void* stream);

/* Host evaluation of the same entries (pins the definition without a GPU). */
int adask_philox_gaussian_host(int64_t m, int64_t col0, int64_t ncols, uint64_t key, double* out_host,
                               int64_t ldo);

/* ======================================================================== */
/* Sketches S*A  (embeddings.py)                                            */
/* ======================================================================== */

/* Gaussian: SA = S A with S = N(0,1/m) (embeddings.py:66-73; Philox instead
 * of numpy's ziggurat by design).  A holds rows [row0, row0+n_local) of the
 * global matrix, so per-shard calls sum to the full sketch.               */
int adask_sketch_gaussian(adask_ctx* ctx, int dtype, const void* A, int64_t n_local, int64_t d,
                          int64_t lda, int64_t row0, int64_t m, uint64_t key, void* SA,
                          int64_t ldsa, uint32_t flags, void* stream);
/* Rows [k0, k0 + mk) of the m_total-row Gaussian sketch (entries scaled by
 * 1/sqrt(m_total)) into SA rows 0 .. mk-1: incremental sketch growth
 * computes only the new rows when m doubles.                               */
int adask_sketch_gaussian_rows(adask_ctx* ctx, int dtype, const void* A, int64_t n_local, int64_t d,
                               int64_t lda, int64_t row0, int64_t m_total, int64_t k0, int64_t mk,
                               uint64_t key, void* SA, int64_t ldsa, uint32_t flags, void* stream);

/* SA = S A for an explicit m x n sketch matrix S (device): the Gaussian
 * sketch with the reference's own numpy draw (embeddings.py:71-73), for the
 * opt-in bitwise-randomness mode; the default Gaussian path is Philox.     */
int adask_sketch_dense(adask_ctx* ctx, int dtype, const void* S, int64_t m, int64_t n, int64_t lds,
                       const void* A, int64_t d, int64_t lda, void* SA, int64_t ldsa, void* stream);

/* SRHT: SA = Y[idx] * sqrt(n_pad/m), Y = fwht(diag(signs) A_padded)/sqrt(n_pad)
 * (embeddings.py:81-102, linalg.py:62-88).  `g` is the fresh generator of
 * the sketch seed; signs are draws [0, n), idx = choice(n_pad, m) after them.
 * Bitwise equal to the reference in fp64.  idx_host (nullable) receives idx. */
int adask_sketch_srht(adask_ctx* ctx, int dtype, const void* A, int64_t n, int64_t d, int64_t lda,
                      const adask_pcg64* g, int64_t m, void* SA, int64_t ldsa,
                      int64_t* idx_host, uint32_t flags, void* stream);

/* SJLT / CountSketch with s = 1 (embeddings.py:105-129): bucket of global row
 * i = draw i of integers(0, m), sign = draw n_total + (accepted offset) of
 * integers(0, 2); SA[b] = sum over rows of bucket b in ascending order.
 * A holds global rows [row0, row0 + n_local).  s > 1 passes host-generated
 * rows (rows_host, n_local*s entries, from the reference's per-column
 * choice(m, s)) and the u32 draw index where the signs start.             */
int adask_sketch_sjlt(adask_ctx* ctx, int dtype, const void* A, int64_t n_local, int64_t d,
                      int64_t lda, int64_t row0, int64_t n_total, int64_t m, int64_t s,
                      const adask_pcg64* g, const int64_t* rows_host, uint64_t sign_u32_first,
                      void* SA, int64_t ldsa, uint32_t flags, void* stream);

/* Natural-order Walsh-Hadamard transform along rows (linalg.py:62-88), in
 * place on an n x d matrix (n a power of two); normalized divides by sqrt(n). */
int adask_fwht(adask_ctx* ctx, int dtype, void* X, int64_t n, int64_t d, int64_t ldx,
               int normalized, void* stream);

/* ======================================================================== */
/* Problem: H X = A^T (A X) + nu^2 Lam X   (problem.py:89-107)              */
/* ======================================================================== */

/* Validation of a problem's inputs (problem.py:72-75: finite A and B, lam
 * entries >= 1) in one pass over A: verdict[0] = 1 if A has a non-finite
 * entry, verdict[1] = 1 if B (nb doubles) has one, verdict[2] = 1 if an entry
 * of lam (nl doubles) is non-finite or < 1.  Synchronizes the stream.      */
int adask_check_problem(adask_ctx* ctx, int dtype, const void* A, int64_t n, int64_t d, int64_t lda,
                        const double* B, int64_t nb, const double* lam, int64_t nl, int* verdict, void* stream);

/* out[:, j] = A^T (A X[:, j]) + nu2 * lam .* X[:, j] - B[:, j]   (B nullable)
 * One pass over A per column.  With ADASK_PARTIAL only A^T A X is formed
 * (multi-GPU: all-reduce, then adask_vec_hess_finish).                     */
int adask_hess_mult(adask_ctx* ctx, int dtype, const void* A, int64_t n, int64_t d, int64_t lda,
                    const double* X, int64_t c, int64_t ldx, double nu2, const double* lam,
                    const double* B, int64_t ldb, double* out, int64_t ldo, uint32_t flags,
                    void* stream);
/* out0 = H x0, out1 = H x1 with ONE pass over A (the adaptive PCG proposal
 * streams A once for [p, x] so that a rejected proposal's restart,
 * solvers.py:243-248, needs no pass of its own).  Each column is bitwise
 * adask_hess_mult's; ineligible shapes fall back to two single passes.     */
int adask_hess_mult_pair(adask_ctx* ctx, int dtype, const void* A, int64_t n, int64_t d, int64_t lda,
                         const double* x0, const double* x1, double nu2, const double* lam, double* out0,
                         double* out1, void* stream);
/* out = part + nu2 lam .* X - B (B nullable), c columns of length d. */
int adask_vec_hess_finish(adask_ctx* ctx, const double* part, int64_t d, int64_t c, int64_t ld,
                          const double* X, double nu2, const double* lam, const double* B,
                          double* out, void* stream);

/* ======================================================================== */
/* Preconditioner H_S = SA^T SA + nu^2 Lam   (preconditioner.py:26-88)      */
/* ======================================================================== */
typedef struct adask_precond adask_precond;

/* build(sa, nu, lam) (preconditioner.py:60-74): m >= d -> Cholesky of the
 * d x d H_S ("cholesky-d"); m < d -> Cholesky of the m x m capacitance
 * W_S = (SA/lam) SA^T + nu^2 I ("woodbury-m").  SA must stay alive while the
 * preconditioner is used (Woodbury reads it on every solve).  On a
 * non-positive pivot returns ADASK_E_NOT_SPD with *info_host = pivot index + 1. */
int adask_precond_build(adask_ctx* ctx, int dtype, const void* SA, int64_t m, int64_t d,
                        int64_t ldsa, double nu, const double* lam, adask_precond** out,
                        int64_t* info_host, void* stream);
int adask_precond_destroy(adask_precond* P);
/* 0 = "cholesky-d", 1 = "woodbury-m" */
int adask_precond_path(const adask_precond* P);
/* Lower Cholesky factor L (k x k, row-major, dtype), k = min(m, d); device. */
int adask_precond_factor(const adask_precond* P, const void** L, int64_t* k, int* dtype);
/* Copy the factor (which: 0 = L, 1 = L^-1, 2 = L^-T) into dst (k x k, ldd). */
int adask_precond_copy_factor(adask_ctx* ctx, const adask_precond* P, int which, void* dst,
                              int64_t ldd, void* stream);
/* Dense symmetric A^T A + nu2 diag(lam) (lam nullable: no regularizer), d x d.
 * Replaces RegularizedProblem.hessian (problem.py:109-111) and
 * Preconditioner.sketched_hessian (preconditioner.py:55-57).               */
int adask_gram(adask_ctx* ctx, int dtype, const void* A, int64_t n, int64_t d, int64_t lda,
               double nu2, const double* lam, void* out, int64_t ldo, void* stream);
/* The same with an explicit output dtype: fp32 A with an fp64 result
 * (accumulated in fp64) is the exact Hessian of direct_solve for fp32 data
 * (problem.py:144-149 with the reference's float64 cast, problem.py:51).    */
int adask_gram_ex(adask_ctx* ctx, int dtype, const void* A, int64_t n, int64_t d, int64_t lda,
                  double nu2, const double* lam, int out_dtype, void* out, int64_t ldo, void* stream);
/* Woodbury capacitance W_S = (SA * (1/lam)) SA^T + nu2 I (m x m, symmetric,
 * dtype), the matrix build() factors when m < d (preconditioner.py:72-73). */
int adask_gram_woodbury(adask_ctx* ctx, int dtype, const void* SA, int64_t m, int64_t d, int64_t ldsa,
                        double nu2, const double* lam, void* out, int64_t ldo, void* stream);
/* out = H_S^{-1} Z (preconditioner.py:42-53), c columns. */
int adask_precond_apply(adask_ctx* ctx, const adask_precond* P, const double* Z, int64_t c,
                        int64_t ldz, double* out, int64_t ldo, void* stream);

/* Dense Cholesky of a symmetric k x k matrix (linalg.py:30-44), L lower
 * (upper triangle zeroed); Linv (nullable) receives L^{-1}.                 */
int adask_cholesky(adask_ctx* ctx, int dtype, const void* M, int64_t k, int64_t ldm, void* L,
                   void* Linv, int64_t* info_host, void* stream);

/* Solve L Y = Z (transposed = 0) or L^T Y = Z (transposed = 1) for lower
 * triangular L (k x k), c right-hand sides stored as rows of Z / Y
 * (linalg.py:47-55).  Not on the solver's hot path.                         */
int adask_tri_solve(adask_ctx* ctx, int dtype, const void* L, int64_t k, int64_t ldl, int transposed,
                    const double* Z, int64_t c, int64_t ldz, double* Y, int64_t ldy, void* stream);

/* ======================================================================== */
/* Fused iteration bodies (solvers.py:227-282 _PcgState, :522-546 _IhsState)*/
/* ======================================================================== */

/* In-place sum-all-reduce of `count` elements (dtype ADASK_F64 / ADASK_F32) across the ranks that share a
 * row-sharded A (stream-ordered on `stream`); return 0 on success.  Supplied
 * by the host runtime (NCCL through torch.distributed in the Python package). */
typedef int (*adask_allreduce_fn)(void* buf, int64_t count, int dtype, void* user, void* stream);

/* Problem operand bundle for the iteration bodies.  A holds this rank's rows;
 * with `allreduce` set, every H x is formed as all_reduce(A_local^T A_local x)
 * + nu^2 Lam x (- B), i.e. one d*c all-reduce per loop pass.               */
typedef struct adask_problem {
  int dtype;
  const void* A;
  int64_t n, d, lda;
  int64_t c;          /* right-hand sides */
  double nu2;         /* nu^2 */
  const double* lam;  /* device, d        */
  const double* B;    /* device, c x d    */
  adask_allreduce_fn allreduce; /* host hook (tests over gloo); null otherwise */
  void* allreduce_user;
  int32_t use_ctx_comm; /* 1: A is this rank's row shard and the exchanges run
                           on the ctx's NCCL communicator (adask_comm_init_nccl) */
  int32_t comm_rank, comm_world; /* with the allreduce hook: rank / world size */
} adask_problem;

/* ---- row-shard communicator (NCCL over NVLink; resolved at run time) ----
 * One process per GPU.  The exchanges of a sharded solve:
 * per loop pass one all-reduce of the partial A_g^T A_g x (PCG proposals: one
 * all-reduce of the 2d pair [p, x]); per resketch a reduce-scatter of the
 * partial S_g A_g, a partial Gram over this rank's m/G rows and an all-reduce
 * of the d x d Gram (dense path), or an all-reduce of SA (Woodbury path).
 * The reference is single-process; these replace nothing
 * in it and are the B200 build's data-parallel extension.                   */
int adask_nccl_available(void);
/* ncclGetUniqueId into a 128-byte buffer (rank 0; broadcast it to the others). */
int adask_nccl_unique_id(void* id_out);
/* ncclCommInitRank on the ctx's device; the ctx owns the communicator. */
int adask_comm_init_nccl(adask_ctx* ctx, const void* id, int rank, int world);
/* Borrow an existing ncclComm_t (the caller keeps ownership). */
int adask_set_comm(adask_ctx* ctx, void* nccl_comm, int rank, int world);
int adask_comm_destroy(adask_ctx* ctx);
/* In-place sum all-reduce of count elements (dtype) on stream (no-op without a communicator). */
int adask_comm_allreduce(adask_ctx* ctx, void* buf, int64_t count, int dtype, void* stream);

/* _PcgState.restart (solvers.py:243-248): r = B - H x; rt = P^-1 r;
 * dt_col = max(colsum(r*rt), 0) with the NegativeValue guard; p = rt.
 * Returns 0.5*sum(dt_col) in *delta_tilde_host (synchronises).             */
int adask_pcg_restart(adask_ctx* ctx, const adask_problem* pb, const adask_precond* P,
                      const double* x, double* r, double* rt, double* p, double* dt_col,
                      double* delta_tilde_host, void* stream);
/* _PcgState.propose (solvers.py:264-275) into the *_new buffers; raises
 * BreakdownDetected / NegativeValue like the reference.  Synchronises.      */
int adask_pcg_propose(adask_ctx* ctx, const adask_problem* pb, const adask_precond* P,
                      const double* x, const double* r, const double* p, const double* dt_col,
                      double* Hp, double* x_new, double* r_new, double* rt_new, double* dt_new,
                      double* delta_tilde_host, void* stream);
/* _PcgState.commit (solvers.py:277-282): p = rt_new + (dt_new/dt_old) p. */
int adask_pcg_commit(adask_ctx* ctx, int64_t d, int64_t c, const double* rt_new,
                     const double* dt_new, const double* dt_old, double* p, void* stream);

/* _IhsState.restart (solvers.py:531-535): g = H x - B; v = P^-1 g;
 * returns 0.5*sum(g*v).                                                      */
int adask_ihs_restart(adask_ctx* ctx, const adask_problem* pb, const adask_precond* P,
                      const double* x, double* g, double* v, double* delta_tilde_host,
                      void* stream);
/* _IhsState.propose (solvers.py:537-542): x_new = x - mu v; g_new; v_new.
 * With x_prev non-null the heavy-ball term beta (x - x_prev) is added
 * (_PolyakState.propose, solvers.py:561-566).                               */
int adask_ihs_propose(adask_ctx* ctx, const adask_problem* pb, const adask_precond* P,
                      const double* x, const double* v, double mu, const double* x_prev,
                      double beta, double* x_new, double* g_new, double* v_new,
                      double* delta_tilde_host, void* stream);

/* ======================================================================== */
/* Native adaptive driver (solvers.py:585-659)                              */
/* ======================================================================== */
enum { ADASK_METHOD_IHS = 0, ADASK_METHOD_PCG = 1, ADASK_METHOD_POLYAK = 2 };
enum { ADASK_GAUSSIAN = 0, ADASK_SRHT = 1, ADASK_SJLT = 2, ADASK_SRHT_BLOCK = 3 };
enum { ADASK_EV_PLAIN = 0, ADASK_EV_ACCEPTED = 1, ADASK_EV_RESKETCH = 2 };

/* AdaptiveConfig (solvers.py:465-519) plus the B200 extras. */
typedef struct adask_adaptive_cfg {
  int method;            /* ADASK_METHOD_*                                   */
  int family;            /* ADASK_GAUSSIAN / SRHT / SJLT / SRHT_BLOCK        */
  double rho;
  int64_t m_init, T;
  uint64_t seed;         /* base seed; resketch K uses derive_seed(seed, K)  */
  int64_t s;             /* SJLT nonzeros per column                         */
  double alpha, phi_rho, c_alpha_rho;
  int64_t block;         /* block-SRHT rows per block                        */
  int64_t row0, n_total; /* this rank's first global row, global row count   */
  uint32_t flags;        /* ADASK_TF32                                       */
} adask_adaptive_cfg;

/* TraceRecord (solvers.py:51-59). */
typedef struct adask_trace_rec {
  int64_t t, m, k;
  double delta_tilde;
  double delta_exact;    /* valid when has_exact */
  double wall_seconds;
  int32_t event;         /* ADASK_EV_*           */
  int32_t has_exact;
} adask_trace_rec;

/* adaptive_run: x0 / x_out are c columns of length d (device); xstar
 * (nullable, device) enables the exact error of every record.  recs needs
 * room for 3*T + 64 records.                                              */
int adask_adaptive_run(adask_ctx* ctx, const adask_problem* pb, const adask_adaptive_cfg* cfg,
                       const double* x0, double* x_out, const double* xstar, adask_trace_rec* recs,
                       int64_t max_recs, int64_t* n_recs, void* stream);

/* 0.5 * sum(a .* b) over c columns of length d (deterministic). */
int adask_dot(adask_ctx* ctx, const double* a, const double* b, int64_t d, int64_t c,
              int64_t ld, double* result_host, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* ADASK_H */
