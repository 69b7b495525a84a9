"""CPU oracle for the adaptive sketching hot path -- TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference algorithm (adasketch, /root/reference/
pkg/src/adasketch) for the path BASELINE.json's north_star names.  Only
tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this module, and only as the checker or the timed
CPU baseline; the product (paper_2104_14101_b200) never calls it.

Pinning: tests/golden/*.npz hold outputs of the reference itself (imported in
the build container by tests/golden/make_golden.py); tests/test_oracle_golden.py
checks every function here against them.  The arithmetic the reference
delegates to third-party code is restated against the same dependency the
reference uses: numpy 2.3.5's Generator (PCG64 + Lemire integers + choice,
unpinned in pkg/pyproject.toml:10-13, pinned by this image) and LAPACK/BLAS
via numpy/scipy.

Deliberate extension (not in the reference): the Gaussian sketch matrix comes
from Philox4x32-10 + Box-Muller (north_star mandates on-device Philox tiles),
restated in `philox_gaussian`; `adaptive_run(..., sketcher=...)` injects it
(or the block-SRHT of config 4) exactly where the reference calls
embeddings.sketch (solvers.py:618, 643-645).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import scipy.linalg
import scipy.sparse

_CONVERGED_REL = 1e-26  # solvers.py:43


# ------------------------------------------------------------- embeddings.py
def derive_seed(base: int, k: int) -> int:
    """embeddings.py:56-58."""
    return int(np.random.SeedSequence((base, k)).generate_state(1, np.uint64)[0])


def padded_rows(n: int) -> int:
    """embeddings.py:76-78."""
    return 1 << max(0, int(np.ceil(np.log2(n))))


def fwht(x: np.ndarray, normalized: bool = True) -> np.ndarray:
    """linalg.py:62-88: radix-2 stages h = 1, 2, 4, ... pairing (j, j+h) inside
    blocks of 2h; (a, b) -> (a + b, a - b); then true division by sqrt(n)."""
    y = np.array(x, dtype=np.float64, copy=True)
    n = y.shape[0]
    if n < 1 or (n & (n - 1)):
        raise ValueError(f"length {n} is not a power of two")
    vec = y.ndim == 1
    y = y.reshape(n, -1)
    h = 1
    while h < n:
        blocks = y.reshape(n // (2 * h), 2, h, y.shape[1])
        top = blocks[:, 0] + blocks[:, 1]
        bot = blocks[:, 0] - blocks[:, 1]
        blocks[:, 0] = top
        blocks[:, 1] = bot
        h *= 2
    if normalized:
        y = y / np.sqrt(n)
    return y[:, 0] if vec else y


def srht_draws(n: int, m: int, seed: int) -> tuple[np.ndarray, np.ndarray]:
    """Sign bits and row subsample in the reference's draw order
    (embeddings.py:95-100): integers(0, 2, n), then choice(n_pad, m)."""
    rng = np.random.default_rng(seed)
    bits = rng.integers(0, 2, size=n)
    idx = rng.choice(padded_rows(n), size=m, replace=False)
    return bits, idx


def sketch_srht(A: np.ndarray, m: int, seed: int) -> np.ndarray:
    """embeddings.py:81-102 (returns SA)."""
    A = np.asarray(A, dtype=np.float64)
    n, d = A.shape
    n_pad = padded_rows(n)
    if m < 1 or m > n_pad:
        raise ValueError("sketch size out of range")
    bits, idx = srht_draws(n, m, seed)
    Y = np.zeros((n_pad, d))
    Y[:n] = A * (bits * 2.0 - 1.0)[:, None]
    Y = fwht(Y, normalized=True)
    return Y[idx] * np.sqrt(n_pad / m)


def sjlt_draws(n: int, m: int, seed: int, s: int = 1) -> tuple[np.ndarray, np.ndarray]:
    """Bucket rows then sign bits (embeddings.py:117-124)."""
    rng = np.random.default_rng(seed)
    if s == 1:
        rows = rng.integers(0, m, size=n)
    else:
        rows = np.empty(n * s, dtype=np.int64)
        for j in range(n):
            rows[j * s:(j + 1) * s] = rng.choice(m, size=s, replace=False)
    bits = rng.integers(0, 2, size=n * s)
    return rows, bits


def sketch_sjlt(A: np.ndarray, m: int, seed: int, s: int = 1) -> np.ndarray:
    """embeddings.py:105-129 (returns SA)."""
    A = np.asarray(A, dtype=np.float64)
    n, d = A.shape
    rows, bits = sjlt_draws(n, m, seed, s)
    vals = (bits * 2.0 - 1.0) / np.sqrt(s)
    S = scipy.sparse.csr_matrix((vals, (rows.ravel(), np.repeat(np.arange(n), s))), shape=(m, n))
    return S @ A


def sjlt_sequential(A: np.ndarray, m: int, seed: int) -> np.ndarray:
    """Same sketch as ascending-row per-bucket sums (the order csr_matvecs
    uses); bitwise equal to sketch_sjlt for s = 1."""
    A = np.asarray(A, dtype=np.float64)
    rows, bits = sjlt_draws(A.shape[0], m, seed, 1)
    SA = np.zeros((m, A.shape[1]))
    for i in range(A.shape[0]):
        SA[rows[i]] += A[i] if bits[i] else -A[i]
    return SA


def sjlt_shard(A_local: np.ndarray, m: int, seed: int, row0: int, n_total: int) -> np.ndarray:
    """Partial SJLT sketch of global rows [row0, row0 + n_local): buckets and
    signs are the reference's draws for those global rows (embeddings.py:
    117-124 over the full n_total), summed in ascending row order."""
    A_local = np.asarray(A_local, dtype=np.float64)
    rows, bits = sjlt_draws(n_total, m, seed, 1)
    SA = np.zeros((m, A_local.shape[1]))
    for i in range(A_local.shape[0]):
        g = row0 + i
        SA[rows[g]] += A_local[i] if bits[g] else -A_local[i]
    return SA


def philox4x32_10(ctr: np.ndarray, key: tuple[int, int]) -> np.ndarray:
    """Philox4x32-10 on a (..., 4) uint32 counter array (Salmon et al. 2011)."""
    M0, M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
    W0, W1 = 0x9E3779B9, 0xBB67AE85
    c = ctr.astype(np.uint64)
    k0, k1 = key[0] & 0xFFFFFFFF, key[1] & 0xFFFFFFFF
    mask = np.uint64(0xFFFFFFFF)
    for _ in range(10):
        p0 = M0 * c[..., 0]
        p1 = M1 * c[..., 2]
        hi0, lo0 = p0 >> np.uint64(32), p0 & mask
        hi1, lo1 = p1 >> np.uint64(32), p1 & mask
        n0 = hi1 ^ c[..., 1] ^ np.uint64(k0)
        n2 = hi0 ^ c[..., 3] ^ np.uint64(k1)
        c = np.stack([n0, lo1, n2, lo0], axis=-1)
        k0 = (k0 + W0) & 0xFFFFFFFF
        k1 = (k1 + W1) & 0xFFFFFFFF
    return c.astype(np.uint32)


def philox_gaussian(m: int, n: int, seed: int, col0: int = 0) -> np.ndarray:
    """Gaussian sketch matrix S (m x n), columns [col0, col0+n) of the global
    matrix (the product's definition, rng.cuh: gaussian_quad_f64, restated).
    For global column i and row group g = k >> 2, Philox4x32-10 with counter
    (i_lo, i_hi, g, 0) and key = 64-bit seed gives words o0..o3;
    u_j = (o_j >> 9) 2^-23; (z0, z1) = sqrt(-2 ln(1 - u0)) (cos, sin)(2 pi u1),
    (z2, z3) likewise from (u2, u3); S[k, i] = z_{k & 3} / sqrt(m)."""
    key = (int(seed) & 0xFFFFFFFF, (int(seed) >> 32) & 0xFFFFFFFF)
    ngrp = (m + 3) // 4
    i = np.arange(col0, col0 + n, dtype=np.uint64)
    g = np.arange(ngrp, dtype=np.uint64)
    ctr = np.zeros((ngrp, n, 4), dtype=np.uint64)
    ctr[..., 0] = (i & np.uint64(0xFFFFFFFF))[None, :]
    ctr[..., 1] = (i >> np.uint64(32))[None, :]
    ctr[..., 2] = g[:, None]
    o = philox4x32_10(ctr, key)
    u = (o >> np.uint32(9)).astype(np.float64) * 2.0**-23
    Z = np.empty((ngrp, 4, n))
    for p in range(2):
        rad = np.sqrt(-2.0 * np.log(1.0 - u[..., 2 * p]))
        th = 6.283185307179586 * u[..., 2 * p + 1]
        Z[:, 2 * p] = rad * np.cos(th)
        Z[:, 2 * p + 1] = rad * np.sin(th)
    return Z.reshape(4 * ngrp, n)[:m] / np.sqrt(m)


def sketch_gaussian(A: np.ndarray, m: int, seed: int, S: np.ndarray | None = None) -> np.ndarray:
    """embeddings.py:66-73 with the Philox S (or an injected S)."""
    A = np.asarray(A, dtype=np.float64)
    if S is None:
        S = philox_gaussian(m, A.shape[0], seed)
    return S @ A


def numpy_gaussian(A: np.ndarray, m: int, seed: int) -> np.ndarray:
    """The reference's own Gaussian sketch (embeddings.py:66-73: ziggurat
    normals from default_rng(seed), divided by sqrt(m)); used to pin the
    oracle's driver against the reference's traces."""
    A = np.asarray(A, dtype=np.float64)
    S = np.random.default_rng(seed).standard_normal((m, A.shape[0])) / np.sqrt(m)
    return S @ A


def block_srht(A: np.ndarray, m: int, seed: int, block: int) -> np.ndarray:
    """Config 4's block-SRHT: SA = sum_b sketch_srht(A_b, m, derive_seed(seed, b))
    over row blocks of `block` rows, accumulated in block order."""
    n = A.shape[0]
    SA = None
    for b, r0 in enumerate(range(0, n, block)):
        part = sketch_srht(A[r0:r0 + block], m, derive_seed(seed, b))
        SA = part if SA is None else SA + part
    return SA


def sketch(A, family: str, m: int, seed: int, s: int = 1):
    """embeddings.py:132-140."""
    if family == "gaussian":
        return sketch_gaussian(A, m, seed)
    if family == "srht":
        return sketch_srht(A, m, seed)
    if family == "sjlt":
        return sketch_sjlt(A, m, seed, s)
    raise ValueError(family)


# --------------------------------------------------------- preconditioner.py
def cholesky(M: np.ndarray) -> np.ndarray:
    """linalg.py:30-44 (symmetrize, LAPACK potrf)."""
    M = np.asarray(M, dtype=np.float64)
    return np.linalg.cholesky((M + M.T) / 2.0)


@dataclass
class Precond:
    SA: np.ndarray
    nu: float
    lam: np.ndarray
    path: str
    L: np.ndarray

    def solve(self, Z: np.ndarray) -> np.ndarray:
        """preconditioner.py:42-53."""
        Z = np.asarray(Z, dtype=np.float64)
        vec = Z.ndim == 1
        Zm = Z[:, None] if vec else Z
        tri = scipy.linalg.solve_triangular
        if self.path == "cholesky-d":
            out = tri(self.L, tri(self.L, Zm, lower=True), lower=True, trans=1)
        else:
            Y = Zm / self.lam[:, None]
            u = tri(self.L, tri(self.L, self.SA @ Y, lower=True), lower=True, trans=1)
            out = (Y - (self.SA.T @ u) / self.lam[:, None]) / self.nu**2
        return out[:, 0] if vec else out


def build(SA: np.ndarray, nu: float, lam: np.ndarray) -> Precond:
    """preconditioner.py:60-74."""
    SA = np.asarray(SA, dtype=np.float64)
    m, d = SA.shape
    lam = np.asarray(lam, dtype=np.float64)
    if m >= d:
        return Precond(SA, nu, lam, "cholesky-d", cholesky(SA.T @ SA + (nu**2) * np.diag(lam)))
    W = (SA * (1.0 / lam)[None, :]) @ SA.T + (nu**2) * np.eye(m)
    return Precond(SA, nu, lam, "woodbury-m", cholesky(W))


# ---------------------------------------------------------------- problem.py
@dataclass
class Problem:
    A: np.ndarray
    B: np.ndarray
    nu: float
    lam: np.ndarray

    @staticmethod
    def make(A, B, nu, lam=None) -> "Problem":
        A = np.asarray(A, dtype=np.float64)
        B = np.asarray(B, dtype=np.float64)
        if B.ndim == 1:
            B = B[:, None]
        lam = np.ones(A.shape[1]) if lam is None else np.asarray(lam, dtype=np.float64)
        return Problem(A, B, float(nu), lam)

    @property
    def n(self):
        return self.A.shape[0]

    @property
    def d(self):
        return self.A.shape[1]

    def hess_mult(self, X):
        """problem.py:89-95."""
        X = np.asarray(X, dtype=np.float64)
        vec = X.ndim == 1
        Xm = X[:, None] if vec else X
        out = self.A.T @ (self.A @ Xm) + (self.nu**2) * (self.lam[:, None] * Xm)
        return out[:, 0] if vec else out

    def gradient(self, X):
        """problem.py:97-107."""
        X = np.asarray(X, dtype=np.float64)
        vec = X.ndim == 1
        Xm = X[:, None] if vec else X
        out = self.hess_mult(Xm) - self.B
        return out[:, 0] if vec else out

    def hessian(self):
        return self.A.T @ self.A + (self.nu**2) * np.diag(self.lam)


def direct_solve(p: Problem) -> np.ndarray:
    """problem.py:144-149 (returns x_star, d x c)."""
    L = cholesky(p.hessian())
    y = scipy.linalg.solve_triangular(L, p.B, lower=True)
    return scipy.linalg.solve_triangular(L, y, lower=True, trans=1)


def exact_error(p: Problem, x, x_star) -> float:
    """problem.py:152-158."""
    x = np.asarray(x, dtype=np.float64)
    x = x[:, None] if x.ndim == 1 else x
    diff = x - x_star
    return 0.5 * float(np.sum(diff * p.hess_mult(diff)))


# ---------------------------------------------------------------- solvers.py
class PcgState:
    """solvers.py:227-282."""

    def __init__(self, p: Problem, P: Precond, x: np.ndarray, rho=None):
        self.p = p
        self.x = x.copy()
        self.restart(P)

    def restart(self, P):
        self.P = P
        self.r = self.p.B - self.p.hess_mult(self.x)
        self.rt = P.solve(self.r)
        self.dt_col = self._scalars(self.r, self.rt)
        self.pdir = self.rt.copy()

    @staticmethod
    def _scalars(r, rt):
        dt = np.sum(r * rt, axis=0)
        if np.any(dt < -1e-12 * np.sum(r * r, axis=0)):
            raise ArithmeticError("NegativeValue")
        return np.maximum(dt, 0.0)

    @property
    def delta_tilde(self):
        return 0.5 * float(self.dt_col.sum())

    def propose(self):
        active = self.dt_col > 0.0
        Hp = self.p.hess_mult(self.pdir)
        pHp = np.sum(self.pdir * Hp, axis=0)
        if np.any(active & (pHp <= 0.0)):
            raise ArithmeticError("BreakdownDetected")
        alpha = np.where(active, self.dt_col / np.where(pHp > 0, pHp, 1.0), 0.0)
        x_new = self.x + self.pdir * alpha
        r_new = self.r - Hp * alpha
        rt_new = self.P.solve(r_new)
        dt_new = self._scalars(r_new, rt_new)
        return 0.5 * float(dt_new.sum()), (x_new, r_new, rt_new, dt_new)

    def commit(self, dt_scalar, stash):
        x_new, r_new, rt_new, dt_new = stash
        old = self.dt_col
        ratio = np.where(old > 0, dt_new / np.where(old > 0, old, 1.0), 0.0)
        self.pdir = rt_new + self.pdir * ratio
        self.x, self.r, self.rt, self.dt_col = x_new, r_new, rt_new, dt_new


class IhsState:
    """solvers.py:522-546."""

    def __init__(self, p, P, x, rho):
        self.p = p
        self.mu = 1.0 - rho
        self.x = x
        self.restart(P)

    def restart(self, P):
        self.P = P
        self.g = self.p.gradient(self.x)
        self.v = P.solve(self.g)
        self.delta_tilde = 0.5 * float(np.sum(self.g * self.v))

    def propose(self):
        x_new = self.x - self.mu * self.v
        g_new = self.p.gradient(x_new)
        v_new = self.P.solve(g_new)
        return 0.5 * float(np.sum(g_new * v_new)), (x_new, g_new, v_new)

    def commit(self, dt_new, stash):
        self.x, self.g, self.v = stash
        self.delta_tilde = dt_new


def method_constants(method: str, rho: float) -> tuple[float, float]:
    """solvers.py:453-462 (ihs / pcg)."""
    if method == "ihs":
        return 1.0, rho
    root = np.sqrt(1.0 - rho)
    return 4.0, (1.0 - root) / (1.0 + root)


@dataclass
class Record:
    t: int
    m: int
    k: int
    delta_tilde: float
    delta_exact: float | None
    event: str


@dataclass
class Trace:
    records: list = field(default_factory=list)

    def schedule(self):
        return [(r.t, r.m) for r in self.records if r.event == "resketch"]


class IncrementalSketcher:
    """The library's incremental sketch growth (driver.cu: make_sketch_incr),
    restated: every sketch uses the seed of sketch 0 (derive_seed(seed, 0)).
    Gaussian (Philox S): the first sketch is S(m) A;
    growing to m' keeps the rows as SA * sqrt(m / m') and appends rows
    [m, m') of S(m') A.  SRHT / block SRHT: Y_b = fwht(D_b pad(A_b)) /
    sqrt(n_pad_b) once per block (signs = integers(0, 2, n_b) of the block's
    generator), perm_b = choice(n_pad_b, n_pad_b, replace=False) drawn next;
    SA(m) = sum_b Y_b[perm_b[:m]] * sqrt(n_pad_b / m)."""

    def __init__(self, family: str, seed: int, block: int | None = None):
        self.family, self.seed0, self.block = family, derive_seed(seed, 0), block
        self.SA = None
        self.m = 0
        self.Y = None

    def __call__(self, A, m: int, _seed=None):
        A = np.asarray(A, dtype=np.float64)
        if self.family == "gaussian":
            gen = philox_gaussian
            if self.SA is None:
                self.SA = gen(m, A.shape[0], self.seed0) @ A
            elif m != self.m:
                new = gen(m, A.shape[0], self.seed0)[self.m:] @ A
                self.SA = np.vstack([self.SA * np.sqrt(self.m / m), new])
            self.m = m
            return self.SA.copy()
        if self.family in ("srht", "srht-block"):
            if self.Y is None:
                n = A.shape[0]
                B = n if self.family == "srht" else self.block
                self.Y = []
                for b, r0 in enumerate(range(0, n, B)):
                    Ab = A[r0:r0 + B]
                    nb = Ab.shape[0]
                    npad = padded_rows(nb)
                    sd = self.seed0 if self.family == "srht" else derive_seed(self.seed0, b)
                    rng = np.random.default_rng(sd)
                    bits = rng.integers(0, 2, size=nb)
                    X = np.zeros((npad, Ab.shape[1]))
                    X[:nb] = Ab * (bits * 2.0 - 1.0)[:, None]
                    Y = fwht(X, normalized=True)
                    perm = rng.choice(npad, size=npad, replace=False)
                    self.Y.append((Y, perm, npad))
            SA = None
            for Y, perm, npad in self.Y:
                part = Y[perm[:m]] * np.sqrt(npad / m)
                SA = part if SA is None else SA + part
            return SA
        raise ValueError(f"no incremental rule for family {self.family!r}")


def adaptive_run(p: Problem, x0, method: str, rho: float, m_init: int, T: int, family: str,
                 seed: int, s: int = 1, x_star=None, sketcher=None, cap=None, log=None):
    """solvers.py:585-659 (ihs / pcg).  `sketcher(A, m, seed)` replaces
    embeddings.sketch (Gaussian Philox S, block-SRHT); `log` collects the
    decision ratios dt_new / (threshold * dt_I)."""
    alpha, phi = method_constants(method, rho)
    sq = np.sqrt(rho)
    c_ar = (1.0 + sq) / (1.0 - sq) * alpha
    x = np.asarray(x0, dtype=np.float64)
    x = (x[:, None] if x.ndim == 1 else x).copy()
    if cap is None:
        cap = padded_rows(p.n) if family == "srht" else p.n
    sk = sketcher or (lambda A, m_, sd: sketch(A, family, m_, sd, s))
    m = min(m_init, cap)
    K = 0
    P = build(sk(p.A, m, derive_seed(seed, 0)), p.nu, p.lam)
    state = (IhsState if method == "ihs" else PcgState)(p, P, x, rho)
    trace = Trace()
    err = (lambda xx: exact_error(p, xx, x_star)) if x_star is not None else (lambda xx: None)
    dt_first = dt_I = state.delta_tilde
    t = I = 0
    capped_retry = False
    trace.records.append(Record(0, m, 0, state.delta_tilde, err(state.x), "plain"))
    while t < T:
        dt_new, stash = state.propose()
        ell = t + 1 - I
        thr = c_ar * phi**ell
        if log is not None and dt_I > 0:
            log.append(dt_new / (thr * dt_I))
        converged = dt_I <= 0.0 or dt_new <= _CONVERGED_REL * dt_first
        reject = (not converged) and dt_new > thr * dt_I
        if reject and capped_retry:
            reject = False
        if reject:
            K += 1
            at_cap = m >= cap
            m = min(2 * m, cap)
            capped_retry = at_cap
            P = build(sk(p.A, m, derive_seed(seed, K)), p.nu, p.lam)
            state.restart(P)
            dt_I = state.delta_tilde
            I = t
            trace.records.append(Record(t, m, K, dt_I, err(state.x), "resketch"))
        else:
            state.commit(dt_new, stash)
            t += 1
            capped_retry = False
            trace.records.append(Record(t, m, K, state.delta_tilde, err(state.x), "accepted"))
    return state.x, trace


# ------------------------------------------------------- config generators
def make_config_problem(n: int, d: int, sigma: np.ndarray, nu: float, lam_uniform: bool,
                        data_seed: int = 0, dtype=np.float64, chunk: int | None = None):
    """SURVEY.md 8(d) instance: A = G diag(sigma) V^T, G iid N(0, 1/n),
    V = qr(N(0,1) d x d).Q, b = A^T (A x0 + 0.01 eps), Lam = I or
    default_rng(123).uniform(1, 10, d).  Row-chunked generation reproduces
    the monolithic stream."""
    rng = np.random.default_rng(data_seed)
    chunk = chunk or n
    G_parts = []
    for r0 in range(0, n, chunk):
        G_parts.append(rng.standard_normal((min(chunk, n - r0), d)) / np.sqrt(n))
    V, _ = np.linalg.qr(rng.standard_normal((d, d)))
    x0 = rng.standard_normal(d)
    eps = rng.standard_normal(n)
    W = (sigma[:, None] * V.T)  # diag(sigma) V^T
    A = np.empty((n, d), dtype=dtype)
    r0 = 0
    for Gp in G_parts:
        A[r0:r0 + Gp.shape[0]] = Gp @ W
        r0 += Gp.shape[0]
    A64 = A.astype(np.float64, copy=False)
    b = A64.T @ (A64 @ x0 + 0.01 * eps)
    lam = np.random.default_rng(123).uniform(1.0, 10.0, d) if lam_uniform else np.ones(d)
    return A, b, lam


CONFIGS = {
    # name: (method, family, n, d, sigma(j), nu, lam_uniform, m_init, target, dtype)
    0: ("ihs", "gaussian", 4096, 256, lambda j: j**-1.0, 1e-1, False, 16, 1e-10, "float64"),
    1: ("pcg", "srht", 1 << 16, 1024, lambda j: 0.98**j, 1e-2, False, 32, 1e-10, "float64"),
    2: ("pcg", "sjlt", 1 << 20, 2048, lambda j: j**-0.5, 1e-3, True, 64, 1e-10, "float64"),
    3: ("ihs", "gaussian", 1 << 21, 4096, lambda j: j**-1.0, 1e-2, False, 128, 1e-6, "float32"),
    4: ("pcg", "srht-block", 1 << 24, 1024, lambda j: 0.995**j, 1e-3, True, 64, 1e-6, "float32"),
}


def config_sigma(cfg: int, d: int) -> np.ndarray:
    j = np.arange(1, d + 1, dtype=np.float64)
    return CONFIGS[cfg][4](j)
