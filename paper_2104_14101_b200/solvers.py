"""Sketched solvers and the adaptive sketch-size driver, on the B200.

Drop-in for adasketch/solvers.py.  The control logic (thresholds
c(alpha, rho) phi(rho)^ell, the converged floor, the cap and capped-retry
rules, the derive_seed(seed, K) redraw chain, the trace records) is kept on
the host and follows solvers.py:450-659 statement by statement, so the
accept/reject schedule is decided by the same arithmetic on the same
decrement values.  Everything else -- sketches, preconditioner factorization,
the A^T A passes, the solves and the d-vector updates -- runs in libadask on
the device; each loop pass makes one 64-byte device->host readback (the new
decrement).
"""
from __future__ import annotations

import ctypes as C
import os
import time
import warnings
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from . import device as dv
from .embeddings import SketchSpec, derive_seed, gaussian_rng, padded_rows, sketch_dev
from .errors import BreakdownDetected
from .preconditioner import Preconditioner, build_dev
from .problem import ExactSolution, RegularizedProblem, exact_error_dev

__all__ = [
    "TraceRecord",
    "SolverTrace",
    "AdaptiveConfig",
    "ihs_step",
    "ihs_run",
    "pcg_run",
    "polyak_coefficients",
    "polyak_ihs_run",
    "adaptive_run",
    "cg",
]

# Relative floor (vs delta_tilde at t = 0) below which an iterate counts as
# converged to working precision (solvers.py:40-43).
_CONVERGED_REL = 1e-26


@dataclass
class TraceRecord:
    t: int
    m: int
    k: int
    delta_tilde: float
    delta_exact: float | None
    wall_seconds: float
    event: str  # "plain" | "accepted" | "resketch"


@dataclass
class SolverTrace:
    records: list[TraceRecord] = field(default_factory=list)

    def append(self, rec: TraceRecord) -> None:
        self.records.append(rec)

    @property
    def final(self) -> TraceRecord:
        return self.records[-1]

    @property
    def resketch_count(self) -> int:
        return self.final.k if self.records else 0

    def delta_exact_series(self) -> list[float]:
        return [r.delta_exact for r in self.records]

    def schedule(self) -> list[tuple[int, int]]:
        """(t, m) of every resketch event -- the m_t schedule."""
        return [(r.t, r.m) for r in self.records if r.event == "resketch"]

    def __len__(self) -> int:
        return len(self.records)


class _Clock:
    def __init__(self):
        self.t0 = time.perf_counter()

    def read(self) -> float:
        return time.perf_counter() - self.t0


def _promote(p: RegularizedProblem, x0) -> tuple[torch.Tensor, bool]:
    Xt, vec = dv.as_columns(x0, p.d)
    return Xt.clone(), vec


def _record(trace, clock, p, sol_t, t, m, k, dt, Xt, event):
    de = exact_error_dev(p, Xt, sol_t) if sol_t is not None else None
    trace.append(TraceRecord(t, m, k, float(dt), de, clock.read(), event))


def _sol_cols(sol: ExactSolution | None):
    return None if sol is None else sol.columns_dev()


def _ctx_stream():
    return dv.ctx().handle, dv.stream()


# ------------------------------------------------------------------- states
class _PcgState:
    """Columnwise PCG recursion (solvers.py:227-282) on device columns."""

    method = "pcg"

    def __init__(self, p: RegularizedProblem, P: Preconditioner, Xt: torch.Tensor, rho=None):
        self.p = p
        self.pb = p.descriptor()
        c, d = p.c, p.d
        z = lambda: torch.empty((c, d), dtype=dv.F64, device=Xt.device)  # noqa: E731
        self.x = Xt.clone()
        self.r, self.rt, self.pdir, self.Hp = z(), z(), z(), z()
        self.x_new, self.r_new, self.rt_new = z(), z(), z()
        self.dt_col = torch.empty(c, dtype=dv.F64, device=Xt.device)
        self.dt_new = torch.empty(c, dtype=dv.F64, device=Xt.device)
        self.delta_tilde = 0.0
        self.restart(P)

    def restart(self, P: Preconditioner) -> None:
        self.P = P
        h, s = _ctx_stream()
        out = C.c_double()
        _lib.check(_lib.lib().adask_pcg_restart(h, C.byref(self.pb), P.handle, self.x.data_ptr(),
                                                self.r.data_ptr(), self.rt.data_ptr(), self.pdir.data_ptr(),
                                                self.dt_col.data_ptr(), C.byref(out), s), "pcg_restart")
        self.delta_tilde = out.value

    def done(self) -> bool:
        return not bool((self.dt_col > 0.0).any())

    def propose(self):
        h, s = _ctx_stream()
        out = C.c_double()
        _lib.check(_lib.lib().adask_pcg_propose(h, C.byref(self.pb), self.P.handle, self.x.data_ptr(),
                                                self.r.data_ptr(), self.pdir.data_ptr(), self.dt_col.data_ptr(),
                                                self.Hp.data_ptr(), self.x_new.data_ptr(), self.r_new.data_ptr(),
                                                self.rt_new.data_ptr(), self.dt_new.data_ptr(), C.byref(out), s),
                   "pcg_propose")
        return out.value, None

    def commit(self, dt_scalar, stash) -> None:
        h, s = _ctx_stream()
        c, d = self.p.c, self.p.d
        _lib.check(_lib.lib().adask_pcg_commit(h, d, c, self.rt_new.data_ptr(), self.dt_new.data_ptr(),
                                               self.dt_col.data_ptr(), self.pdir.data_ptr(), s), "pcg_commit")
        self.x, self.x_new = self.x_new, self.x
        self.r, self.r_new = self.r_new, self.r
        self.rt, self.rt_new = self.rt_new, self.rt
        self.dt_col, self.dt_new = self.dt_new, self.dt_col
        self.delta_tilde = dt_scalar


class _IhsState:
    """Sketched Newton recursion (solvers.py:522-546) on device columns."""

    method = "ihs"

    def __init__(self, p: RegularizedProblem, P: Preconditioner, Xt: torch.Tensor, rho: float):
        self.p = p
        self.pb = p.descriptor()
        self.mu = 1.0 - rho
        self.beta = 0.0
        c, d = p.c, p.d
        z = lambda: torch.empty((c, d), dtype=dv.F64, device=Xt.device)  # noqa: E731
        self.x = Xt.clone()
        self.x_prev = None
        self.g, self.v, self.x_new, self.g_new, self.v_new = z(), z(), z(), z(), z()
        self.delta_tilde = 0.0
        self.restart(P)

    def restart(self, P: Preconditioner) -> None:
        self.P = P
        h, s = _ctx_stream()
        out = C.c_double()
        _lib.check(_lib.lib().adask_ihs_restart(h, C.byref(self.pb), P.handle, self.x.data_ptr(),
                                                self.g.data_ptr(), self.v.data_ptr(), C.byref(out), s),
                   "ihs_restart")
        self.delta_tilde = out.value

    def propose(self):
        h, s = _ctx_stream()
        out = C.c_double()
        xp = None if self.x_prev is None else self.x_prev.data_ptr()
        _lib.check(_lib.lib().adask_ihs_propose(h, C.byref(self.pb), self.P.handle, self.x.data_ptr(),
                                                self.v.data_ptr(), self.mu, xp, self.beta,
                                                self.x_new.data_ptr(), self.g_new.data_ptr(),
                                                self.v_new.data_ptr(), C.byref(out), s), "ihs_propose")
        return out.value, None

    def commit(self, dt_new, stash):
        self.x, self.x_new = self.x_new, self.x
        self.g, self.g_new = self.g_new, self.g
        self.v, self.v_new = self.v_new, self.v
        self.delta_tilde = dt_new


class _PolyakState(_IhsState):
    """Heavy-ball variant (solvers.py:549-571)."""

    method = "polyak"

    def __init__(self, p, P, Xt, rho):
        mu, beta = polyak_coefficients(rho)
        super().__init__(p, P, Xt, rho)
        self.mu, self.beta = mu, beta

    def restart(self, P):
        super().restart(P)
        self.x_prev = self.x.clone()  # momentum resets with the sketch

    def commit(self, dt_new, stash):
        # x_prev <- x; x <- x_new (buffers rotate)
        old_prev = self.x_prev
        self.x_prev = self.x
        self.x = self.x_new
        self.x_new = old_prev
        self.g, self.g_new = self.g_new, self.g
        self.v, self.v_new = self.v_new, self.v
        self.delta_tilde = dt_new


# ------------------------------------------------------------ fixed sketch
def _fixed_sketch_setup(p: RegularizedProblem, m, family, seed, s, tf32=False):
    SA = sketch_dev(p.A_dev, SketchSpec(family, m, seed, s=s), tf32=tf32)
    return build_dev(SA, p.nu, p.lam_dev)


def ihs_step(p: RegularizedProblem, P: Preconditioner, x, mu: float):
    """One sketched Newton update x - mu H_S^-1 grad f(x) (solvers.py:143-149)."""
    Xt, vec = dv.as_columns(x, p.d)
    st = _IhsState(p, P, Xt, 1.0 - mu)
    st.x_prev = None
    st.propose()
    return dv.from_columns(st.x_new, vec, x)


def ihs_run(p, x0, m, rho, family, seed, T, sol=None, s=1, *, tf32=False):
    """Sketch once, then x_{t+1} = x_t - (1 - rho) H_S^-1 grad (solvers.py:157-190)."""
    if not (0.0 < rho < 1.0):
        raise ValueError(f"rho must lie in (0, 1), got {rho}")
    clock = _Clock()
    P = _fixed_sketch_setup(p, m, family, seed, s, tf32)
    Xt, vec = _promote(p, x0)
    trace = SolverTrace()
    sol_t = _sol_cols(sol)
    st = _IhsState(p, P, Xt, rho)
    _record(trace, clock, p, sol_t, 0, m, 0, st.delta_tilde, st.x, "plain")
    for t in range(1, T + 1):
        dt, _ = st.propose()
        st.commit(dt, None)
        _record(trace, clock, p, sol_t, t, m, 0, dt, st.x, "plain")
    return dv.from_columns(st.x, vec, x0), trace


def pcg_run(p, x0, m, family, seed, T, tol=0.0, sol=None, s=1, *, tf32=False):
    """PCG with one sketched-Hessian preconditioner (solvers.py:193-224)."""
    clock = _Clock()
    P = _fixed_sketch_setup(p, m, family, seed, s, tf32)
    Xt, vec = _promote(p, x0)
    trace = SolverTrace()
    sol_t = _sol_cols(sol)
    state = _PcgState(p, P, Xt)
    _record(trace, clock, p, sol_t, 0, m, 0, state.delta_tilde, state.x, "plain")
    for t in range(1, T + 1):
        if state.done() or (tol > 0.0 and state.delta_tilde <= tol):
            break
        dt_new, stash = state.propose()
        state.commit(dt_new, stash)
        _record(trace, clock, p, sol_t, t, m, 0, state.delta_tilde, state.x, "plain")
    return dv.from_columns(state.x, vec, x0), trace


def polyak_coefficients(rho: float) -> tuple[float, float]:
    """Heavy-ball step and momentum (mu_rho, beta_rho) (solvers.py:285-290)."""
    if not (0.0 < rho < 1.0):
        raise ValueError(f"rho must lie in (0, 1), got {rho}")
    root = np.sqrt(1.0 - rho)
    return 2.0 * (1.0 - rho) / (1.0 + root), (1.0 - root) / (1.0 + root)


def polyak_ihs_run(p, x0, m, rho, family, seed, T, sol=None, s=1, *, tf32=False):
    """Sketched Newton with heavy-ball momentum (solvers.py:293-328)."""
    mu, beta = polyak_coefficients(rho)
    clock = _Clock()
    P = _fixed_sketch_setup(p, m, family, seed, s, tf32)
    Xt, vec = _promote(p, x0)
    trace = SolverTrace()
    sol_t = _sol_cols(sol)
    st = _PolyakState(p, P, Xt, rho)
    _record(trace, clock, p, sol_t, 0, m, 0, st.delta_tilde, st.x, "plain")
    for t in range(1, T + 1):
        dt, _ = st.propose()
        st.commit(dt, None)
        _record(trace, clock, p, sol_t, t, m, 0, dt, st.x, "plain")
    return dv.from_columns(st.x, vec, x0), trace


def cg(p, x0, T, tol=0.0, sol=None):
    """Conjugate gradient on H x = b, columnwise (solvers.py:104-140): the
    fused PCG bodies with the identity preconditioner -- the Woodbury path of
    an all-zero 1 x d sketch with nu = 1, lam = 1, so H_S = I exactly and the
    trace's delta_tilde is (1/2)||r||_F^2 as in the reference.  Stops after T
    iterations or once that value falls to tol."""
    clock = _Clock()
    Xt, vec = _promote(p, x0)
    P = build_dev(torch.zeros((1, p.d), dtype=p.A_dev.dtype, device=Xt.device), 1.0,
                  torch.ones(p.d, dtype=dv.F64, device=Xt.device))
    trace = SolverTrace()
    sol_t = _sol_cols(sol)
    state = _PcgState(p, P, Xt)
    _record(trace, clock, p, sol_t, 0, 0, 0, state.delta_tilde, state.x, "plain")
    for t in range(1, T + 1):
        if state.done() or state.delta_tilde <= tol:
            break
        dt_new, stash = state.propose()
        state.commit(dt_new, stash)
        _record(trace, clock, p, sol_t, t, 0, 0, state.delta_tilde, state.x, "plain")
    return dv.from_columns(state.x, vec, x0), trace


# ------------------------------------------------------------------ adaptive
_METHODS = ("ihs", "pcg", "polyak")


def _method_constants(method: str, rho: float) -> tuple[float, float]:
    """(alpha, phi(rho)) for the adaptive acceptance threshold (solvers.py:453-462)."""
    if method == "ihs":
        return 1.0, rho
    if method == "pcg":
        root = np.sqrt(1.0 - rho)
        return 4.0, (1.0 - root) / (1.0 + root)
    if method == "polyak":
        return 1.0, polyak_coefficients(rho)[1]
    raise ValueError(f"unknown method {method!r}; expected one of {_METHODS}")


@dataclass
class AdaptiveConfig:
    """Knobs for adaptive_run (solvers.py:465-519).  Build with for_method so
    that (alpha, phi_rho, c_alpha_rho) stay consistent with the solver."""

    rho: float
    m_init: int
    T: int
    family: str
    seed: int
    alpha: float
    phi_rho: float
    c_alpha_rho: float
    s: int = 1

    def __post_init__(self):
        if not (0.0 < self.rho < 1.0):
            raise ValueError(f"rho must lie in (0, 1), got {self.rho}")
        if self.m_init < 1:
            raise ValueError(f"m_init must be >= 1, got {self.m_init}")
        if self.T < 0:
            raise ValueError(f"T must be >= 0, got {self.T}")
        sq = np.sqrt(self.rho)
        expected_c = (1.0 + sq) / (1.0 - sq) * self.alpha
        if abs(self.c_alpha_rho - expected_c) > 1e-12 * max(1.0, abs(expected_c)):
            raise ValueError(
                f"c_alpha_rho = {self.c_alpha_rho} inconsistent with alpha = "
                f"{self.alpha} and rho = {self.rho} (expected {expected_c})"
            )
        if self.rho >= 0.25:
            warnings.warn(
                f"rho = {self.rho} is outside the guaranteed range (0, 1/4); "
                "the adaptive bounds may not hold",
                UserWarning,
            )

    @property
    def rho_in_guarantee_range(self) -> bool:
        return self.rho < 0.25

    @classmethod
    def for_method(cls, method, rho, m_init, T, family, seed, s=1) -> "AdaptiveConfig":
        alpha, phi = _method_constants(method, rho)
        sq = np.sqrt(rho)
        c = (1.0 + sq) / (1.0 - sq) * alpha
        return cls(rho, m_init, T, family, seed, alpha, phi, c, s=s)


def heavy_ball_bound(t, rho: float) -> float:
    """Per-iteration heavy-ball envelope (solvers.py:331-355); scalar."""
    if not (0.0 < rho < 1.0):
        raise ValueError(f"rho must lie in (0, 1), got {rho}")
    _, beta = polyak_coefficients(rho)
    if np.isinf(t):
        return float(beta)
    if t < 1:
        raise ValueError(f"t must be >= 1, got {t}")
    nu_t = np.log2(t) + 1.0
    omega = t - 2.0 * nu_t
    logv = (nu_t * (nu_t + 1.0) * np.log(3.0) + 2.0 * nu_t * np.log1p(4.0 * beta + beta * beta)
            + omega * np.log(beta))
    return float(np.exp(logv / t))


def _segment_threshold(cfg: AdaptiveConfig, method: str, ell: int) -> float:
    """Acceptance threshold for a segment of ell steps (solvers.py:574-582)."""
    if method == "polyak":
        sq = np.sqrt(cfg.rho)
        c_geom = (1.0 + sq) / (1.0 - sq)
        return c_geom * heavy_ball_bound(ell, cfg.rho) ** ell
    return cfg.c_alpha_rho * cfg.phi_rho**ell


def _adaptive_sketch(p: RegularizedProblem, cfg: AdaptiveConfig, m: int, K: int, sketcher, tf32: bool):
    spec = SketchSpec(cfg.family, m, derive_seed(cfg.seed, K), s=cfg.s)
    if sketcher is not None:
        return sketcher(p, spec)
    return sketch_dev(p.A_dev, spec, tf32=tf32)


_FAMILY_CODE = {"gaussian": 0, "srht": 1, "sjlt": 2, "srht-block": 3}
_EVENTS = ("plain", "accepted", "resketch")


def _adaptive_native(p: RegularizedProblem, x0, cfg: AdaptiveConfig, method: str, sol, tf32: bool,
                     block: int, incremental: bool = False):
    """The same algorithm as the Python loop below, run by libadask's native
    driver (adask_adaptive_run): no Python / ctypes round trips per pass."""
    Xt, vec = _promote(p, x0)
    xout = torch.empty_like(Xt)
    c = _lib.AdaptiveCfg()
    c.method = _METHODS.index(method)
    c.family = _FAMILY_CODE[cfg.family]
    c.rho, c.m_init, c.T, c.seed, c.s = float(cfg.rho), int(cfg.m_init), int(cfg.T), int(cfg.seed), int(cfg.s)
    c.alpha, c.phi_rho, c.c_alpha_rho = float(cfg.alpha), float(cfg.phi_rho), float(cfg.c_alpha_rho)
    c.block, c.row0, c.n_total = int(block), int(p.row0), int(p.n_total)
    c.flags = (_lib.TF32 if tf32 else 0) | (_lib.INCREMENTAL if incremental else 0)
    if method == "polyak":
        c.phi_rho = 0.0  # the polyak threshold is evaluated on the host (see below)
    nmax = 3 * int(cfg.T) + 200
    recs = (_lib.TraceRec * nmax)()
    nrec = C.c_int64()
    xs = _sol_cols(sol)
    pb = p.descriptor()
    _lib.check(_lib.lib().adask_adaptive_run(dv.ctx().handle, C.byref(pb), C.byref(c), Xt.data_ptr(),
                                             xout.data_ptr(), None if xs is None else xs.data_ptr(), recs,
                                             nmax, C.byref(nrec), dv.stream()), "adaptive_run")
    trace = SolverTrace()
    for r in recs[:nrec.value]:
        trace.append(TraceRecord(int(r.t), int(r.m), int(r.k), float(r.delta_tilde),
                                 float(r.delta_exact) if r.has_exact else None, float(r.wall_seconds),
                                 _EVENTS[r.event]))
    return dv.from_columns(xout, vec, x0), trace


def adaptive_run(p: RegularizedProblem, x0, cfg: AdaptiveConfig, method: str = "pcg",
                 sol: ExactSolution | None = None, experimental: bool = False, *,
                 tf32: bool = False, sketcher=None, block: int = 1 << 21, native: bool | None = None,
                 incremental: bool = False):
    """Run a sketched method with on-line sketch-size adaptation
    (solvers.py:585-659).  Keyword-only extras: tf32 (fp32 Gaussian sketch on
    tensor cores), block (rows per block for family "srht-block", config 4),
    sketcher(p, spec) -> SA device tensor (custom sketches; forces the Python
    loop), native (default: the libadask driver whenever no custom sketcher
    is given; set ADASK_PY_DRIVER=1 to force the Python loop), incremental
    (grow the sketch when m doubles instead of redrawing it: Gaussian keeps
    its rows and adds new ones, SRHT keeps its transform and adds sampled
    rows; not reference semantics -- the oracle's adaptive_run has the same
    mode -- native driver only)."""
    if method not in _METHODS:
        raise ValueError(f"unknown method {method!r}; expected one of {_METHODS}")
    if method == "polyak" and not experimental:
        raise ValueError("method 'polyak' is experimental; pass experimental=True")
    if native is None:
        native = (sketcher is None and method != "polyak" and 0 <= int(cfg.seed) < 2**64
                  and not (cfg.family == "gaussian" and gaussian_rng() == "numpy")
                  and cfg.family in _FAMILY_CODE and os.environ.get("ADASK_PY_DRIVER") != "1")
    if incremental:
        if sketcher is not None or method == "polyak":
            raise ValueError("incremental sketch growth runs on the native driver (no custom sketcher / polyak)")
        return _adaptive_native(p, x0, cfg, method, sol, tf32, block, incremental=True)
    if native:
        return _adaptive_native(p, x0, cfg, method, sol, tf32, block)
    if sketcher is None and cfg.family == "srht-block":
        from .parallel import block_srht_sketcher

        sketcher = block_srht_sketcher(block)
    clock = _Clock()
    Xt, vec = _promote(p, x0)
    cap = padded_rows(p.n_total) if cfg.family == "srht" else p.n_total
    if cfg.family == "srht-block":
        cap = min(cap, padded_rows(min(block, p.n_total)))  # each block sketch needs m <= padded rows
    m = min(cfg.m_init, cap)
    K = 0
    SA = _adaptive_sketch(p, cfg, m, K, sketcher, tf32)
    P = build_dev(SA, p.nu, p.lam_dev)
    state = {"ihs": _IhsState, "pcg": _PcgState, "polyak": _PolyakState}[method](p, P, Xt, cfg.rho)
    trace = SolverTrace()
    sol_t = _sol_cols(sol)
    dt_first = state.delta_tilde
    dt_I = state.delta_tilde
    t = 0
    I = 0  # noqa: E741
    capped_retry = False
    _record(trace, clock, p, sol_t, 0, m, 0, state.delta_tilde, state.x, "plain")
    while t < cfg.T:
        dt_new, stash = state.propose()
        ell = t + 1 - I
        threshold = _segment_threshold(cfg, method, ell)
        converged = dt_I <= 0.0 or dt_new <= _CONVERGED_REL * dt_first
        reject = (not converged) and dt_new > threshold * dt_I
        if reject and capped_retry:
            reject = False  # m already at cap and one redraw failed: accept
        if reject:
            K += 1
            at_cap = m >= cap
            m = min(2 * m, cap)
            capped_retry = at_cap
            del P
            SA = _adaptive_sketch(p, cfg, m, K, sketcher, tf32)
            P = build_dev(SA, p.nu, p.lam_dev)
            state.restart(P)
            dt_I = state.delta_tilde
            I = t  # noqa: E741
            _record(trace, clock, p, sol_t, t, m, K, dt_I, state.x, "resketch")
        else:
            state.commit(dt_new, stash)
            t += 1
            capped_retry = False
            _record(trace, clock, p, sol_t, t, m, K, state.delta_tilde, state.x, "accepted")
    return dv.from_columns(state.x, vec, x0), trace
