"""Quadratically regularized least-squares problems (device resident).

Drop-in for the hot part of adasketch/problem.py:41-158.  The objective is
f(x) = (1/2) <x, H x> - <b, x> with H = A.T A + nu^2 Lambda.  A lives in HBM
(float64 by default like the reference, problem.py:51; dtype="float32" for
the fp32 configurations); H X is one fused pass over A per column
(libadask adask_hess_mult).  Error quantities are summed over columns.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from . import device as dv
from .errors import DimensionMismatch

__all__ = ["RegularizedProblem", "ExactSolution", "direct_solve", "exact_error"]


class RegularizedProblem:
    """Data matrix A (n x d), targets B (d x c), scale nu, diagonal lam
    (problem.py:41-111).  Keyword-only extras: dtype (matrix precision),
    row0 / n_total (this object holds rows [row0, row0+n) of a row-sharded A)."""

    def __init__(self, A, B, nu: float, lam=None, *, dtype=None, row0: int = 0,
                 n_total: int | None = None, validate: bool = True):
        t = dv.resolve_dtype(dtype) if dtype is not None else (
            A.dtype if isinstance(A, torch.Tensor) and A.dtype in (dv.F64, dv.F32) else dv.F64)
        self._like = A
        self._A_host = A if isinstance(A, np.ndarray) and A.dtype == np.float64 and A.ndim == 2 else None
        self.A_dev = dv.to_device(A, t)
        if self.A_dev.dim() != 2:
            raise DimensionMismatch(f"A must be 2-D, got shape {tuple(self.A_dev.shape)}")
        n, d = self.A_dev.shape
        Bd = dv.to_device(B, dv.F64)
        if Bd.dim() == 1:
            Bd = Bd[:, None]
        if Bd.shape[0] != d:
            raise DimensionMismatch(f"B has {Bd.shape[0]} rows, expected d = {d}")
        self.Bt = Bd.t().contiguous()  # c x d
        self.nu = float(nu)
        if not np.isfinite(self.nu) or self.nu <= 0:
            raise ValueError(f"nu must be positive and finite, got {self.nu}")
        lam_d = torch.ones(d, dtype=dv.F64, device=self.A_dev.device) if lam is None else dv.to_device(lam, dv.F64)
        if tuple(lam_d.shape) != (d,):
            raise DimensionMismatch(f"lam must have shape ({d},), got {tuple(lam_d.shape)}")
        self.lam_dev = lam_d.contiguous()
        if validate:
            # one pass over A on the device (csrc/check.cu), one synchronization
            verdict = (C.c_int * 3)()
            _lib.check(_lib.lib().adask_check_problem(
                dv.ctx().handle, dv.dtype_code(self.A_dev.dtype), self.A_dev.data_ptr(), n, d,
                self.A_dev.stride(0) if n > 0 else d, self.Bt.data_ptr(), self.Bt.numel(), self.lam_dev.data_ptr(),
                d, verdict, dv.stream()), "check_problem")
            if verdict[2]:
                raise ValueError("lam entries must be finite and >= 1")
            if verdict[0] or verdict[1]:
                raise ValueError("A and B must be finite")
        self.row0 = int(row0)
        self.n_total = n if n_total is None else int(n_total)

    # ---- reference properties
    @property
    def A(self):
        """The data matrix like the caller passed it: numpy float64 for a
        numpy input (the reference's cast, problem.py:51), else the device
        tensor.  The solvers use A_dev."""
        if isinstance(self._like, torch.Tensor):
            return self.A_dev
        if self._A_host is None:
            self._A_host = dv.to_host_like(self.A_dev, self._like)
        return self._A_host

    @property
    def n(self) -> int:
        return self.A_dev.shape[0]

    @property
    def d(self) -> int:
        return self.A_dev.shape[1]

    @property
    def c(self) -> int:
        return self.Bt.shape[0]

    @property
    def B(self):
        return dv.to_host_like(self.Bt.t(), self._like)

    @property
    def lam(self):
        return dv.to_host_like(self.lam_dev, self._like)

    @property
    def dtype(self) -> torch.dtype:
        return self.A_dev.dtype

    def descriptor(self) -> _lib.Problem:
        pb = _lib.Problem()
        pb.dtype = dv.dtype_code(self.A_dev.dtype)
        pb.A = self.A_dev.data_ptr()
        pb.n, pb.d = self.A_dev.shape
        pb.lda = self.A_dev.stride(0)
        pb.c = self.c
        pb.nu2 = self.nu**2
        pb.lam = self.lam_dev.data_ptr()
        pb.B = self.Bt.data_ptr()
        return pb

    # ---- device-layout kernels (c x d columns)
    def hess_mult_dev(self, Xt: torch.Tensor, out: torch.Tensor | None = None, *, minus_B: bool = False,
                      partial: bool = False) -> torch.Tensor:
        Xt = Xt.contiguous()
        c, d = Xt.shape
        if d != self.d:
            raise DimensionMismatch(f"iterate has {d} rows, expected {self.d}")
        out = torch.empty_like(Xt) if out is None else out
        B = self.Bt if minus_B else None
        _lib.check(_lib.lib().adask_hess_mult(dv.ctx().handle, dv.dtype_code(self.A_dev.dtype), self.A_dev.data_ptr(),
                                              self.n, d, self.A_dev.stride(0), Xt.data_ptr(), c, d,
                                              self.nu**2, self.lam_dev.data_ptr(),
                                              None if B is None else B.data_ptr(), d, out.data_ptr(), d,
                                              _lib.PARTIAL if partial else 0, dv.stream()),
                   "hess_mult")
        return out

    # ---- reference API
    def hess_mult(self, X):
        """H @ X without forming H, one pass over A per column (problem.py:89-95)."""
        Xt, vec = dv.as_columns(X, self.d)
        return dv.from_columns(self.hess_mult_dev(Xt), vec, X)

    def gradient(self, X):
        """grad f(x) = H x - b, columnwise (problem.py:97-107)."""
        Xt, vec = dv.as_columns(X, self.d)
        if Xt.shape != (self.c, self.d):
            shape = tuple(X.shape) if hasattr(X, "shape") else np.shape(X)
            raise DimensionMismatch(f"iterate has shape {shape}, expected ({self.d}, {self.c})")
        return dv.from_columns(self.hess_mult_dev(Xt, minus_B=True), vec, X)

    def hessian(self):
        """Dense d x d Hessian (problem.py:109-111)."""
        from .preconditioner import gram_dev

        return dv.to_host_like(gram_dev(self.A_dev, self.nu**2, self.lam_dev), self._like)


@dataclass
class ExactSolution:
    """Minimizer x_star (d x c) of the regularized objective (problem.py:114-123)."""

    x_star: object

    def __post_init__(self):
        if isinstance(self.x_star, torch.Tensor):
            if self.x_star.dim() == 1:
                self.x_star = self.x_star[:, None]
        else:
            self.x_star = np.asarray(self.x_star, dtype=np.float64)
            if self.x_star.ndim == 1:
                self.x_star = self.x_star[:, None]

    def columns_dev(self) -> torch.Tensor:
        return dv.to_device(self.x_star, dv.F64).t().contiguous()


def direct_solve(p: RegularizedProblem) -> ExactSolution:
    """Solve H x = B by a dense Cholesky factorization of H (problem.py:144-149).
    fp64 data: the preconditioner built from A itself (H_S = H, m = n >= d).
    fp32 data: H is accumulated in fp64 over row blocks of A (each block
    widened to fp64, Gram by libadask), then an fp64 Cholesky and two
    triangular solves -- the exact solution for configs 3-4."""
    from .linalg import cholesky, tri_solve
    from .preconditioner import build_dev

    if p.n < p.d:
        raise DimensionMismatch("direct_solve needs n >= d on the device path")
    if p.A_dev.dtype == dv.F64:
        P = build_dev(p.A_dev, p.nu, p.lam_dev)
        X = P.solve_dev(p.Bt)
        return ExactSolution(x_star=dv.to_host_like(X.t().contiguous(), p._like))
    H = gram_fp64(p.A_dev, p.nu**2, p.lam_dev)
    L = cholesky(H)
    Y = tri_solve(L, p.Bt.t().contiguous())
    X = tri_solve(L, Y, transposed=True)
    return ExactSolution(x_star=dv.to_host_like(X, p._like))


def gram_fp64(A: torch.Tensor, nu2: float = 0.0, lam: torch.Tensor | None = None) -> torch.Tensor:
    """A^T A (+ nu2 diag(lam)) in fp64 for an fp32 or fp64 A: one DMMA Gram
    (fp32 entries widened at the fragment load, fp64 accumulation)."""
    A = A if A.stride(1) == 1 else A.contiguous()
    n, d = A.shape
    H = torch.empty((d, d), dtype=dv.F64, device=A.device)
    _lib.check(_lib.lib().adask_gram_ex(dv.ctx().handle, dv.dtype_code(A.dtype), A.data_ptr(), n, d, A.stride(0),
                                        float(nu2), None if lam is None else lam.data_ptr(), dv.dtype_code(dv.F64),
                                        H.data_ptr(), d, dv.stream()), "gram")
    return H


def exact_error_dev(p: RegularizedProblem, Xt: torch.Tensor, Xstar_t: torch.Tensor) -> float:
    """delta_x = (1/2) ||x - x*||_H^2 summed over columns, on device columns."""
    diff = Xt - Xstar_t
    Hd = p.hess_mult_dev(diff)
    c, d = diff.shape
    val = C.c_double()
    _lib.check(_lib.lib().adask_dot(dv.ctx().handle, diff.data_ptr(), Hd.data_ptr(), d, c, d,
                                    C.byref(val), dv.stream()), "dot")
    return float(val.value)


def exact_error(p: RegularizedProblem, x, sol: ExactSolution) -> float:
    """delta_x = (1/2) ||x - x_star||_H^2, summed over columns (problem.py:152-158)."""
    Xt, _ = dv.as_columns(x, p.d)
    return exact_error_dev(p, Xt, sol.columns_dev())
