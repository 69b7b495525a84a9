"""Sketched-Hessian preconditioner H_S = (SA).T (SA) + nu^2 Lambda.

Drop-in for adasketch/preconditioner.py:26-88.  Two factorization paths,
chosen by shape exactly like the reference (m >= d, ties included, factors
the d x d H_S; m < d factors the m x m capacitance matrix
W_S = SA Lam^-1 SA.T + nu^2 I and solves through the matrix inversion
identity).  The Gram/capacitance GEMM, the Cholesky factorization, the
triangular inverse and every solve run on the device (libadask).
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from . import device as dv
from .embeddings import SketchedData
from .errors import NegativeValue

__all__ = ["Preconditioner", "build", "approx_newton_decrement"]

PATHS = ("cholesky-d", "woodbury-m")


class Preconditioner:
    """Factored H_S.  Attributes mirror the reference dataclass
    (preconditioner.py:26-32): SA, nu, lam, path, L (L is fetched from the
    device on first access)."""

    def __init__(self, handle: C.c_void_p, SA_dev: torch.Tensor, nu: float, lam_dev: torch.Tensor,
                 like=None):
        self._h = handle
        self._SA = SA_dev  # kept alive: the Woodbury solve reads it
        self._lam = lam_dev
        self.nu = float(nu)
        self._like = like
        self.path = PATHS[_lib.lib().adask_precond_path(handle)]
        self._L = None

    # ---- reference attributes
    @property
    def SA(self):
        return dv.to_host_like(self._SA, self._like) if self._like is not None else self._SA

    @property
    def lam(self):
        return dv.to_host_like(self._lam, self._like) if self._like is not None else self._lam

    @property
    def L(self):
        if self._L is None:
            k = C.c_int64()
            dt = C.c_int()
            _lib.check(_lib.lib().adask_precond_factor(self._h, None, C.byref(k), C.byref(dt)))
            tdt = dv.F64 if dt.value == _lib.F64 else dv.F32
            Ld = torch.empty((k.value, k.value), dtype=tdt, device=self._SA.device)
            _lib.check(_lib.lib().adask_precond_copy_factor(dv.ctx().handle, self._h, 0, Ld.data_ptr(),
                                                            k.value, dv.stream()), "copy_factor")
            self._L = Ld
        return dv.to_host_like(self._L, self._like) if self._like is not None else self._L

    @property
    def m(self) -> int:
        return self._SA.shape[0]

    @property
    def d(self) -> int:
        return self._SA.shape[1]

    @property
    def handle(self):
        return self._h

    def solve_dev(self, Zt: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        """H_S^-1 on c x d device columns."""
        Zt = Zt.contiguous()
        c, d = Zt.shape
        if d != self.d:
            from .errors import DimensionMismatch

            raise DimensionMismatch(f"rhs has {d} rows, expected {self.d}")
        out = torch.empty_like(Zt) if out is None else out
        _lib.check(_lib.lib().adask_precond_apply(dv.ctx().handle, self._h, Zt.data_ptr(), c, d,
                                                  out.data_ptr(), d, dv.stream()), "precond_apply")
        return out

    def solve(self, Z):
        """H_S^-1 Z, columnwise (preconditioner.py:42-53)."""
        Zt, vec = dv.as_columns(Z, self.d)
        return dv.from_columns(self.solve_dev(Zt), vec, Z)

    def sketched_hessian(self):
        """Dense H_S; d x d (preconditioner.py:55-57)."""
        H = gram_dev(self._SA, self.nu**2, self._lam)
        return dv.to_host_like(H, self._like) if self._like is not None else H

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib._lib is not None:
            try:
                _lib.lib().adask_precond_destroy(h)
            except Exception:
                pass
            self._h = None


def gram_dev(A: torch.Tensor, nu2: float, lam: torch.Tensor | None) -> torch.Tensor:
    """Dense symmetric A.T A + nu2 diag(lam) on the device (libadask DMMA Gram)."""
    A = A.contiguous()
    n, d = A.shape
    H = torch.empty((d, d), dtype=A.dtype, device=A.device)
    _lib.check(_lib.lib().adask_gram(dv.ctx().handle, dv.dtype_code(A.dtype), A.data_ptr(), n, d,
                                     A.stride(0), float(nu2), None if lam is None else lam.data_ptr(),
                                     H.data_ptr(), d, dv.stream()), "gram")
    return H


def woodbury_gram_dev(SA: torch.Tensor, nu2: float, lam: torch.Tensor) -> torch.Tensor:
    """W_S = (SA * (1/lam)) SA^T + nu2 I (preconditioner.py:72-73), symmetric m x m."""
    SA = SA if SA.stride(1) == 1 else SA.contiguous()
    m, d = SA.shape
    W = torch.empty((m, m), dtype=SA.dtype, device=SA.device)
    _lib.check(_lib.lib().adask_gram_woodbury(dv.ctx().handle, dv.dtype_code(SA.dtype), SA.data_ptr(), m, d,
                                              SA.stride(0), float(nu2), lam.data_ptr(), W.data_ptr(), m,
                                              dv.stream()), "gram_woodbury")
    return W


def build_dev(SA_dev: torch.Tensor, nu: float, lam_dev: torch.Tensor, like=None) -> Preconditioner:
    m, d = SA_dev.shape
    SA_dev = SA_dev.contiguous()
    h = C.c_void_p()
    info = C.c_int64(0)
    _lib.check(_lib.lib().adask_precond_build(dv.ctx().handle, dv.dtype_code(SA_dev.dtype), SA_dev.data_ptr(),
                                              m, d, SA_dev.stride(0), float(nu), lam_dev.data_ptr(),
                                              C.byref(h), C.byref(info), dv.stream()), "build")
    return Preconditioner(h, SA_dev, nu, lam_dev, like)


def build(sa, nu: float, lam, *, dtype=None) -> Preconditioner:
    """Factor H_S from sketched data (SketchedData or a raw m x d array);
    ties at m = d take the dense d-path (preconditioner.py:60-74)."""
    raw = sa.SA if isinstance(sa, SketchedData) else sa
    like = None if isinstance(raw, torch.Tensor) else np.empty(0)
    if isinstance(raw, torch.Tensor):
        t = dtype if dtype is not None else (raw.dtype if raw.dtype in (dv.F64, dv.F32) else dv.F64)
    else:
        t = dv.resolve_dtype(dtype)
    SA_dev = dv.to_device(raw, t)
    if SA_dev.dim() != 2:
        from .errors import DimensionMismatch

        raise DimensionMismatch(f"SA must be 2-D, got shape {tuple(SA_dev.shape)}")
    lam_dev = dv.to_device(lam, dv.F64).reshape(-1)
    if lam_dev.shape[0] != SA_dev.shape[1]:
        from .errors import DimensionMismatch

        raise DimensionMismatch(f"lam must have shape ({SA_dev.shape[1]},)")
    return build_dev(SA_dev, nu, lam_dev, like)


def approx_newton_decrement(P: Preconditioner, grad) -> float:
    """delta_tilde = (1/2) trace(grad.T H_S^-1 grad) with the NegativeValue
    guard at -1e-12 ||grad||_F^2 (preconditioner.py:77-88)."""
    Gt, _ = dv.as_columns(grad, P.d)
    V = P.solve_dev(Gt)
    c, d = Gt.shape
    val = C.c_double()
    _lib.check(_lib.lib().adask_dot(dv.ctx().handle, Gt.data_ptr(), V.data_ptr(), d, c, d,
                                    C.byref(val), dv.stream()), "dot")
    val = 2.0 * val.value * 0.5  # adask_dot returns 0.5 * sum
    sq = C.c_double()
    _lib.check(_lib.lib().adask_dot(dv.ctx().handle, Gt.data_ptr(), Gt.data_ptr(), d, c, d,
                                    C.byref(sq), dv.stream()), "dot")
    floor = 1e-12 * (2.0 * sq.value)
    if val < -floor:
        raise NegativeValue(f"quadratic form {val} below -1e-12 * ||grad||^2")
    return max(val, 0.0)
