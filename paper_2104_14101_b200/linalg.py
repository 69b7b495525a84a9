"""Dense factorizations and transforms (drop-in for adasketch/linalg.py:20-88),
computed on the device by libadask."""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from . import device as dv
from .errors import DimensionMismatch, NotPowerOfTwo

__all__ = ["cholesky", "tri_solve", "fwht", "is_power_of_two"]

_SYM_RTOL = 1e-12


def is_power_of_two(n: int) -> bool:
    return n >= 1 and (n & (n - 1)) == 0


def _square(M, name: str) -> torch.Tensor:
    t = dv.to_device(M, M.dtype if isinstance(M, torch.Tensor) and M.dtype in (dv.F64, dv.F32) else dv.F64)
    if t.dim() != 2 or t.shape[0] != t.shape[1]:
        raise DimensionMismatch(f"{name} must be square, got shape {tuple(t.shape)}")
    return t


def cholesky(M):
    """Lower-triangular L with L L.T == M (linalg.py:30-44): asymmetry beyond
    1e-12 relative is rejected, M is symmetrized, non-SPD raises
    NotPositiveDefinite."""
    Md = _square(M, "M")
    scale = float(Md.abs().max()) if Md.numel() else 0.0
    if scale > 0 and float((Md - Md.t()).abs().max()) > _SYM_RTOL * scale:
        raise DimensionMismatch("matrix is not symmetric within 1e-12 relative")
    Ms = ((Md + Md.t()) / 2.0).contiguous()
    k = Ms.shape[0]
    L = torch.empty_like(Ms)
    info = C.c_int64(0)
    _lib.check(_lib.lib().adask_cholesky(dv.ctx().handle, dv.dtype_code(Ms.dtype), Ms.data_ptr(), k, k,
                                         L.data_ptr(), None, C.byref(info), dv.stream()), "cholesky")
    return dv.to_host_like(L, M)


def tri_solve(L, z, transposed: bool = False):
    """Solve L y = z (or L.T y = z) for lower-triangular L (linalg.py:47-55)."""
    Ld = _square(L, "L")
    k = Ld.shape[0]
    if np.ndim(z) == 0 or np.shape(z)[0] != k:
        raise DimensionMismatch(f"rhs has leading dimension {np.shape(z)[0] if np.ndim(z) else 0}, "
                                f"factor is {k}")
    zt, vec = dv.as_columns(z, k)
    Yt = torch.empty_like(zt)
    c = zt.shape[0]
    _lib.check(_lib.lib().adask_tri_solve(dv.ctx().handle, dv.dtype_code(Ld.dtype), Ld.data_ptr(), k,
                                          Ld.stride(0), 1 if transposed else 0, zt.data_ptr(), c, k,
                                          Yt.data_ptr(), k, dv.stream()), "tri_solve")
    return dv.from_columns(Yt, vec, z)


def fwht(x, normalized: bool = True):
    """Natural-order Walsh-Hadamard transform along axis 0 (linalg.py:62-88)."""
    like = x
    t = x.dtype if isinstance(x, torch.Tensor) and x.dtype in (dv.F64, dv.F32) else dv.F64
    X = dv.to_device(x, t)
    n = X.shape[0]
    if not is_power_of_two(n):
        raise NotPowerOfTwo(f"length {n} is not a power of two")
    squeeze = X.dim() == 1
    Y = X.reshape(n, -1).clone().contiguous()
    _lib.check(_lib.lib().adask_fwht(dv.ctx().handle, dv.dtype_code(Y.dtype), Y.data_ptr(), n, Y.shape[1],
                                     Y.stride(0), 1 if normalized else 0, dv.stream()), "fwht")
    Y = Y[:, 0] if squeeze else Y
    return dv.to_host_like(Y, like)
