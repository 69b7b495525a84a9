"""Device-side array plumbing for the drop-in API.

The reference takes array-likes, casts them to float64 and returns numpy
arrays (solvers.py:84-88, problem.py:51).  Here every public entry point
accepts numpy arrays or torch tensors; compute runs on the CUDA device via
libadask, and results come back in the caller's kind: numpy in -> numpy out,
torch in -> torch (device) out.  d x c blocks of right-hand sides are held on
the device transposed (c x d, each column contiguous), which is the layout
the C ABI expects.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _lib

F64 = torch.float64
F32 = torch.float32


def device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2104_14101_b200 needs a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def ctx() -> _lib.Context:
    return _lib.Context.get(device().index)


def stream() -> int:
    return _lib.stream_ptr()


def dtype_code(t: torch.dtype) -> int:
    if t == F64:
        return _lib.F64
    if t == F32:
        return _lib.F32
    raise TypeError(f"unsupported dtype {t}")


def resolve_dtype(dtype) -> torch.dtype:
    if dtype is None:
        return F64
    if isinstance(dtype, torch.dtype):
        if dtype in (F64, F32):
            return dtype
    else:
        s = str(np.dtype(dtype)) if not isinstance(dtype, str) else dtype
        if s in ("float64", "f64", "double"):
            return F64
        if s in ("float32", "f32", "float"):
            return F32
    raise TypeError(f"unsupported dtype {dtype!r}; use float64 or float32")


def is_torch(x) -> bool:
    return isinstance(x, torch.Tensor)


def to_device(x, dtype: torch.dtype = F64, contiguous: bool = True) -> torch.Tensor:
    """Array-like -> CUDA tensor of `dtype` (copies only when needed)."""
    dev = device()
    if isinstance(x, torch.Tensor):
        t = x.to(device=dev, dtype=dtype)
    else:
        arr = np.asarray(x)
        if arr.dtype == object:
            arr = arr.astype(np.float64)
        t = torch.from_numpy(np.ascontiguousarray(arr)).to(device=dev, dtype=dtype)
    return t.contiguous() if contiguous else t


def as_columns(X, d: int) -> tuple[torch.Tensor, bool]:
    """d or d x c array -> (c x d float64 device tensor, was_vector)."""
    if isinstance(X, torch.Tensor):
        t = X.to(device=device(), dtype=F64)
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(X, dtype=np.float64))).to(device())
    vec = t.dim() == 1
    if vec:
        t = t[None, :]
    else:
        t = t.t()
    return t.contiguous(), vec


def from_columns(Xt: torch.Tensor, vec: bool, like):
    """c x d device tensor -> d (vec) or d x c, in the kind of `like`."""
    out = Xt[0] if vec else Xt.t()
    if isinstance(like, torch.Tensor):
        return out.contiguous()
    return out.detach().cpu().numpy().copy()


def to_host_like(t: torch.Tensor, like):
    if isinstance(like, torch.Tensor):
        return t
    return t.detach().cpu().numpy()


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()
