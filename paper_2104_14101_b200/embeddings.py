"""Randomized embeddings: Gaussian, SRHT, and sparse (SJLT) sketches.

Drop-in for adasketch/embeddings.py.  Same names and signatures; the sketch
S*A is computed on the B200 by libadask:

* sketch_srht / sketch_sjlt consume numpy's PCG64 stream exactly (signs,
  buckets, SRHT row subsample), so their SA is bitwise equal to the
  reference's in fp64 (embeddings.py:81-129).
* sketch_gaussian draws S from Philox4x32-10 (shard-invariant, generated on
  the device) instead of numpy's ziggurat, by design (BASELINE north_star);
  entries are N(0, 1/m) like embeddings.py:66-73.  `gaussian_matrix` exposes
  the exact S for oracle comparison.

Keyword-only extras (not in the reference): dtype= (float64 default, or
float32), tf32= (fp32 Gaussian on tensor cores), accumulate_into=.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from . import device as dv
from .errors import InvalidProbability, InvalidSparsity, SketchTooLarge

__all__ = [
    "SketchSpec",
    "SketchedData",
    "sketch",
    "sketch_gaussian",
    "sketch_srht",
    "sketch_sjlt",
    "critical_m_srht",
    "critical_m_gaussian",
    "padded_rows",
    "derive_seed",
    "gaussian_matrix",
]

FAMILIES = ("gaussian", "srht", "sjlt")


@dataclass(frozen=True)
class SketchSpec:
    family: str
    m: int
    seed: int
    s: int = 1


@dataclass
class SketchedData:
    """Sketch output SA (m x d) plus the spec that produced it and the
    original row count n (embeddings.py:42-53).  SA is a numpy array when the
    input was numpy, a CUDA tensor when it was a tensor."""

    SA: object
    spec: SketchSpec
    n: int

    @property
    def m(self) -> int:
        return self.SA.shape[0]


def derive_seed(base: int, k: int) -> int:
    """Deterministic child seed for the k-th redraw under a base seed
    (embeddings.py:56-58: SeedSequence((base, k)).generate_state(1, u64)[0]),
    computed natively."""
    base, k = int(base), int(k)
    if base < 0 or k < 0:
        raise ValueError("expected non-negative integer")
    words = _lib.int_words(base) + _lib.int_words(k)
    arr = (C.c_uint32 * len(words))(*words)
    out = (C.c_uint32 * 2)()
    _lib.check(_lib.lib().adask_seedseq_generate(arr, len(words), out, 2), "derive_seed")
    return int(out[0]) | (int(out[1]) << 32)


def _check_m(m: int, n: int) -> None:
    if int(m) != m or m < 1:
        raise SketchTooLarge(f"sketch size must be a positive integer, got {m}")


def padded_rows(n: int) -> int:
    """Rows after zero-padding to the next power of two (embeddings.py:76-78)."""
    n = int(n)
    return 1 << max(0, (n - 1).bit_length()) if n > 1 else 1


def _prep(A, dtype):
    if dv.is_torch(A):
        t = dtype if dtype is not None else (A.dtype if A.dtype in (dv.F64, dv.F32) else dv.F64)
    else:
        t = dv.resolve_dtype(dtype)
    Ad = dv.to_device(A, t)
    if Ad.dim() != 2:
        raise ValueError(f"A must be 2-D, got shape {tuple(Ad.shape)}")
    return Ad


def _result(SA: torch.Tensor, spec: SketchSpec, n: int, like) -> SketchedData:
    return SketchedData(SA=dv.to_host_like(SA, like), spec=spec, n=n)


# ----------------------------------------------------------------- device cores
_GAUSSIAN_RNG = "philox"


def set_gaussian_rng(mode: str) -> str:
    """Select the Gaussian sketch's randomness; returns the previous mode.

    "philox" (default): S is generated on the device from Philox4x32-10
    keyed by (seed, sketch row, global A row) -- the product's definition,
    shard-invariant, never materialized on the host.
    "numpy": S is the reference's own draw, default_rng(seed).standard_normal
    ((m, n)) / sqrt(m) (embeddings.py:71-72), generated on the host and
    applied on the GPU (adask_sketch_dense) -- for running the reference's
    seed-pinned tests unchanged.  Forces the Python driver loop."""
    global _GAUSSIAN_RNG
    if mode not in ("philox", "numpy"):
        raise ValueError(f"unknown Gaussian rng mode {mode!r}")
    prev, _GAUSSIAN_RNG = _GAUSSIAN_RNG, mode
    return prev


def gaussian_rng() -> str:
    return _GAUSSIAN_RNG


def _gaussian_numpy_dev(Ad: torch.Tensor, m: int, seed: int) -> torch.Tensor:
    n, d = Ad.shape
    S = np.random.default_rng(seed).standard_normal((m, n)) / np.sqrt(m)
    Sd = torch.from_numpy(S).to(device=Ad.device, dtype=Ad.dtype)
    SA = torch.empty((m, d), dtype=Ad.dtype, device=Ad.device)
    _lib.check(_lib.lib().adask_sketch_dense(dv.ctx().handle, dv.dtype_code(Ad.dtype), Sd.data_ptr(), m, n,
                                             Sd.stride(0), Ad.data_ptr(), d, Ad.stride(0), SA.data_ptr(),
                                             SA.stride(0), dv.stream()), "sketch_dense")
    return SA


def gaussian_dev(Ad: torch.Tensor, m: int, seed: int, *, row0: int = 0, tf32: bool = False,
                 out: torch.Tensor | None = None, accumulate: bool = False) -> torch.Tensor:
    n, d = Ad.shape
    _check_m(m, n)
    m = int(m)
    if _GAUSSIAN_RNG == "numpy" and row0 == 0 and out is None and not accumulate:
        return _gaussian_numpy_dev(Ad, m, seed)
    SA = out if out is not None else torch.empty((m, d), dtype=Ad.dtype, device=Ad.device)
    flags = (_lib.ACCUMULATE if accumulate else 0) | (_lib.TF32 if tf32 else 0)
    key = int(seed) & 0xFFFFFFFFFFFFFFFF
    _lib.check(
        _lib.lib().adask_sketch_gaussian(dv.ctx().handle, dv.dtype_code(Ad.dtype), Ad.data_ptr(), n, d,
                                         Ad.stride(0), int(row0), m, key, SA.data_ptr(), SA.stride(0),
                                         flags, dv.stream()),
        "sketch_gaussian")
    return SA


def gaussian_rows_dev(Ad: torch.Tensor, m_total: int, k0: int, mk: int, seed: int, *, row0: int = 0,
                      tf32: bool = False) -> torch.Tensor:
    """Rows [k0, k0 + mk) of the m_total-row Gaussian sketch (entries scaled by
    1/sqrt(m_total)): the building block of incremental sketch growth."""
    n, d = Ad.shape
    SA = torch.empty((int(mk), d), dtype=Ad.dtype, device=Ad.device)
    _lib.check(
        _lib.lib().adask_sketch_gaussian_rows(dv.ctx().handle, dv.dtype_code(Ad.dtype), Ad.data_ptr(), n, d,
                                              Ad.stride(0), int(row0), int(m_total), int(k0), int(mk),
                                              int(seed) & 0xFFFFFFFFFFFFFFFF, SA.data_ptr(), SA.stride(0),
                                              _lib.TF32 if tf32 else 0, dv.stream()),
        "sketch_gaussian_rows")
    return SA


def srht_dev(Ad: torch.Tensor, m: int, seed: int, *, out: torch.Tensor | None = None,
             accumulate: bool = False, return_idx: bool = False):
    n, d = Ad.shape
    _check_m(m, n)
    m = int(m)
    n_pad = padded_rows(n)
    if m > n_pad:
        raise SketchTooLarge(f"m = {m} exceeds padded row count {n_pad}")
    g = _lib.pcg64_from_seed(seed)
    SA = out if out is not None else torch.empty((m, d), dtype=Ad.dtype, device=Ad.device)
    idx = (C.c_int64 * m)() if return_idx else None
    _lib.check(
        _lib.lib().adask_sketch_srht(dv.ctx().handle, dv.dtype_code(Ad.dtype), Ad.data_ptr(), n, d,
                                     Ad.stride(0), C.byref(g), m, SA.data_ptr(), SA.stride(0), idx,
                                     _lib.ACCUMULATE if accumulate else 0, dv.stream()),
        "sketch_srht")
    if return_idx:
        return SA, np.frombuffer(idx, dtype=np.int64).copy()
    return SA


def sjlt_rows_host(seed: int, n: int, m: int, s: int) -> tuple[np.ndarray, int]:
    """rows[j*s:(j+1)*s] = choice(m, s, replace=False) per column j
    (embeddings.py:121-123) -- sequential integer bookkeeping, native host
    code.  Returns (rows, number of 32-bit draws consumed)."""
    g = _lib.pcg64_from_seed(seed)
    rows = np.empty(n * s, dtype=np.int64)
    draws = C.c_uint64(0)
    _lib.check(_lib.lib().adask_sjlt_rows(C.byref(g), n, m, s,
                                          rows.ctypes.data_as(C.POINTER(C.c_int64)), C.byref(draws)),
               "sjlt_rows")
    return rows, int(draws.value)


def sjlt_dev(Ad: torch.Tensor, m: int, seed: int, s: int = 1, *, row0: int = 0,
             n_total: int | None = None, out: torch.Tensor | None = None,
             accumulate: bool = False) -> torch.Tensor:
    n, d = Ad.shape
    _check_m(m, n)
    m = int(m)
    if int(s) != s or not (1 <= s <= m):
        raise InvalidSparsity(f"need 1 <= s <= m = {m}, got s = {s}")
    s = int(s)
    n_total = n if n_total is None else int(n_total)
    g = _lib.pcg64_from_seed(seed)
    rows_ptr = None
    sign_first = 0
    if s > 1:
        if row0 != 0 or n_total != n:
            raise NotImplementedError("row-sharded SJLT with s > 1")
        rows, sign_first = sjlt_rows_host(seed, n, m, s)
        rows_ptr = rows.ctypes.data_as(C.POINTER(C.c_int64))
    SA = out if out is not None else torch.empty((m, d), dtype=Ad.dtype, device=Ad.device)
    _lib.check(
        _lib.lib().adask_sketch_sjlt(dv.ctx().handle, dv.dtype_code(Ad.dtype), Ad.data_ptr(), n, d,
                                     Ad.stride(0), int(row0), n_total, m, s, C.byref(g), rows_ptr,
                                     sign_first, SA.data_ptr(), SA.stride(0),
                                     _lib.ACCUMULATE if accumulate else 0, dv.stream()),
        "sketch_sjlt")
    return SA


def gaussian_matrix(m: int, n: int, seed: int, *, col0: int = 0, dtype=torch.float64) -> torch.Tensor:
    """The Gaussian sketch matrix S (m x n) that sketch_gaussian applies
    (device tensor), for oracle comparison."""
    S = torch.empty((int(m), int(n)), dtype=dtype, device=dv.device())
    _lib.check(_lib.lib().adask_philox_gaussian(dv.ctx().handle, dv.dtype_code(dtype), int(m), int(col0),
                                                int(n), int(seed) & 0xFFFFFFFFFFFFFFFF, S.data_ptr(),
                                                S.stride(0), dv.stream()),
               "philox_gaussian")
    return S


# ----------------------------------------------------------------- public API
def sketch_gaussian(A, m: int, seed: int, *, dtype=None, tf32: bool = False) -> SketchedData:
    """Dense Gaussian embedding, entries N(0, 1/m) (embeddings.py:66-73)."""
    Ad = _prep(A, dtype)
    SA = gaussian_dev(Ad, m, seed, tf32=tf32)
    return _result(SA, SketchSpec("gaussian", int(m), seed), Ad.shape[0], A)


def sketch_srht(A, m: int, seed: int, *, dtype=None) -> SketchedData:
    """Subsampled randomized Hadamard transform S = R H E (embeddings.py:81-102)."""
    Ad = _prep(A, dtype)
    SA = srht_dev(Ad, m, seed)
    return _result(SA, SketchSpec("srht", int(m), seed), Ad.shape[0], A)


def sketch_sjlt(A, m: int, seed: int, s: int = 1, *, dtype=None) -> SketchedData:
    """Sparse embedding with s nonzeros +-1/sqrt(s) per column (embeddings.py:105-129)."""
    Ad = _prep(A, dtype)
    n = Ad.shape[0]
    _check_m(m, n)
    if int(s) != s or not (1 <= s <= m):
        raise InvalidSparsity(f"need 1 <= s <= m = {m}, got s = {s}")
    SA = sjlt_dev(Ad, m, seed, s)
    return _result(SA, SketchSpec("sjlt", int(m), seed, s=int(s)), n, A)


def sketch(A, spec: SketchSpec, **kw) -> SketchedData:
    """Dispatch on spec.family (embeddings.py:132-140)."""
    if spec.family == "gaussian":
        return sketch_gaussian(A, spec.m, spec.seed, **kw)
    if spec.family == "srht":
        return sketch_srht(A, spec.m, spec.seed, **kw)
    if spec.family == "sjlt":
        return sketch_sjlt(A, spec.m, spec.seed, s=spec.s, **kw)
    raise ValueError(f"unknown sketch family {spec.family!r}")


def sketch_dev(Ad: torch.Tensor, spec: SketchSpec, *, tf32: bool = False) -> torch.Tensor:
    """Device-resident dispatch used by the solvers (no host round trip)."""
    if spec.family == "gaussian":
        return gaussian_dev(Ad, spec.m, spec.seed, tf32=tf32)
    if spec.family == "srht":
        return srht_dev(Ad, spec.m, spec.seed)
    if spec.family == "sjlt":
        return sjlt_dev(Ad, spec.m, spec.seed, spec.s)
    raise ValueError(f"unknown sketch family {spec.family!r}")


# ------------------------------------------------------ critical sketch sizes
def _check_tail(delta: float, d_e: float) -> None:
    if not (0.0 < delta < 1.0):
        raise InvalidProbability(f"delta must lie in (0, 1), got {delta}")
    if d_e < 1.0:
        raise ValueError(f"d_e must be >= 1, got {d_e}")


def critical_m_srht(d_e: float, n: int, delta: float) -> float:
    """16 log(16 d_e / delta) (sqrt(d_e) + sqrt(8 log(2 n / delta)))^2
    (embeddings.py:150-161; scalar formula)."""
    _check_tail(delta, d_e)
    if n < 1:
        raise ValueError(f"n must be >= 1, got {n}")
    tail = np.sqrt(d_e) + np.sqrt(8.0 * np.log(2.0 * n / delta))
    return float(16.0 * np.log(16.0 * d_e / delta) * tail**2)


def critical_m_gaussian(d_e: float, delta: float) -> float:
    """(sqrt(d_e) + sqrt(8 log(16 / delta)))^2 (embeddings.py:164-169)."""
    _check_tail(delta, d_e)
    return float((np.sqrt(d_e) + np.sqrt(8.0 * np.log(16.0 / delta))) ** 2)
