"""ctypes binding of libadask.so (the C ABI declared in include/adask.h).

The library is required: importing the compute modules without it raises
immediately — there is no CPU fallback for any compute path.  Host-only
entry points (seeding, PCG64 bookkeeping) work without a GPU.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

from . import errors

LIB_PATH = Path(os.environ.get("ADASK_LIB") or Path(__file__).resolve().parent / "libadask.so")

ADASK_OK = 0
E_DIM, E_NOT_SPD, E_NOT_POW2, E_SKETCH_TOO_LARGE, E_SPARSITY = 1, 2, 3, 4, 5
E_NEGATIVE, E_BREAKDOWN, E_ARG, E_CUDA, E_NOMEM = 6, 7, 8, 9, 10
F64, F32 = 0, 1
ACCUMULATE, PARTIAL, TF32 = 0x1, 0x2, 0x4
INCREMENTAL = 0x8

_STATUS_EXC = {
    E_DIM: errors.DimensionMismatch,
    E_NOT_SPD: errors.NotPositiveDefinite,
    E_NOT_POW2: errors.NotPowerOfTwo,
    E_SKETCH_TOO_LARGE: errors.SketchTooLarge,
    E_SPARSITY: errors.InvalidSparsity,
    E_NEGATIVE: errors.NegativeValue,
    E_BREAKDOWN: errors.BreakdownDetected,
    E_ARG: ValueError,
    E_CUDA: RuntimeError,
    E_NOMEM: MemoryError,
}


class PCG64State(C.Structure):
    _fields_ = [
        ("state_hi", C.c_uint64),
        ("state_lo", C.c_uint64),
        ("inc_hi", C.c_uint64),
        ("inc_lo", C.c_uint64),
        ("has_uint32", C.c_int32),
        ("uinteger", C.c_uint32),
    ]


ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int64, C.c_int, C.c_void_p, C.c_void_p)


class Problem(C.Structure):
    _fields_ = [
        ("dtype", C.c_int),
        ("A", C.c_void_p),
        ("n", C.c_int64),
        ("d", C.c_int64),
        ("lda", C.c_int64),
        ("c", C.c_int64),
        ("nu2", C.c_double),
        ("lam", C.c_void_p),
        ("B", C.c_void_p),
        ("allreduce", ALLREDUCE_FN),
        ("allreduce_user", C.c_void_p),
        ("use_ctx_comm", C.c_int32),
        ("comm_rank", C.c_int32),
        ("comm_world", C.c_int32),
    ]


class AdaptiveCfg(C.Structure):
    _fields_ = [
        ("method", C.c_int),
        ("family", C.c_int),
        ("rho", C.c_double),
        ("m_init", C.c_int64),
        ("T", C.c_int64),
        ("seed", C.c_uint64),
        ("s", C.c_int64),
        ("alpha", C.c_double),
        ("phi_rho", C.c_double),
        ("c_alpha_rho", C.c_double),
        ("block", C.c_int64),
        ("row0", C.c_int64),
        ("n_total", C.c_int64),
        ("flags", C.c_uint32),
    ]


class TraceRec(C.Structure):
    _fields_ = [
        ("t", C.c_int64),
        ("m", C.c_int64),
        ("k", C.c_int64),
        ("delta_tilde", C.c_double),
        ("delta_exact", C.c_double),
        ("wall_seconds", C.c_double),
        ("event", C.c_int32),
        ("has_exact", C.c_int32),
    ]


vp, i64, u64, u32, i32, dbl = C.c_void_p, C.c_int64, C.c_uint64, C.c_uint32, C.c_int32, C.c_double
P = C.POINTER
_PROTOS = {
    "adask_last_error": (C.c_char_p, []),
    "adask_version": (C.c_int, []),
    "adask_device_count": (C.c_int, []),
    "adask_seedseq_generate": (C.c_int, [P(u32), i64, P(u32), i64]),
    "adask_derive_seed": (u64, [u64, u64]),
    "adask_pcg64_seed": (C.c_int, [P(u32), i64, P(PCG64State)]),
    "adask_pcg64_advance": (C.c_int, [P(PCG64State), u64]),
    "adask_pcg64_skip_u32": (C.c_int, [P(PCG64State), u64]),
    "adask_pcg64_next_u64": (u64, [P(PCG64State)]),
    "adask_pcg64_next_u32": (u32, [P(PCG64State)]),
    "adask_pcg64_bounded_u32": (u32, [P(PCG64State), u32]),
    "adask_choice_noreplace": (C.c_int, [P(PCG64State), i64, i64, P(i64)]),
    "adask_pcg64_integers_host": (C.c_int, [P(PCG64State), u32, i64, P(i64)]),
    "adask_sjlt_rows": (C.c_int, [P(PCG64State), i64, i64, i64, P(i64), P(u64)]),
    "adask_ctx_create": (C.c_int, [C.c_int, P(vp)]),
    "adask_ctx_destroy": (C.c_int, [vp]),
    "adask_ctx_launches": (i64, [vp]),
    "adask_prof_enable": (C.c_int, [vp, C.c_int]),
    "adask_prof_reset": (C.c_int, [vp]),
    "adask_prof_query": (C.c_int, [vp, C.c_int, P(i64), P(dbl), P(dbl), P(dbl)]),
    "adask_pcg64_integers": (C.c_int, [vp, P(PCG64State), u64, i64, u32, vp, P(u64), vp]),
    "adask_philox_gaussian": (C.c_int, [vp, C.c_int, i64, i64, i64, u64, vp, i64, vp]),
    "adask_philox_gaussian_host": (C.c_int, [i64, i64, i64, u64, vp, i64]),
    "adask_sketch_gaussian": (C.c_int, [vp, C.c_int, vp, i64, i64, i64, i64, i64, u64, vp, i64, u32, vp]),
    "adask_sketch_gaussian_rows": (C.c_int, [vp, C.c_int, vp, i64, i64, i64, i64, i64, i64, i64, u64, vp, i64, C.c_uint32, vp]),
    "adask_sketch_dense": (C.c_int, [vp, C.c_int, vp, i64, i64, i64, vp, i64, i64, vp, i64, vp]),
    "adask_sketch_srht": (C.c_int, [vp, C.c_int, vp, i64, i64, i64, P(PCG64State), i64, vp, i64, P(i64), u32, vp]),
    "adask_sketch_sjlt": (C.c_int, [vp, C.c_int, vp, i64, i64, i64, i64, i64, i64, i64, P(PCG64State),
                                    P(i64), u64, vp, i64, u32, vp]),
    "adask_fwht": (C.c_int, [vp, C.c_int, vp, i64, i64, i64, C.c_int, vp]),
    "adask_check_problem": (C.c_int, [vp, C.c_int, vp, i64, i64, i64, vp, i64, vp, i64, P(C.c_int), vp]),
    "adask_hess_mult": (C.c_int, [vp, C.c_int, vp, i64, i64, i64, vp, i64, i64, dbl, vp, vp, i64, vp, i64, u32, vp]),
    "adask_hess_mult_pair": (C.c_int, [vp, C.c_int, vp, i64, i64, i64, vp, vp, dbl, vp, vp, vp, vp]),
    "adask_vec_hess_finish": (C.c_int, [vp, vp, i64, i64, i64, vp, dbl, vp, vp, vp, vp]),
    "adask_precond_build": (C.c_int, [vp, C.c_int, vp, i64, i64, i64, dbl, vp, P(vp), P(i64), vp]),
    "adask_precond_destroy": (C.c_int, [vp]),
    "adask_precond_path": (C.c_int, [vp]),
    "adask_precond_factor": (C.c_int, [vp, P(vp), P(i64), P(C.c_int)]),
    "adask_precond_apply": (C.c_int, [vp, vp, vp, i64, i64, vp, i64, vp]),
    "adask_precond_copy_factor": (C.c_int, [vp, vp, C.c_int, vp, i64, vp]),
    "adask_gram": (C.c_int, [vp, C.c_int, vp, i64, i64, i64, dbl, vp, vp, i64, vp]),
    "adask_gram_ex": (C.c_int, [vp, C.c_int, vp, i64, i64, i64, dbl, vp, C.c_int, vp, i64, vp]),
    "adask_gram_woodbury": (C.c_int, [vp, C.c_int, vp, i64, i64, i64, dbl, vp, vp, i64, vp]),
    "adask_cholesky": (C.c_int, [vp, C.c_int, vp, i64, i64, vp, vp, P(i64), vp]),
    "adask_tri_solve": (C.c_int, [vp, C.c_int, vp, i64, i64, C.c_int, vp, i64, i64, vp, i64, vp]),
    "adask_pcg_restart": (C.c_int, [vp, P(Problem), vp, vp, vp, vp, vp, vp, P(dbl), vp]),
    "adask_pcg_propose": (C.c_int, [vp, P(Problem), vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, P(dbl), vp]),
    "adask_pcg_commit": (C.c_int, [vp, i64, i64, vp, vp, vp, vp, vp]),
    "adask_ihs_restart": (C.c_int, [vp, P(Problem), vp, vp, vp, vp, P(dbl), vp]),
    "adask_ihs_propose": (C.c_int, [vp, P(Problem), vp, vp, vp, dbl, vp, dbl, vp, vp, vp, P(dbl), vp]),
    "adask_dot": (C.c_int, [vp, vp, vp, i64, i64, i64, P(dbl), vp]),
    "adask_nccl_available": (C.c_int, []),
    "adask_nccl_unique_id": (C.c_int, [vp]),
    "adask_comm_init_nccl": (C.c_int, [vp, vp, C.c_int, C.c_int]),
    "adask_set_comm": (C.c_int, [vp, vp, C.c_int, C.c_int]),
    "adask_comm_destroy": (C.c_int, [vp]),
    "adask_comm_allreduce": (C.c_int, [vp, vp, i64, C.c_int, vp]),
    "adask_adaptive_run": (C.c_int, [vp, P(Problem), P(AdaptiveCfg), vp, vp, vp, P(TraceRec), i64, P(i64), vp]),
}

_lib = None
_missing: list[str] = []
_lock = threading.Lock()


def lib():
    """Load libadask.so (once).  Raises if it has not been built."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not LIB_PATH.exists():
                    raise ImportError(
                        f"{LIB_PATH} is missing: build it with "
                        "`python -m paper_2104_14101_b200.buildlib` (there is no CPU fallback)"
                    )
                h = C.CDLL(str(LIB_PATH))
                for name, (res, args) in _PROTOS.items():
                    fn = getattr(h, name, None)
                    if fn is None:
                        _missing.append(name)
                        continue
                    fn.restype = res
                    fn.argtypes = args
                _lib = _Serialized(h)
    return _lib


_call_lock = threading.RLock()


class _Serialized:
    """libadask with every entry point serialized by one re-entrant lock.
    The device context (workspaces, pinned scalars, the order of its stream)
    is shared by all host threads of the process -- the reference CLI's
    `compare`, for one, runs its solver jobs on a thread pool -- while the C
    ABI allows one caller per context at a time (include/adask.h)."""

    def __init__(self, h):
        self._h = h

    def __getattr__(self, name):
        fn = getattr(self._h, name)
        if not name.startswith("adask_"):
            return fn

        def call(*args, _fn=fn):
            with _call_lock:
                return _fn(*args)

        setattr(self, name, call)
        return call


def exported_symbols() -> list[str]:
    return list(_PROTOS)


def missing_symbols() -> list[str]:
    lib()
    return list(_missing)


def check(status: int, what: str = "") -> None:
    if status == ADASK_OK:
        return
    msg = lib().adask_last_error().decode(errors="replace")
    exc = _STATUS_EXC.get(status, RuntimeError)
    raise exc(f"{what}: {msg}" if what else msg)


class Context:
    """One libadask device context per CUDA device (workspaces, pinned scalars)."""

    _by_device: dict[int, "Context"] = {}

    def __init__(self, device: int):
        self.device = device
        h = C.c_void_p()
        check(lib().adask_ctx_create(device, C.byref(h)), "ctx_create")
        self.handle = h

    @classmethod
    def get(cls, device: int | None = None) -> "Context":
        import torch

        if device is None:
            device = torch.cuda.current_device()
        ctx = cls._by_device.get(device)
        if ctx is None:
            ctx = cls._by_device[device] = Context(device)
        return ctx

    def launches(self) -> int:
        return int(lib().adask_ctx_launches(self.handle))

    PROF_KINDS = ("hess_mult", "srht", "sjlt", "gaussian", "build", "apply", "gram", "chol")

    def prof_enable(self, on: bool = True) -> None:
        check(lib().adask_prof_enable(self.handle, 1 if on else 0))

    def prof_reset(self) -> None:
        check(lib().adask_prof_reset(self.handle))

    def prof_query(self) -> dict:
        out = {}
        for k, name in enumerate(self.PROF_KINDS):
            cnt, ms, by, fl = C.c_int64(), C.c_double(), C.c_double(), C.c_double()
            check(lib().adask_prof_query(self.handle, k, C.byref(cnt), C.byref(ms), C.byref(by), C.byref(fl)))
            out[name] = {"count": cnt.value, "ms": ms.value, "bytes": by.value, "flops": fl.value}
        return out


def int_words(v: int) -> list[int]:
    """numpy _int_to_uint32_array: little-endian 32-bit words (>= 1 word)."""
    if v < 0:
        raise ValueError("expected non-negative integer")
    w = []
    while True:
        w.append(v & 0xFFFFFFFF)
        v >>= 32
        if v == 0:
            break
    return w


def pcg64_from_seed(seed) -> PCG64State:
    """State of np.random.default_rng(seed).bit_generator, computed natively."""
    if isinstance(seed, (list, tuple)):
        words = [w for s in seed for w in int_words(int(s))]
    else:
        words = int_words(int(seed))
    arr = (C.c_uint32 * len(words))(*words)
    g = PCG64State()
    check(lib().adask_pcg64_seed(arr, len(words), C.byref(g)), "pcg64_seed")
    return g


def stream_ptr(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def env_flag(name: str, default: str = "") -> str:
    return os.environ.get(name, default)
