"""The C ABI: libadask.so loads on a CPU-only host and exports every
function include/adask.h declares; the ctypes binding covers all of them."""
import re
import subprocess
from pathlib import Path

from paper_2104_14101_b200 import _lib

ROOT = Path(__file__).resolve().parents[1]


def header_functions() -> set[str]:
    text = (ROOT / "include" / "adask.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(r"\b(adask_[a-z0-9_]+)\s*\(", text))


def test_library_loads_and_exports_header():
    lib = _lib.lib()
    assert lib.adask_version() >= 1
    declared = header_functions()
    assert len(declared) > 30
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\b(adask_[a-z0-9_]+)\b", out))
    assert declared <= exported, sorted(declared - exported)


def test_binding_covers_header():
    assert header_functions() <= set(_lib.exported_symbols()) | {"adask_last_error"}
    assert _lib.missing_symbols() == []


def test_status_codes_map_to_reference_exceptions():
    from paper_2104_14101_b200 import errors

    assert _lib._STATUS_EXC[_lib.E_NOT_SPD] is errors.NotPositiveDefinite
    assert _lib._STATUS_EXC[_lib.E_SKETCH_TOO_LARGE] is errors.SketchTooLarge
    assert _lib._STATUS_EXC[_lib.E_SPARSITY] is errors.InvalidSparsity
    assert _lib._STATUS_EXC[_lib.E_BREAKDOWN] is errors.BreakdownDetected
    assert _lib._STATUS_EXC[_lib.E_NEGATIVE] is errors.NegativeValue
    assert _lib._STATUS_EXC[_lib.E_DIM] is errors.DimensionMismatch


def test_no_device_context_without_gpu():
    import ctypes as C

    import torch

    if torch.cuda.is_available():
        return
    h = C.c_void_p()
    assert _lib.lib().adask_ctx_create(0, C.byref(h)) == _lib.E_CUDA
