"""ADSK1 matrix files (drop-in for adasketch/problem.py:337-365) and a
streaming loader that moves a large file straight into HBM.

Format: magic b"ADSK1", u64 rows, u64 cols (little-endian), then float64
entries in row-major order.  `load_matrix_device` reads the payload in row
chunks into two pinned staging buffers and copies each chunk to the device on
a side stream while the next chunk is read, optionally narrowing to float32
on the device (configs 3-4 keep A in fp32), so a 16-64 GB A never needs a
full host copy.
"""
from __future__ import annotations

import struct

import numpy as np
import torch

from . import device as dv
from .errors import DimensionMismatch, IoFormatError

__all__ = ["save_matrix", "load_matrix", "read_header", "load_matrix_device"]

MAGIC = b"ADSK1"
HEADER = len(MAGIC) + 16


def save_matrix(path, M) -> None:
    """Write M (host array or device tensor) as ADSK1 float64."""
    if isinstance(M, torch.Tensor):
        M = M.detach().to("cpu", torch.float64).numpy()
    M = np.ascontiguousarray(np.asarray(M, dtype=np.float64))
    if M.ndim != 2:
        raise DimensionMismatch(f"expected a matrix, got shape {M.shape}")
    with open(path, "wb") as fh:
        fh.write(MAGIC)
        fh.write(struct.pack("<QQ", M.shape[0], M.shape[1]))
        fh.write(M.astype("<f8").tobytes())


def read_header(path) -> tuple[int, int]:
    with open(path, "rb") as fh:
        magic = fh.read(len(MAGIC))
        if magic != MAGIC:
            raise IoFormatError(f"bad magic {magic!r} in {path}")
        header = fh.read(16)
    if len(header) != 16:
        raise IoFormatError(f"truncated header in {path}")
    return struct.unpack("<QQ", header)


def load_matrix(path) -> np.ndarray:
    """Read a matrix written by save_matrix (host numpy array)."""
    rows, cols = read_header(path)
    with open(path, "rb") as fh:
        fh.seek(HEADER)
        buf = fh.read(rows * cols * 8)
    if len(buf) != rows * cols * 8:
        raise IoFormatError(f"truncated payload in {path}")
    return np.frombuffer(buf, dtype="<f8").reshape(rows, cols).copy()


def load_matrix_device(path, dtype=torch.float64, chunk_bytes: int = 256 << 20) -> torch.Tensor:
    """Stream an ADSK1 file into a device tensor of `dtype` (float64 or
    float32) through two pinned staging buffers: the read of chunk k+1
    overlaps the host-to-device copy (and fp32 narrowing) of chunk k."""
    dt = dv.resolve_dtype(dtype) if not isinstance(dtype, torch.dtype) else dtype
    rows, cols = read_header(path)
    dev = dv.device()
    out = torch.empty((rows, cols), dtype=dt, device=dev)
    if rows == 0 or cols == 0:
        return out
    rchunk = max(1, chunk_bytes // (8 * cols))
    stage = [torch.empty((rchunk, cols), dtype=torch.float64).pin_memory() for _ in range(2)]
    tmp = None if dt == torch.float64 else torch.empty((rchunk, cols), dtype=torch.float64, device=dev)
    stream = torch.cuda.Stream(device=dev)
    done = [torch.cuda.Event(), torch.cuda.Event()]
    with open(path, "rb", buffering=0) as fh:
        fh.seek(HEADER)
        for k, r0 in enumerate(range(0, rows, rchunk)):
            r = min(rchunk, rows - r0)
            b = k & 1
            done[b].synchronize()  # staging buffer b is free again
            view = stage[b][:r].numpy().reshape(-1).view(np.uint8)
            got = fh.readinto(memoryview(view))
            if got != view.nbytes:
                raise IoFormatError(f"truncated payload in {path}")
            with torch.cuda.stream(stream):
                if tmp is None:
                    out[r0:r0 + r].copy_(stage[b][:r], non_blocking=True)
                else:
                    tmp[:r].copy_(stage[b][:r], non_blocking=True)
                    out[r0:r0 + r].copy_(tmp[:r])
                done[b].record(stream)
    stream.synchronize()
    torch.cuda.current_stream(dev).wait_stream(stream)
    return out
