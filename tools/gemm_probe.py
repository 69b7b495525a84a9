"""Gram (SA^T SA) timing for the preconditioner shapes (fp64 / fp32)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_14101_b200.preconditioner import gram_dev  # noqa: E402


def t(fn, k=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k


for dt in (torch.float64, torch.float32):
    for m, d in [(1024, 1024), (2048, 1024), (4096, 1024), (65536, 2048), (2048, 4096)]:
        SA = torch.randn(m, d, dtype=dt, device="cuda")
        ms = t(lambda: gram_dev(SA, 0.0, None))
        fl = 2.0 * m * d * d / 2  # lower triangle
        ref = t(lambda: SA.t() @ SA)
        print(f"{str(dt):14s} m={m:6d} d={d}: gram {ms*1e3:8.1f} us  {fl/ms/1e9:6.1f} TFLOP/s (lower)   "
              f"torch full {ref*1e3:8.1f} us {2.0*m*d*d/ref/1e9:6.1f} TFLOP/s", flush=True)
