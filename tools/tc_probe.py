"""Throughput probe of the TF32 tcgen05 Gaussian sketch at config-3 shapes."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_14101_b200.embeddings import gaussian_dev  # noqa: E402
from bench import ClockSampler  # noqa: E402

n = int(os.environ.get("N", 1 << 21))
d = int(os.environ.get("D", 4096))
A = torch.randn(n, d, device="cuda", dtype=torch.float32)
for m in [int(x) for x in os.environ.get("MS", "128,256,512,1024,2048").split(",")]:
    out = torch.empty(m, d, device="cuda")
    gaussian_dev(A, m, 7, tf32=True, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = int(os.environ.get("REPS", 3))
    with ClockSampler(0) as clk:
        e0.record()
        for _ in range(reps):
            gaussian_dev(A, m, 7, tf32=True, out=out)
        e1.record()
        torch.cuda.synchronize()
    cs = clk.summary()
    ms = e0.elapsed_time(e1) / reps
    tf = 2.0 * m * n * d / (ms * 1e-3) / 1e12
    gbs = n * d * 4 / (ms * 1e-3) / 1e9
    print(f"m={m:5d} n={n} d={d}: {ms:8.3f} ms  {tf:7.1f} TFLOP/s  A-stream {gbs:7.1f} GB/s  sm {cs['sm_mhz']} MHz {cs['reasons']}", flush=True)
