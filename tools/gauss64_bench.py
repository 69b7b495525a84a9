"""fp64 Gaussian sketch: DMMA path (default) against the FP64-pipe GEMM
(ADASK_GAUSS_DMMA=0, read once per process -> run twice).  Prints TFLOP/s."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_14101_b200.embeddings import gaussian_dev  # noqa: E402

shapes = [(4096, 256, 256), (65536, 1024, 256), (65536, 1024, 1024), (1 << 18, 512, 2048)]
if os.environ.get("SHAPES"):
    shapes = [shapes[int(i)] for i in os.environ["SHAPES"].split(",")]
for n, d, m in shapes:
    A = torch.randn((n, d), dtype=torch.float64, device="cuda")
    for _ in range(2):
        gaussian_dev(A, m, 1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    reps = 5
    for _ in range(reps):
        gaussian_dev(A, m, 1)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"dmma={os.environ.get('ADASK_GAUSS_DMMA', '1')} n={n} d={d} m={m}: {ms:.3f} ms "
          f"{2.0 * m * n * d / ms / 1e9:.2f} TFLOP/s", flush=True)

if os.environ.get("GAUSS_PROFILE"):
    from torch.profiler import ProfilerActivity, profile
    n, d, m = shapes[-1]
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        gaussian_dev(A, m, 1)
        torch.cuda.synchronize()
    for e in prof.key_averages():
        print(f"  {e.key[:70]:70s} x{e.count:4d} {e.device_time_total / 1e3:9.3f} ms")
