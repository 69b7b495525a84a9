"""Dev probe: preconditioner build time per sketch size for the cfg1 shape."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2104_14101_b200.preconditioner import build_dev, gram_dev
d = int(os.environ.get("D", "1024"))
lam = torch.ones(d, dtype=torch.float64, device="cuda")
for m in (32, 64, 128, 256, 512, 1024, 2048, 4096):
    SA = torch.randn(m, d, dtype=torch.float64, device="cuda") / m**0.5
    for _ in range(2):
        P = build_dev(SA, 0.01, lam); del P
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); e0.record()
    for _ in range(5):
        P = build_dev(SA, 0.01, lam); del P
    e1.record(); torch.cuda.synchronize()
    w = (time.perf_counter() - t0) / 5 * 1e3
    # gram only
    src = SA if m >= d else SA.t().contiguous()
    g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g0.record()
    for _ in range(5):
        gram_dev(src, 0.0, None)
    g1.record(); torch.cuda.synchronize()
    print(f"m={m:5d} k={min(m, d):5d}: build {e0.elapsed_time(e1)/5:.3f} ms (wall {w:.3f}), gram {g0.elapsed_time(g1)/5:.3f} ms", flush=True)
