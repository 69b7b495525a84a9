"""Dev probe: fused A^T A x bandwidth for the config shapes."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2104_14101_b200 as ak
shapes = [(4096, 256, torch.float64), (1 << 16, 1024, torch.float64), (1 << 20, 2048, torch.float64),
          (1 << 21, 4096, torch.float32), (1 << 24, 1024, torch.float32)]
sel = os.environ.get("SHAPES")
if sel:
    shapes = [shapes[int(i)] for i in sel.split(",")]
for n, d, dt in shapes:
    A = torch.empty(n, d, dtype=dt, device="cuda").normal_()
    p = ak.RegularizedProblem(A, torch.zeros(d, dtype=torch.float64, device="cuda"), 0.01, validate=False)
    X = torch.randn(1, d, dtype=torch.float64, device="cuda")
    for _ in range(3):
        p.hess_mult_dev(X)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    k = 20
    e0.record()
    for _ in range(k):
        p.hess_mult_dev(X)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / k
    print(f"n={n} d={d} {dt}: {ms*1e3:.1f} us  {A.numel()*A.element_size()/ms/1e6:.0f} GB/s", flush=True)
    del A, p
    torch.cuda.empty_cache()
