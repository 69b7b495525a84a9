"""Dev: preconditioner apply time (dense and Woodbury) at d = 1024 fp64."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2104_14101_b200.preconditioner import build_dev
d = 1024
lam = torch.ones(d, dtype=torch.float64, device="cuda")
z = torch.randn(1, d, dtype=torch.float64, device="cuda")
for m in (64, 256, 512, 4096):
    SA = torch.randn(m, d, dtype=torch.float64, device="cuda") / m ** 0.5
    P = build_dev(SA, 1e-2, lam)
    for _ in range(3): P.solve_dev(z)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50): P.solve_dev(z)
    e1.record(); torch.cuda.synchronize()
    print(f"m={m}: apply {e0.elapsed_time(e1)/50*1e3:.1f} us", flush=True)
