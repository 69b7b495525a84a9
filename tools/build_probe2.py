"""Dev: preconditioner build time by m at d = 1024 (fp64), Cholesky alone, Gram alone."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2104_14101_b200 as ak
from paper_2104_14101_b200.preconditioner import build_dev
def t(fn, k=10):
    fn(); fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k * 1e3
d = int(os.environ.get("D", 1024))
lam = torch.ones(d, dtype=torch.float64, device="cuda")
for m in (32, 64, 128, 256, 512, 1024, 2048, 4096):
    SA = torch.randn(m, d, dtype=torch.float64, device="cuda") / m ** 0.5
    us = t(lambda: build_dev(SA, 1e-2, lam))
    k = min(m, d)
    G = SA.t() @ SA if m >= d else SA @ SA.t()
    G += torch.eye(k, dtype=torch.float64, device="cuda")
    uc = t(lambda: ak.cholesky(G))
    ug = t(lambda: torch.mm(SA.t(), SA) if m >= d else torch.mm(SA, SA.t()))
    print(f"m={m:5d} build {us:8.1f} us | cholesky(k={k}) {uc:8.1f} us | torch gram {ug:7.1f} us", flush=True)
