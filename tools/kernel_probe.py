"""Dev probe: the cfg1 hot kernels in isolation (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2104_14101_b200 as ak
from paper_2104_14101_b200.embeddings import srht_dev, sjlt_dev
n, d = 1 << 16, 1024
A = torch.randn(n, d, dtype=torch.float64, device="cuda")
p = ak.RegularizedProblem(A, torch.zeros(d, dtype=torch.float64, device="cuda"), 0.01, validate=False)
X = torch.randn(1, d, dtype=torch.float64, device="cuda")
for _ in range(2):
    p.hess_mult_dev(X)
for m in (64, 4096):
    for _ in range(2):
        srht_dev(A, m, 12345)
torch.cuda.synchronize()
print("ok")
