"""Dev: one k x k Cholesky (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2104_14101_b200 as ak
k = int(os.environ.get("K", 1024))
X = torch.randn(k + 10, k, dtype=torch.float64, device="cuda")
M = X.t() @ X + torch.eye(k, dtype=torch.float64, device="cuda")
for _ in range(int(os.environ.get("REPS", 1))):
    L = ak.cholesky(M)
torch.cuda.synchronize()
