"""Dev probe: phase timing of the cooperative Cholesky (ADASK_CHOL_TRACE=1)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["ADASK_CHOL_TRACE"] = "1"
import numpy as np, torch
import paper_2104_14101_b200 as ak
W = torch.randn(8192, 8192, device="cuda")
def spin(ms=300):
    if os.environ.get("NOSPIN"): return
    t0 = time.perf_counter()
    while (time.perf_counter() - t0) * 1e3 < ms:
        W @ W
    torch.cuda.synchronize()
for k in [int(v) for v in os.environ.get("KS", "1024,2048").split(",")]:
    X = torch.randn(k + 10, k, dtype=torch.float64, device="cuda")
    M = X.t() @ X + torch.eye(k, dtype=torch.float64, device="cuda")
    for _ in range(2):
        spin(100)
        torch.cuda.synchronize(); t0 = time.perf_counter()
        L = ak.cholesky(M)
        torch.cuda.synchronize(); print(k, "wall", (time.perf_counter() - t0) * 1e3, "ms", flush=True)
