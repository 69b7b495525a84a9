"""Dev: one SRHT sketch (for ncu).  env N, D, M, DT (f32/f64), PIPE."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2104_14101_b200.embeddings import srht_dev
n = int(os.environ.get("N", 1 << 21)); d = int(os.environ.get("D", 1024)); m = int(os.environ.get("M", 64))
dt = torch.float32 if os.environ.get("DT", "f32") == "f32" else torch.float64
A = torch.randn(n, d, dtype=dt, device="cuda")
for _ in range(int(os.environ.get("REPS", 2))):
    srht_dev(A, m, 7)
torch.cuda.synchronize()
print("done")
