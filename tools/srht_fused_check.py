"""Dev: fused SRHT vs the two-launch path on one shape for several Z budgets /
lags; prints mismatching rows and columns."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2104_14101_b200.embeddings import srht_dev

n, d = int(os.environ.get("N", 65536)), int(os.environ.get("D", 72))
A = torch.randn(n, d, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(1))
for m in [int(x) for x in os.environ.get("MS", "64,4096").split(",")]:
    os.environ["ADASK_SRHT_FUSED"] = "0"
    ref = srht_dev(A, m, 3)
    os.environ["ADASK_SRHT_FUSED"] = "1"
    for zmb, lag in [(1000, 1), (1, 1), (1, 3), (4, 1)]:
        os.environ["ADASK_SRHT_FUSED_ZMB"] = str(zmb)
        os.environ["ADASK_SRHT_FUSED_LAG"] = str(lag)
        for rep in range(2):
            got = srht_dev(A, m, 3)
            bad = (got != ref)
            rows = bad.any(1).nonzero().flatten().tolist()
            cols = bad.any(0).nonzero().flatten().tolist()
            print(f"m={m} zmb={zmb} lag={lag} rep={rep}: bad {int(bad.sum())} rows {len(rows)} {rows[:6]} cols {cols[:20]}", flush=True)
