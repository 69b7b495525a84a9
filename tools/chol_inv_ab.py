"""Dev probe: fused row-wise L^-1 (ADASK_CHOL_INV=1) vs recursive doubling (0):
preconditioner solves against each other and build timings, interleaved."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2104_14101_b200 as ak
from paper_2104_14101_b200.preconditioner import build_dev


def t(fn, k=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k


g = torch.Generator(device="cuda").manual_seed(0)
for m, d in [(8, 1), (40, 31), (40, 32), (50, 33), (100, 64), (100, 65), (200, 97), (3000, 1030), (1500, 2000),
             (4096, 1024), (8192, 2048), (16384, 4096), (512, 1024), (2048, 4096)]:
    SA = torch.randn(m, d, dtype=torch.float64, device="cuda", generator=g) / m ** 0.5
    lam = torch.rand(d, dtype=torch.float64, device="cuda", generator=g) * 9 + 1
    Z = torch.randn(3, d, dtype=torch.float64, device="cuda", generator=g)
    res = {}
    for inv in ("0", "1"):
        os.environ["ADASK_CHOL_INV"] = inv
        P = build_dev(SA, 0.05, lam)
        res[inv] = P.solve_dev(Z.clone()).clone()
    H = SA.t() @ SA + 0.0025 * torch.diag(lam)
    r = {k: float(torch.linalg.norm(H @ v.t() - Z.t()) / torch.linalg.norm(Z)) for k, v in res.items()}
    diff = float(torch.linalg.norm(res["0"] - res["1"]) / torch.linalg.norm(res["0"]))
    tm = {"0": [], "1": []}
    for _ in range(3):
        for inv in ("0", "1"):
            os.environ["ADASK_CHOL_INV"] = inv
            tm[inv].append(t(lambda: build_dev(SA, 0.05, lam)))
    print(f"m={m} d={d}: resid doubling {r['0']:.2e} fused {r['1']:.2e} reldiff {diff:.2e}  "
          f"build ms doubling {min(tm['0']):.3f} fused {min(tm['1']):.3f}", flush=True)
