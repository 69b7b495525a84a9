"""Dev probe: dense Gram as two GEMMs over the lower triangle (ADASK_GRAM_SPLIT=1)
vs the full square (0): preconditioner solves and build timings, interleaved."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

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
for m, d, dt in [(300, 256, torch.float64), (1030, 1000, torch.float64), (1024, 1024, torch.float64),
                 (2048, 1024, torch.float64), (4096, 1024, torch.float64), (4096, 1024, torch.float32),
                 (32768, 1024, torch.float32), (2000, 700, torch.float64)]:
    SA = (torch.randn(m, d, dtype=torch.float64, device="cuda", generator=g) / m ** 0.5).to(dt)
    lam = torch.rand(d, dtype=torch.float64, device="cuda", generator=g) * 9 + 1
    Z = torch.randn(3, d, dtype=torch.float64, device="cuda", generator=g)
    res = {}
    for sp in ("0", "1"):
        os.environ["ADASK_GRAM_SPLIT"] = sp
        res[sp] = build_dev(SA, 0.05, lam).solve_dev(Z.clone()).clone()
    diff = float(torch.linalg.norm(res["0"] - res["1"]) / torch.linalg.norm(res["0"]))
    tm = {"0": [], "1": []}
    for _ in range(3):
        for sp in ("0", "1"):
            os.environ["ADASK_GRAM_SPLIT"] = sp
            tm[sp].append(t(lambda: build_dev(SA, 0.05, lam)))
    print(f"m={m} d={d} {dt}: reldiff {diff:.2e}  build ms full {min(tm['0']):.3f} split {min(tm['1']):.3f}",
          flush=True)
