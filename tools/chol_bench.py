"""Time the preconditioner's Cholesky + inverse unit (CUDA events on the
launching stream, adask_prof 'chol') for k = 32 .. 4096, fp64 and fp32.

    python tools/chol_bench.py            # current kernel
    ADASK_CHOL_OLD=1 python tools/chol_bench.py   # round-1 cooperative kernel
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_14101_b200 import device as dv  # noqa: E402
from paper_2104_14101_b200.preconditioner import build_dev  # noqa: E402


def main():
    ks = [int(x) for x in sys.argv[1:]] or [32, 64, 128, 256, 512, 1024, 2048, 4096]
    ctx = dv.ctx()
    for dt in (torch.float64, torch.float32):
        for k in ks:
            SA = torch.randn(2 * k, k, dtype=dt, device="cuda") / (2 * k) ** 0.5
            lam = torch.ones(k, dtype=torch.float64, device="cuda")
            for _ in range(3):
                build_dev(SA, 0.1, lam)
            torch.cuda.synchronize()
            ctx.prof_reset()
            ctx.prof_enable(True)
            reps = 10
            for _ in range(reps):
                build_dev(SA, 0.1, lam)
            torch.cuda.synchronize()
            ctx.prof_enable(False)
            pr = ctx.prof_query()
            c, g = pr["chol"], pr["gram"]
            print(json.dumps({"dtype": str(dt).split(".")[-1], "k": k,
                              "chol_us": round(c["ms"] / max(c["count"], 1) * 1e3, 1),
                              "gram_us": round(g["ms"] / max(g["count"], 1) * 1e3, 1),
                              "chol_tflops": round(c["flops"] / max(c["ms"], 1e-9) / 1e9, 2),
                              "old": bool(os.environ.get("ADASK_CHOL_OLD"))}), flush=True)


if __name__ == "__main__":
    main()
