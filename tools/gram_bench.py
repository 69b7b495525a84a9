"""Time the DMMA Gram (gram.cu) against cuBLAS (torch) on the preconditioner
shapes of configs 1-4: dense SA^T SA (d x d) and Woodbury (SA/lam) SA^T.

    python tools/gram_bench.py
"""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2104_14101_b200.preconditioner import gram_dev, woodbury_gram_dev  # noqa: E402


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    rows = []
    cases = [("dense", torch.float64, m, 1024) for m in (1024, 2048, 4096)]
    cases += [("dense", torch.float64, m, 2048) for m in (2048, 8192, 32768, 65536)]
    cases += [("dense", torch.float32, m, 1024) for m in (1024, 8192, 32768)]
    cases += [("woodbury", torch.float64, m, 1024) for m in (64, 256, 512)]
    cases += [("woodbury", torch.float64, m, 2048) for m in (512, 1024)]
    cases += [("woodbury", torch.float32, m, 4096) for m in (256, 1024, 2048)]
    for kind, dt, m, d in cases:
        SA = torch.randn(m, d, dtype=dt, device="cuda") / m**0.5
        lam = torch.rand(d, dtype=torch.float64, device="cuda") * 9 + 1
        if kind == "dense":
            ours = timeit(lambda: gram_dev(SA, 1e-4, lam))
            flops = m * d * (d + 1)
            lib = timeit(lambda: SA.t() @ SA)
        else:
            ours = timeit(lambda: woodbury_gram_dev(SA, 1e-4, lam))
            flops = m * (m + 1) * d
            T = SA / lam.to(dt)
            lib = timeit(lambda: T @ SA.t())
        rows.append({"kind": kind, "dtype": str(dt).split(".")[-1], "m": m, "d": d, "ours_ms": round(ours, 4),
                     "ours_tflops": round(flops / ours / 1e9, 2), "cublas_full_ms": round(lib, 4)})
        print(json.dumps(rows[-1]), flush=True)


if __name__ == "__main__":
    main()
