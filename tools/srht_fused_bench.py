"""Time the SRHT sketch on the config-1 shape (2^16 x 1024 fp64; fp32 with
--f32) for the fused kernel's variants against the two-launch path, checking
every result bitwise against the two-launch one.

    python tools/srht_fused_bench.py [--f32] [--n LOG2] [--d D]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import json
VARIANTS = [
    ("two-launch", {"ADASK_SRHT_FUSED": "0"}),
    ("fused sig0", {"ADASK_SRHT_FUSED": "1", "ADASK_SRHT_FUSED_SIG": "0"}),
    ("fused sig1", {"ADASK_SRHT_FUSED": "1", "ADASK_SRHT_FUSED_SIG": "1"}),
    ("fused sig2", {"ADASK_SRHT_FUSED": "1", "ADASK_SRHT_FUSED_SIG": "2"}),
    ("fused sig2 z12 lag3", {"ADASK_SRHT_FUSED": "1", "ADASK_SRHT_FUSED_SIG": "2", "ADASK_SRHT_FUSED_ZMB": "12",
                             "ADASK_SRHT_FUSED_LAG": "3"}),
]


def main():
    global VARIANTS
    if os.environ.get("ONLY"):
        VARIANTS = [v for v in VARIANTS if v[0] in os.environ["ONLY"].split(";")]
    ap = argparse.ArgumentParser()
    ap.add_argument("--f32", action="store_true")
    ap.add_argument("--n", type=int, default=16)
    ap.add_argument("--d", type=int, default=1024)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--ms", default="32,128,512,1024,2048,4096")
    args = ap.parse_args()
    from paper_2104_14101_b200 import device as dv
    from paper_2104_14101_b200.embeddings import srht_dev

    dt = torch.float32 if args.f32 else torch.float64
    g = torch.Generator(device="cuda").manual_seed(0)
    A = torch.randn((1 << args.n, args.d), dtype=dt, device="cuda", generator=g)
    esz = A.element_size()
    ctx = dv.ctx()
    ms = [int(x) for x in args.ms.split(",")]
    ref = {}
    for name, env in VARIANTS:
        for k in ("ADASK_SRHT_FUSED", "ADASK_SRHT_FUSED_ZMB", "ADASK_SRHT_FUSED_LAG", "ADASK_SRHT_FUSED_SIG"):
            os.environ.pop(k, None)
        os.environ.update(env)
        row = []
        for m in ms:
            for _ in range(3):
                SA = srht_dev(A, m, 1234)
            torch.cuda.synchronize()
            ctx.prof_reset()
            ctx.prof_enable(True)
            for _ in range(args.reps):
                SA = srht_dev(A, m, 1234)
            torch.cuda.synchronize()
            ctx.prof_enable(False)
            u = ctx.prof_query()["srht"]
            us = u["ms"] / u["count"] * 1e3
            gbs = (A.shape[0] + m) * A.shape[1] * esz / us / 1e3
            if m not in ref:
                ref[m] = SA.clone()
            ok = torch.equal(SA, ref[m])
            row.append(f"m={m}: {us:7.1f} us {gbs:6.0f} GB/s {'ok' if ok else 'DIFF'}")
        print(f"{name:20s} | " + " | ".join(row), flush=True)


if __name__ == "__main__":
    main()
