"""Time the SRHT sketch (prof unit 'srht') on config-1 shapes for a list of m,
and check the result bitwise against the one-group schedule
(ADASK_SRHT_ZBUDGET_MB=1000000 in a subprocess gives the single-group result).

    python tools/srht_bench.py [budget_mb ...]
"""
import json
import os
import subprocess
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def run(ms, reps=10):
    from paper_2104_14101_b200 import device as dv
    from paper_2104_14101_b200.embeddings import srht_dev

    g = torch.Generator(device="cuda").manual_seed(0)
    A = torch.randn((1 << 16, 1024), dtype=torch.float64, device="cuda", generator=g)
    ctx = dv.ctx()
    out = {}
    for m in ms:
        for _ in range(3):
            SA = srht_dev(A, m, 1234)
        torch.cuda.synchronize()
        ctx.prof_reset()
        ctx.prof_enable(True)
        for _ in range(reps):
            SA = srht_dev(A, m, 1234)
        torch.cuda.synchronize()
        ctx.prof_enable(False)
        u = ctx.prof_query()["srht"]
        out[m] = {"us": u["ms"] / u["count"] * 1e3, "gbs": u["bytes"] / u["ms"] / 1e6,
                  "sum": float(SA.sum().item()), "crc": int(torch.sum(SA.view(torch.int64) % 1000003).item())}
    return out


if __name__ == "__main__":
    ms = [32, 512, 1024, 2048, 4096]
    if len(sys.argv) > 1 and sys.argv[1] == "--child":
        print(json.dumps(run(ms)))
        sys.exit(0)
    budgets = sys.argv[1:] or ["1000000", "32", "48", "64", "96"]
    res = {}
    for b in budgets:
        env = dict(os.environ, ADASK_SRHT_ZBUDGET_MB=b)
        o = subprocess.run([sys.executable, __file__, "--child"], env=env, capture_output=True, text=True)
        res[b] = json.loads(o.stdout.strip().splitlines()[-1]) if o.returncode == 0 else o.stderr[-500:]
    ref = res[budgets[0]]
    for b, r in res.items():
        if isinstance(r, str):
            print(b, "ERR", r)
            continue
        print(b, {m: (round(v["us"], 1), round(v["gbs"]), v["crc"] == ref[str(m)]["crc"]) for m, v in
                  ((int(k), v) for k, v in r.items())})
