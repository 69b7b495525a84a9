"""Dev: run-to-run determinism soak.  Every adaptive solve (method x sketch
family, two sizes) is repeated and must return the same schedule and the same
bits of x each time: split-K sums, the dataflow Cholesky, the fused SRHT and the
streamed SJLT all fix their summation order, so a difference means a race."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_14101_b200 as ak  # noqa: E402
from oracle import adasketch_oracle as O  # noqa: E402

t0 = time.time()
budget = float(os.environ.get("SECONDS", 120))
cases = [("pcg", "srht"), ("pcg", "sjlt"), ("ihs", "gaussian"), ("ihs", "srht"), ("pcg", "gaussian")]
sizes = [(4096, 64, 0.95), (1 << 15, 512, 0.99)]
total = 0
for n, d, dec in sizes:
    j = np.arange(1, d + 1, dtype=float)
    A, b, lam = O.make_config_problem(n, d, dec**j, 1e-2, False, data_seed=3)
    p = ak.RegularizedProblem(A, b, 1e-2, lam)
    for method, fam in cases:
        cfg = ak.AdaptiveConfig.for_method(method, 0.125, 8, 10, fam, 1)
        ref = None
        reps = 0
        t1 = time.time()
        while time.time() - t1 < budget / (len(cases) * len(sizes)):
            x, tr = ak.adaptive_run(p, np.zeros(d), cfg, method=method)
            key = ([(r.t, r.m, r.k, r.event) for r in tr.records], np.asarray(x).tobytes())
            if ref is None:
                ref = key
            assert key[0] == ref[0], (n, d, method, fam, "schedule changed between runs")
            assert key[1] == ref[1], (n, d, method, fam, "x changed between runs")
            reps += 1
        total += reps
        print(f"n={n} d={d} {method}/{fam}: {reps} identical solves, schedule {tr.schedule()}", flush=True)
print(f"soak ok: {total} solves, {time.time() - t0:.0f} s")
