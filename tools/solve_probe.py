"""Per-solve wall times and per-record driver timestamps for a BASELINE config
(device instance), with and without unit profiling."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_14101_b200 as ak  # noqa: E402
from paper_2104_14101_b200 import device as dv  # noqa: E402
from paper_2104_14101_b200.configs import CONFIGS, make_instance_device  # noqa: E402

cfg = CONFIGS[int(os.environ.get("CFG", 2))]
T = int(os.environ.get("T", cfg.t_star))
A, b, lam = make_instance_device(cfg)
p = ak.RegularizedProblem(A, b, cfg.nu, lam, validate=False)
x0 = torch.zeros(cfg.d, dtype=torch.float64, device="cuda")
acfg = ak.AdaptiveConfig.for_method(cfg.method, 0.125, cfg.m_init, T, cfg.family, 1)
kw = {"tf32": cfg.dtype == "float32" and cfg.family == "gaussian", "block": cfg.block or (1 << 21)}
for prof in [False] * int(os.environ.get("ROUNDS", 1)) + [True, False]:
    dv.ctx().prof_enable(prof)
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        x, tr = ak.adaptive_run(p, x0, acfg, method=cfg.method, **kw)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(f"prof={prof} rep={rep}: {dt*1e3:8.1f} ms  schedule={tr.schedule()}", flush=True)
        if dt > 0.3:  # slow solve: where did the time go
            last = 0.0
            for r in tr.records:
                if r.wall_seconds - last > 0.02:
                    print(f"    slow step before record t={r.t} m={r.m} ev={r.event}: +{(r.wall_seconds-last)*1e3:.1f} ms")
                last = r.wall_seconds
    if prof:
        q = dv.ctx().prof_query()
        print({k: (v['count'], round(v['ms'], 1)) for k, v in q.items() if v['count']})
        dv.ctx().prof_reset()
last = 0.0
for r in tr.records:
    print(f"  t={r.t:3d} m={r.m:6d} K={r.k if hasattr(r,'k') else ''} ev={r.event:9s} wall={r.wall_seconds*1e3:9.2f} ms (+{(r.wall_seconds-last)*1e3:8.2f})")
    last = r.wall_seconds
