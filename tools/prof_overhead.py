"""Dev: config-1 solve time with and without the per-unit event profiling."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2104_14101_b200 as ak
from paper_2104_14101_b200 import configs, device as dv
cfg = configs.CONFIGS[1]
A, b, lam = configs.make_instance(cfg)
p = ak.RegularizedProblem(A, b, cfg.nu, lam)
x0 = torch.zeros(cfg.d, dtype=torch.float64, device="cuda")
acfg = ak.AdaptiveConfig.for_method(cfg.method, 0.125, cfg.m_init, 11, cfg.family, 1)
for _ in range(3):
    ak.adaptive_run(p, x0, acfg, method=cfg.method)
for prof in (False, True, False, True):
    dv.ctx().prof_enable(prof)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(10):
        ak.adaptive_run(p, x0, acfg, method=cfg.method)
    e1.record(); torch.cuda.synchronize()
    print(f"prof={prof}: {e0.elapsed_time(e1)/10:.3f} ms/solve (host {1e3*(time.perf_counter()-t0)/10:.3f} ms)", flush=True)
