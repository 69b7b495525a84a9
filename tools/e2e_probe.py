"""Dev: where the config-1 end-to-end time goes (pinned host inputs -> x on the host)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden"))
import numpy as np, torch
import paper_2104_14101_b200 as ak
from recipes import baseline_instance
A, b, lam = baseline_instance(1, 65536)
A_pin = torch.from_numpy(A).pin_memory(); b_pin = torch.from_numpy(b).pin_memory(); lam_pin = torch.from_numpy(lam).pin_memory()
x0 = torch.zeros(1024, dtype=torch.float64).pin_memory()
acfg = ak.AdaptiveConfig.for_method("pcg", 0.125, 32, 11, "srht", 1)
def ev():
    e = torch.cuda.Event(enable_timing=True); e.record(); return e
for rep in range(4):
    torch.cuda.synchronize()
    e0 = ev(); t0 = time.perf_counter()
    Ad = A_pin.to("cuda", non_blocking=True)
    e1 = ev()
    p = ak.RegularizedProblem(Ad, b_pin, 1e-2, lam_pin, validate=True)
    e2 = ev(); t2 = time.perf_counter()
    x, tr = ak.adaptive_run(p, x0, acfg, method="pcg")
    e3 = ev()
    xh = x.cpu() if isinstance(x, torch.Tensor) else x
    e4 = ev(); torch.cuda.synchronize(); t4 = time.perf_counter()
    print(f"copy {e0.elapsed_time(e1):.2f} problem {e1.elapsed_time(e2):.2f} solve {e2.elapsed_time(e3):.2f} "
          f"x {e3.elapsed_time(e4):.2f} total {e0.elapsed_time(e4):.2f} ms (host {1e3*(t4-t0):.2f}; problem host {1e3*(t2-t0):.2f})")
