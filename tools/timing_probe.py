"""Dev probe: solve time with / without live profiling and the clock sampler."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2104_14101_b200 as ak
from paper_2104_14101_b200 import device as dv
from paper_2104_14101_b200.configs import CONFIGS, make_instance
import bench

cfg = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 1]
A, b, lam = make_instance(cfg)
p = ak.RegularizedProblem(A, b, cfg.nu, lam, dtype=cfg.dtype)
x0 = torch.zeros(cfg.d, dtype=torch.float64, device="cuda")
acfg = ak.AdaptiveConfig.for_method(cfg.method, 0.125, cfg.m_init, cfg.t_star, cfg.family, 1)
def solve(): return ak.adaptive_run(p, x0, acfg, method=cfg.method)
for _ in range(3): solve()
def timed(label, k=5):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(k): solve()
    torch.cuda.synchronize(); print(label, (time.perf_counter() - t0) / k * 1e3, "ms", flush=True)
timed("plain")
ctx = dv.ctx(); ctx.prof_reset(); ctx.prof_enable(True)
timed("prof")
ctx.prof_enable(False)
with bench.ClockSampler(0): timed("sampler")
timed("plain2")
# per-phase host timings
import paper_2104_14101_b200.solvers as S
from paper_2104_14101_b200.embeddings import SketchSpec, sketch_dev, derive_seed
from paper_2104_14101_b200.preconditioner import build_dev
for m in (64, 1024, 4096):
    spec = SketchSpec(cfg.family, m, derive_seed(1, 3))
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(5): SA = sketch_dev(p.A, spec)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    for _ in range(5): P = build_dev(SA, p.nu, p.lam_dev); del P
    torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"m={m} sketch {(t1-t0)/5*1e3:.3f} ms build {(t2-t1)/5*1e3:.3f} ms", flush=True)
P = build_dev(SA, p.nu, p.lam_dev)
st = S._PcgState(p, P, x0[None, :].clone()) if cfg.method == "pcg" else S._IhsState(p, P, x0[None, :].clone(), 0.125)
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(20): st.propose()
torch.cuda.synchronize(); print("propose", (time.perf_counter() - t0) / 20 * 1e3, "ms")
Xt = torch.randn(1, cfg.d, dtype=torch.float64, device="cuda")
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(20): p.hess_mult_dev(Xt)
torch.cuda.synchronize(); print("hess_mult", (time.perf_counter() - t0) / 20 * 1e3, "ms", A.nbytes / ((time.perf_counter() - t0) / 20) / 1e9, "GB/s")
