"""Benchmark: time-to-solution of the adaptive sketching solver on the B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

A "step" is one complete adaptive solve (Alg. 2 / Alg. 1 of arXiv 2104.14101)
of the configuration's synthetic instance, from A and b resident in HBM to x
at the target relative error: every sketch, Gram, Cholesky and loop pass.
T = T* accepted iterations (adaptive_run has no tolerance stop,
solvers.py:630); T* comes from a tracked run (exact error per record) done
before timing, and the final relative error is re-checked after timing.

Default workload: BASELINE.json configs[1] (adaptive PCG, SRHT, fp64,
n = 2^16, d = 1024).  A (512 MiB) exceeds L2 (126 MB), so no explicit flush.
N > 1: the SRHT does not shard, so each rank solves its own replica
("replicas only", scaling weak); value = device time per solve, max over ranks.

--impl reference times the reference algorithm on the host CPU (the oracle
port under oracle/, numpy/OpenBLAS on all host cores) on the same instance.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "time-to-solution (rel err 1e-10) & S·A sketch GB/s, % roofline, 1/2/4/8 GPU"


def _peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return {"hbm_gbs": float(pk["hbm_gbs"]), "bf16_tflops": float(pk["bf16_tflops"]),
                "source": "MEASURED_PEAKS.json (measured)"}
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "source": "B200_PROFILING.md fallback"}


class ClockSampler:
    """Samples SM clock and throttle reasons with NVML during the timed region."""

    REASONS = {
        0x0000000000000001: "gpu_idle", 0x0000000000000002: "applications_clocks_setting",
        0x0000000000000004: "sw_power_cap", 0x0000000000000008: "hw_slowdown",
        0x0000000000000010: "sync_boost", 0x0000000000000020: "sw_thermal_slowdown",
        0x0000000000000040: "hw_thermal_slowdown", 0x0000000000000080: "hw_power_brake_slowdown",
    }

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                mhz = self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)
                util = self.nv.nvmlDeviceGetUtilizationRates(self.h).gpu
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                if util > 0:
                    self.samples.append(mhz)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.05)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self) -> dict:
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _cfg(idx: int):
    from paper_2104_14101_b200.configs import CONFIGS

    return CONFIGS[idx]


# --------------------------------------------------------------- reference arm
def run_reference(args) -> None:
    ws, rank, _ = _dist()
    if rank != 0:
        return
    from oracle import adasketch_oracle as O
    from paper_2104_14101_b200.configs import make_instance

    cfg = _cfg(args.config)
    A, b, lam = make_instance(cfg)
    A = A.astype(np.float64)
    p = O.Problem.make(A, b, cfg.nu, lam)
    x0 = np.zeros(cfg.d)

    def solve(pp):
        return O.adaptive_run(pp, x0 if pp is p else np.zeros(pp.d), cfg.method, args.rho, cfg.m_init,
                              cfg.t_star, cfg.family, args.seed)

    # warm-up steps: the same solve on a 1/64 row sample (numpy has no JIT to warm)
    small = O.Problem.make(A[: max(cfg.d, cfg.n // 64)], b, cfg.nu, lam)
    for _ in range(args.warmup):
        solve(small)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        solve(p)
        times.append(time.perf_counter() - t0)
    v = float(np.mean(times))
    cores = os.cpu_count()
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": v * 1e3, "higher_is_better": False,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg.name(), "T": cfg.t_star, "rho": args.rho, "seed": args.seed},
        "cpu_baseline": {"value": v, "unit": "s", "cores": cores, "kind": "port",
                         "sample": f"{args.steps} full solves of {cfg.name()} (warm-up on a 1/64 row sample)"},
        "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- our arm
def run_ours(args) -> None:
    import torch

    import paper_2104_14101_b200 as ak
    from paper_2104_14101_b200 import device as dv
    from paper_2104_14101_b200.configs import make_instance

    ws, rank, local = _dist()
    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist_mod

        dist_mod.init_process_group("nccl", device_id=torch.device("cuda", local))
        dist = dist_mod
    cfg = _cfg(args.config)
    dev = torch.device("cuda", local)

    A, b, lam = make_instance(cfg)
    p = ak.RegularizedProblem(A, b, cfg.nu, lam, dtype=cfg.dtype)
    x0 = torch.zeros(cfg.d, dtype=torch.float64, device=dev)

    # ---- T* from a tracked run (exact error per record), untimed
    sol = ak.direct_solve(p)
    cfg_tr = ak.AdaptiveConfig.for_method(cfg.method, args.rho, cfg.m_init, 3 * cfg.t_star + 10,
                                          cfg.family, args.seed)
    _, tr = ak.adaptive_run(p, x0, cfg_tr, method=cfg.method, sol=sol)
    d0 = tr.records[0].delta_exact
    t_star = next((r.t for r in tr.records if r.event != "resketch" and r.delta_exact <= cfg.target * d0),
                  None)
    if t_star is None:
        t_star = cfg.t_star
    acfg = ak.AdaptiveConfig.for_method(cfg.method, args.rho, cfg.m_init, t_star, cfg.family, args.seed)

    def solve():
        return ak.adaptive_run(p, x0, acfg, method=cfg.method)

    for _ in range(args.warmup):
        solve()
    ctx = dv.ctx()
    ctx.prof_reset()
    ctx.prof_enable(True)
    launches0 = ctx.launches()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record()
        for _ in range(args.steps):
            x, trace = solve()
        ev1.record()
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    launches = ctx.launches() - launches0
    ctx.prof_enable(False)
    prof = ctx.prof_query()
    ms = ev0.elapsed_time(ev1) / args.steps
    if dist:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    rel_err = ak.exact_error(p, x, sol) / d0

    # ---- end to end through the public API from pinned host memory
    A_pin = torch.from_numpy(np.ascontiguousarray(A)).pin_memory()
    b_pin = torch.from_numpy(b).pin_memory()
    lam_pin = torch.from_numpy(lam).pin_memory()
    x0_pin = torch.zeros(cfg.d, dtype=torch.float64).pin_memory()

    def e2e_step():
        pe = ak.RegularizedProblem(A_pin, b_pin, cfg.nu, lam_pin, dtype=cfg.dtype)
        xe, _ = ak.adaptive_run(pe, x0_pin, acfg, method=cfg.method)
        return xe.cpu()

    e2e_step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        xh = e2e_step()
    e1.record()
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / args.steps
    if dist:
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    h2d = A_pin.numel() * A_pin.element_size() + b_pin.numel() * 8 + lam_pin.numel() * 8 + x0_pin.numel() * 8
    d2h = xh.numel() * 8

    # ---- roofline of the dominant unit
    pk = _peaks()
    dom = max(prof, key=lambda k: prof[k]["ms"])
    u = prof[dom]
    per_launch_ms = u["ms"] / max(u["count"], 1)
    bytes_per = u["bytes"] / max(u["count"], 1)
    achieved = bytes_per / (per_launch_ms * 1e-3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(f"cfg{cfg.index}", {}).get(dom)
        except Exception:
            traffic = None
    units = {k: {"count": v["count"], "ms_total": round(v["ms"], 4),
                 "gbs": round(v["bytes"] / max(v["ms"], 1e-9) / 1e6, 1)} for k, v in prof.items() if v["count"]}
    sketch_unit = {"srht": "srht", "sjlt": "sjlt", "gaussian": "gaussian", "srht-block": "srht"}[cfg.family]
    su = prof[sketch_unit]
    sketch_gbs = su["bytes"] / max(su["ms"], 1e-9) / 1e6 if su["count"] else None

    # ---- CPU baseline (rank 0, N = 1): the oracle port, one full solve
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        from oracle import adasketch_oracle as O

        po = O.Problem.make(A.astype(np.float64), b, cfg.nu, lam)
        t0 = time.perf_counter()
        O.adaptive_run(po, np.zeros(cfg.d), cfg.method, args.rho, cfg.m_init, t_star, cfg.family, args.seed)
        cpu_s = time.perf_counter() - t0
        cpu = {"value": cpu_s, "unit": "s", "cores": os.cpu_count(), "kind": "port",
               "sample": f"1 full solve of {cfg.name()} (T={t_star}), numpy/OpenBLAS on all host threads"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": ms / 1e3, "unit": "s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64" if cfg.dtype == "float64" else "f32", "data": "synthetic",
            "config": {"workload": cfg.name(), "T": t_star, "rho": args.rho, "seed": args.seed,
                       "parallelism": f"replicas{ws}" if ws > 1 else "single",
                       "l2": "A (%.0f MiB) exceeds the 126 MB L2; no flush" % (A.nbytes / 2**20)},
            "rel_err_final": rel_err,
            "schedule": trace.schedule(),
            "solves_per_s_total": ws * 1e3 / ms,
            "sketch_gbs": sketch_gbs,
            "units": units,
            "roofline": {"bound": "hbm", "unit_name": dom, "achieved": achieved, "peak": pk["hbm_gbs"],
                         "unit": "GB/s", "frac": achieved / pk["hbm_gbs"], "traffic": traffic,
                         "per_launch_ms": per_launch_ms, "alg_bytes_per_launch": bytes_per,
                         "peak_source": pk["source"]},
            "clocks": clk.summary(),
            "e2e": {"value": e2e_ms / 1e3, "unit": "s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h)},
            "gpu_launches": int(launches),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--rho", type=float, default=0.125)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
