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
--config 0..4 selects the other BASELINE configurations; 2-4 are generated on
the device (16-64 GB of A), config 3 runs the TF32 tensor-core sketch.
N > 1: configs 0-1 run one replica per rank (the global SRHT does not shard;
scaling weak); configs 2-4 row-shard A over the ranks with NCCL all-reduces
(scaling strong).  value = device time per solve, max over ranks.

--impl reference times the reference algorithm on the host CPU (the oracle
port under oracle/, numpy/OpenBLAS on all host cores): the same instance for
configs 0-1; a leading row sample for configs 2-4, scaled to full n.
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
        out = {"hbm_gbs": float(pk["hbm_gbs"]), "bf16_tflops": float(pk["bf16_tflops"]),
               "bf16_tflops_sustained": float(pk.get("bf16_tflops_sustained", pk["bf16_tflops"])),
               "source": "MEASURED_PEAKS.json (measured)"}
    except Exception:
        out = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
               "source": "B200_PROFILING.md fallback"}
    # FP64 (DMMA) and TF32 dense peaks: cuBLAS DGEMM / TF32 GEMM 8192^3 measured
    # on this pool's B200s by tools/measure_peaks.py (profiles/r02_peaks.json)
    try:
        with open(os.path.join(ROOT, "profiles", "r02_peaks.json")) as f:
            pk = json.load(f)
        out.update(fp64_tflops=float(pk["fp64"]["burst_tflops"]), tf32_tflops=float(pk["tf32"]["burst_tflops"]),
                   tf32_tflops_sustained=float(pk["tf32"]["sustained_tflops"]),
                   fp_source="profiles/r02_peaks.json (cuBLAS 8192^3 measured, tools/measure_peaks.py)")
    except Exception:
        out.update(fp64_tflops=37.0, tf32_tflops=out["bf16_tflops"] / 2, tf32_tflops_sustained=
                   out["bf16_tflops_sustained"] / 2, fp_source="nominal FP64 / half of bf16 for TF32")
    return out


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
        self._stop, self._on, self.t = threading.Event(), threading.Event(), None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _sample(self):
        try:
            mhz = self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)
            r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            self.samples.append(mhz)
            for bit, name in self.REASONS.items():
                if r & bit and name != "gpu_idle":
                    self.reasons.add(name)
        except Exception:
            pass

    def _run(self):
        # the thread (and NVML) are up before the timed region opens; samples
        # are kept only while it is open (the GPU is busy throughout it)
        while not self._stop.is_set():
            if self._on.is_set():
                self._sample()
            time.sleep(0.001)

    def start(self):
        if self.nv and self.t is None:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __enter__(self):
        self.start()
        self._on.set()
        return self

    def __exit__(self, *a):
        self._on.clear()
        self._stop.set()
        if self.nv:
            self.t.join()
            if not self.samples:  # a timed region shorter than the sampling period
                self._sample()

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


# ------------------------------------------------------------ instance / sample
SAMPLE_ROWS = {0: None, 1: None, 2: 1 << 14, 3: 1 << 15, 4: 1 << 18}


def _host_sample(cfg, A_dev=None, p_dev=None):
    """Host (numpy fp64) instance for the CPU arms.  Configs 0-1: the full
    instance (numpy recipe).  Configs 2-4 (16-64 GB): the first SAMPLE_ROWS
    rows of the device instance with b recomputed for that sample; the CPU
    time is reported per full-size solve by scaling with n / n_sample (every
    per-iteration cost of the algorithm is linear in n at fixed d and T)."""
    from paper_2104_14101_b200.configs import make_instance

    ns = SAMPLE_ROWS[cfg.index]
    if ns is None:
        A, b, lam = make_instance(cfg)
        return A.astype(np.float64), b, lam, 1.0, f"full instance n={cfg.n}"
    import torch

    if cfg.index == 2 and A_dev is not None and p_dev is not None:
        # config 2 (16 GiB fp64): the full instance the GPU solved, copied to
        # the host -- one full-size oracle solve, no extrapolation
        As = A_dev.cpu().numpy()
        return (As, p_dev.Bt[0].cpu().numpy(), p_dev.lam_dev.cpu().numpy(), 1.0,
                f"full instance n={cfg.n} (the device instance, copied to the host)")

    from paper_2104_14101_b200.configs import make_instance_device

    if A_dev is None:
        A_dev, _, lam_d = make_instance_device(cfg, n_local=ns)
    else:
        lam_d = None
    As = A_dev[:ns].double().cpu().numpy()
    rng = np.random.default_rng(7)
    x0 = rng.standard_normal(cfg.d)
    b = As.T @ (As @ x0 + 0.01 * rng.standard_normal(ns))
    lam = (np.random.default_rng(123).uniform(1.0, 10.0, cfg.d) if cfg.lam_uniform else np.ones(cfg.d))
    del lam_d
    torch.cuda.empty_cache()
    return As, b, lam, cfg.n / ns, f"first {ns} of {cfg.n} rows (time x {cfg.n // ns})"


def _oracle_solve(O, cfg, A, b, lam, T, rho, seed):
    p = O.Problem.make(A, b, cfg.nu, lam)
    fam = "srht-block" if cfg.family == "srht-block" else cfg.family
    kw = {}
    if fam == "srht-block":
        blk = min(cfg.block, A.shape[0])
        kw["sketcher"] = lambda A_, m, sd: O.block_srht(A_, m, sd, blk)
        kw["cap"] = min(A.shape[0], O.padded_rows(blk))
        fam = "srht"
    return O.adaptive_run(p, np.zeros(cfg.d), cfg.method, rho, cfg.m_init, T, fam, seed, **kw)


# --------------------------------------------------------------- reference arm
L2_BYTES = 126e6


def _config_dict(cfg, t_star, args, ws, a_mib):
    """The `config` object of the JSON line: identical for both arms (the
    driver compares them key by key)."""
    return {"workload": cfg.name(), "T": t_star, "rho": args.rho, "seed": args.seed,
            "parallelism": (f"replicas{ws}" if cfg.index < 2 else f"rowshard{ws}") if ws > 1 else "single",
            "l2": ("A (%.0f MiB per GPU) exceeds the 126 MB L2; no flush" % a_mib) if a_mib * 2**20 > L2_BYTES
            else ("A (%.0f MiB per GPU) fits in the 126 MB L2: 256 MiB written between timed steps, "
                  "outside the per-step event windows" % a_mib)}


def run_reference(args) -> None:
    ws, rank, _ = _dist()
    if rank != 0:
        return
    from oracle import adasketch_oracle as O

    cfg = _cfg(args.config)
    A, b, lam, scale, sample = _host_sample(cfg)

    def solve():
        return _oracle_solve(O, cfg, A, b, lam, cfg.t_star, args.rho, args.seed)

    # warm-up steps: the same solve on a 1/64 row sample (numpy has no JIT to warm)
    small = max(4 * cfg.d, A.shape[0] // 64)
    for _ in range(args.warmup):
        _oracle_solve(O, cfg, A[:small], A[:small].T @ A[:small].sum(axis=1), lam, 2, args.rho, args.seed)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        solve()
        times.append((time.perf_counter() - t0) * scale)
    v = float(np.mean(times))
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": v * 1e3, "higher_is_better": False,
        "scaling": "weak" if cfg.index < 2 else "strong", "vs_baseline": None,
        "dtype": "f64" if cfg.dtype == "float64" else "f32", "data": "synthetic",
        "config": _config_dict(cfg, cfg.t_star, args, ws,
                               cfg.n * cfg.d * (8 if cfg.dtype == "float64" else 4) / 2**20
                               / (ws if cfg.index >= 2 else 1)),
        "cpu_baseline": {"value": v, "unit": "s", "cores": os.cpu_count(), "kind": "port",
                         "sample": f"{args.steps} solves on {sample}; numpy/OpenBLAS, all host threads"},
        "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- our arm
def _build_problem(cfg, ws, rank, dist, dev):
    """Device problem for this rank.  Configs 0-1: host numpy instance,
    replicated (the global SRHT does not shard).  Configs 2-4: generated on
    the device, rows sharded over the ranks (b all-reduced)."""
    import torch

    import paper_2104_14101_b200 as ak
    from paper_2104_14101_b200.configs import make_instance, make_instance_device

    if cfg.index < 2:
        A, b, lam = make_instance(cfg)
        return ak.RegularizedProblem(A, b, cfg.nu, lam, dtype=cfg.dtype), (A, b, lam), None
    from paper_2104_14101_b200 import parallel as par

    plan = par.shard_rows(cfg.n, ws, rank, align=cfg.block or 1)
    A_d, b_d, lam_d = make_instance_device(cfg, n_local=plan.n_local, row0=plan.row0)
    if ws > 1:
        dist.all_reduce(b_d)
        comm = par.Comm()  # NCCL: libadask's own communicator, exchanges issued by the native driver
        p = par.ShardedProblem(A_d, b_d, cfg.nu, lam_d, plan=plan, comm=comm, validate=False)
    else:
        p = ak.RegularizedProblem(A_d, b_d, cfg.nu, lam_d, validate=False)
    torch.cuda.synchronize()
    return p, None, plan


def _log(msg: str) -> None:
    if int(os.environ.get("RANK", "0")) == 0:
        sys.stderr.write(f"[bench {time.strftime('%H:%M:%S')}] {msg}\n")
        sys.stderr.flush()


def _exact_solution(ak, p, cfg, sharded, dist):
    """x* for the tracked run (untimed): problem.direct_solve -- fp64 Gram
    accumulated over row blocks, fp64 Cholesky, two triangular solves -- with
    the partial Grams all-reduced when A is row-sharded."""
    if not sharded:
        return ak.direct_solve(p)
    from paper_2104_14101_b200.problem import gram_fp64

    H = gram_fp64(p.A_dev)
    dist.all_reduce(H)
    H.diagonal().add_(p.nu**2 * p.lam_dev)
    L = ak.cholesky(H)
    X = ak.tri_solve(L, ak.tri_solve(L, p.Bt.t().contiguous()), transposed=True)
    return ak.ExactSolution(x_star=X)


def run_ours(args) -> None:
    import torch

    import paper_2104_14101_b200 as ak
    from paper_2104_14101_b200 import device as dv

    ws, rank, local = _dist()
    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist_mod

        dist_mod.init_process_group("nccl", device_id=torch.device("cuda", local))
        dist = dist_mod
    cfg = _cfg(args.config)
    dev = torch.device("cuda", local)
    _log(f"building {cfg.name()}")
    p, host_inst, plan = _build_problem(cfg, ws, rank, dist, dev)
    sharded = plan is not None and ws > 1
    x0 = torch.zeros(cfg.d, dtype=torch.float64, device=dev)
    tf32 = cfg.dtype == "float32" and cfg.family == "gaussian" and not args.no_tf32
    # row-sharded problems run the native driver too: every exchange (pair
    # all-reduce per proposal, reduce-scatter + partial Gram + d x d all-reduce
    # per resketch) is issued by libadask on its NCCL communicator
    kw = {"tf32": tf32, "block": cfg.block or (1 << 21)}

    def acfg_for(T):
        return ak.AdaptiveConfig.for_method(cfg.method, args.rho, cfg.m_init, T, cfg.family, args.seed)

    # ---- T* from a tracked run (exact error per record), untimed.  x* is the
    # direct solve: an fp64 Cholesky of H = A^T A + nu^2 Lambda (for fp32 data
    # the Gram is accumulated in fp64 from fp64 row blocks -- measurement
    # support only).  The tracked run is kept short: near the data's rounding
    # floor the adaptive rule rejects every step and doubles m up to n.
    _log(f"instance ready ({p.n} x {p.d} {cfg.dtype}); exact solution")
    sol = _exact_solution(ak, p, cfg, sharded, dist)
    t_star = None
    T_track = cfg.t_star + 2
    for _ in range(4):
        _, tr = ak.adaptive_run(p, x0, acfg_for(T_track), method=cfg.method, sol=sol, **kw)
        d0 = tr.records[0].delta_exact
        t_star = next((r.t for r in tr.records if r.event != "resketch" and r.delta_exact <= cfg.target * d0),
                      None)
        if t_star is not None:
            break
        T_track = int(T_track * 1.5) + 1
    if t_star is None:
        t_star = T_track
    _log(f"T* = {t_star} (tracked run {tr.schedule()})")
    acfg = acfg_for(t_star)

    def solve():
        return ak.adaptive_run(p, x0, acfg, method=cfg.method, **kw)

    clk = ClockSampler(local).start()  # NVML and its thread up before the timed region
    _log("warm-up")
    for _ in range(args.warmup):
        solve()
    _log("timed solves")
    ctx = dv.ctx()
    ctx.prof_enable(False)
    launches0 = ctx.launches()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    # an instance that fits in L2 (config 0) gets the cache flushed between
    # timed steps; each step is then timed by its own event pair
    small = p.A_dev.numel() * p.A_dev.element_size() <= L2_BYTES
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if small else None
    evb = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    with clk:
        ev0.record()
        evs[0].record()
        for k in range(args.steps):
            if small:
                flush.zero_()
                evb[k].record()
            x, trace = solve()
            evs[k + 1].record()
        ev1.record()
        torch.cuda.synchronize()
    if small:
        step_ms = [round(evb[k].elapsed_time(evs[k + 1]), 3) for k in range(args.steps)]
    else:
        step_ms = [round(evs[k].elapsed_time(evs[k + 1]), 3) for k in range(args.steps)]
    _log(f"step ms {step_ms}; torch allocated {torch.cuda.memory_allocated() >> 20} MiB, "
         f"reserved {torch.cuda.memory_reserved() >> 20} MiB")
    if dist:
        dist.barrier()
    launches = ctx.launches() - launches0
    # per-unit kernel times (roofline, `units`): a second pass of the same K
    # steps with a CUDA event pair around every unit on the launching stream
    # (the events cost ~5% of a config-1 step, so `value` is taken without them)
    _log("profiled pass (per-unit CUDA events)")
    ctx.prof_reset()
    ctx.prof_enable(True)
    torch.cuda.synchronize()
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p0.record()
    for k in range(args.steps):
        solve()
    p1.record()
    torch.cuda.synchronize()
    ctx.prof_enable(False)
    prof = ctx.prof_query()
    prof_ms_per_step = p0.elapsed_time(p1) / args.steps
    ms = ev0.elapsed_time(ev1) / args.steps
    if small:
        ms = sum(evb[k].elapsed_time(evs[k + 1]) for k in range(args.steps)) / args.steps
    if dist:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    rel_err = ak.exact_error(p, x, sol) / d0

    # ---- incremental sketch growth (north_star; not reference semantics): the
    # same solve with the sketch grown instead of redrawn when m doubles
    incr = None
    if cfg.family != "sjlt" and not args.no_incremental and not sharded:
        _log("incremental growth variant")
        kw_i = dict(kw, incremental=True)
        T_i = cfg.t_star + 2
        t_i = None
        for _ in range(4):
            _, tr_i = ak.adaptive_run(p, x0, acfg_for(T_i), method=cfg.method, sol=sol, **kw_i)
            d0_i = tr_i.records[0].delta_exact
            t_i = next((r.t for r in tr_i.records if r.event != "resketch" and r.delta_exact <= cfg.target * d0_i),
                       None)
            if t_i is not None:
                break
            T_i = int(T_i * 1.5) + 1
        t_i = t_i if t_i is not None else T_i
        acfg_i = acfg_for(t_i)
        for _ in range(args.warmup):
            ak.adaptive_run(p, x0, acfg_i, method=cfg.method, **kw_i)
        torch.cuda.synchronize()
        i0, i1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        i0.record()
        for _ in range(args.steps):
            x_i, tr_i = ak.adaptive_run(p, x0, acfg_i, method=cfg.method, **kw_i)
        i1.record()
        torch.cuda.synchronize()
        incr = {"ms_per_step": i0.elapsed_time(i1) / args.steps, "T": t_i, "schedule": tr_i.schedule(),
                "rel_err_final": ak.exact_error(p, x_i, sol) / d0_i,
                "note": "sketch grown instead of redrawn at each resketch (SRHT: transform kept, rows added; "
                        "Gaussian: rows kept and rescaled, new rows added); not the reference's draw sequence"}

    # ---- end to end through the public API from pinned host memory
    _log("e2e")
    e2e = _e2e(args, cfg, p, host_inst, acfg, kw, ws, dist, dev)

    # ---- roofline of the dominant unit: the unit with the most device time
    # among ALL units (build is split into its Gram and Cholesky+inverse parts)
    pk = _peaks()
    units_all = ("hess_mult", "srht", "sjlt", "gaussian", "gram", "chol", "apply")
    dom = max(units_all, key=lambda k: prof[k]["ms"])
    rf = {}
    for name in units_all:
        u = prof[name]
        if not u["count"]:
            continue
        per_launch_ms = u["ms"] / u["count"]
        peak_src = pk["source"]
        if name == "gaussian" and tf32:
            # TF32 tcgen05 GEMM inside a long solve under the power cap: sustained TF32
            work_per, unit, bound = u["flops"] / u["count"], "TFLOP/s", "tensor"
            peak, peak_src = pk["tf32_tflops_sustained"], pk["fp_source"] + " (TF32 sustained)"
        elif name in ("gram", "chol") or name == "gaussian":
            # DMMA Gram, Cholesky + triangular inverse, fp64/fp32 Gaussian: FP64 pipe
            work_per, unit, bound = u["flops"] / u["count"], "TFLOP/s", ("tensor" if name == "gram" else "fp64")
            peak, peak_src = pk["fp64_tflops"], pk["fp_source"] + " (FP64 DGEMM)"
        else:
            work_per, unit, bound = u["bytes"] / u["count"], "GB/s", "hbm"
            peak = pk["hbm_gbs"]
        scale = 1e12 if unit == "TFLOP/s" else 1e9
        achieved = work_per / (per_launch_ms * 1e-3) / scale
        rf[name] = {"bound": bound, "unit_name": name, "achieved": achieved, "peak": peak, "unit": unit,
                    "frac": achieved / peak, "per_launch_ms": per_launch_ms, "alg_work_per_launch": work_per,
                    "peak_source": peak_src, "share_of_units": u["ms"] / max(sum(
                        prof[k]["ms"] for k in units_all), 1e-9)}
    roof = dict(rf[dom])
    bound, unit, peak, achieved, per_launch_ms, work_per = (roof["bound"], roof["unit"], roof["peak"],
                                                           roof["achieved"], roof["per_launch_ms"],
                                                           roof["alg_work_per_launch"])
    tensor = bound == "tensor"
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(f"cfg{cfg.index}", {}).get(dom)
        except Exception:
            traffic = None
    units = {k: {"count": v["count"], "ms_total": round(v["ms"], 4),
                 "gbs": round(v["bytes"] / max(v["ms"], 1e-9) / 1e6, 1),
                 "tflops": round(v["flops"] / max(v["ms"], 1e-9) / 1e9, 2)} for k, v in prof.items() if v["count"]}
    for k, r in rf.items():
        units[k].update(bound=r["bound"], frac=round(r["frac"], 4), peak=r["peak"], peak_unit=r["unit"])
    if "build" in units:
        units["build"]["note"] = "gram + chol (+ small copies); see those units"
    sketch_unit = {"srht": "srht", "sjlt": "sjlt", "gaussian": "gaussian", "srht-block": "srht"}[cfg.family]
    su = prof[sketch_unit]
    sketch_gbs = su["bytes"] / max(su["ms"], 1e-9) / 1e6 if su["count"] else None

    # ---- CPU baseline (rank 0, N = 1): the oracle port on a bounded sample
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        from oracle import adasketch_oracle as O

        _log("cpu baseline")
        A_s, b_s, lam_s, scale, sample = _host_sample(cfg, None if cfg.index < 2 else p.A_dev, p)
        t0 = time.perf_counter()
        _oracle_solve(O, cfg, A_s, b_s, lam_s, t_star, args.rho, args.seed)
        cpu_s = (time.perf_counter() - t0) * scale
        cpu = {"value": cpu_s, "unit": "s", "cores": os.cpu_count(), "kind": "port",
               "sample": f"1 solve (T={t_star}) on {sample}; numpy/OpenBLAS on all host threads"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": ms / 1e3, "unit": "s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False,
            "scaling": "weak" if cfg.index < 2 else "strong",
            "vs_baseline": None, "dtype": "f64" if cfg.dtype == "float64" else ("tf32" if tf32 else "f32"),
            "data": "synthetic (seeded; BASELINE.json recipe, device Philox for configs 2-4)",
            "config": _config_dict(cfg, t_star, args, ws, p.A_dev.numel() * p.A_dev.element_size() / 2**20),
            "rel_err_final": rel_err,
            "step_ms": step_ms,
            "schedule": trace.schedule(),
            "solves_per_s_total": (ws if cfg.index < 2 else 1) * 1e3 / ms,
            "sketch_gbs": sketch_gbs,
            "units": units,
            "units_pass": {"ms_per_step": prof_ms_per_step,
                           "note": "units and roofline from a second pass of the same steps with per-unit CUDA "
                                   "events on the launching stream; value/ms_per_step from the pass without them"},
            "roofline": dict(roof, traffic=traffic),
            "clocks": clk.summary(),
            "e2e": e2e,
            "incremental": incr,
            "gpu_launches": int(launches),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def _e2e(args, cfg, p, host_inst, acfg, kw, ws, dist, dev):
    """Same solve through the public API with A, b, lam, x0 in pinned host
    memory; the H2D copies and the D2H read of x are inside the timed region."""
    import torch

    import paper_2104_14101_b200 as ak

    if host_inst is not None:
        A, b, lam = host_inst
        A_pin = torch.from_numpy(np.ascontiguousarray(A)).pin_memory()
        b_pin = torch.from_numpy(b).pin_memory()
        lam_pin = torch.from_numpy(lam).pin_memory()
    else:
        try:
            import psutil

            need = p.A_dev.numel() * p.A_dev.element_size()
            if psutil.virtual_memory().available < 1.5 * need:
                return {"value": None, "unit": "s", "skipped": f"host RAM < 1.5 x {need >> 30} GiB for pinned A"}
        except Exception:
            pass
        A_pin = torch.empty(p.A_dev.shape, dtype=p.A_dev.dtype, pin_memory=True)
        A_pin.copy_(p.A_dev)
        b_pin = p.Bt[0].cpu().pin_memory()
        lam_pin = p.lam_dev.cpu().pin_memory()
    x0_pin = torch.zeros(cfg.d, dtype=torch.float64).pin_memory()
    kw = {k: v for k, v in kw.items() if k != "sketcher"}

    def step():
        if ws > 1 and cfg.index >= 2:
            from paper_2104_14101_b200 import parallel as par

            pe = par.ShardedProblem(A_pin, b_pin, cfg.nu, lam_pin, plan=p.plan, comm=p.comm, validate=False)
            kk = dict(kw, sketcher=par.sharded_sketcher(p.comm, block=cfg.block or (1 << 21), tf32=kw["tf32"]))
        else:
            pe = ak.RegularizedProblem(A_pin, b_pin, cfg.nu, lam_pin, dtype=cfg.dtype, validate=cfg.index < 2)
            kk = kw
        xe, _ = ak.adaptive_run(pe, x0_pin, acfg, method=cfg.method, **kk)
        return xe.cpu() if isinstance(xe, torch.Tensor) else xe

    step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        xh = step()
    e1.record()
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / args.steps
    if dist:
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    h2d = A_pin.numel() * A_pin.element_size() + b_pin.numel() * 8 + lam_pin.numel() * 8 + x0_pin.numel() * 8
    d2h = int(np.asarray(xh).size) * 8
    return {"value": e2e_ms / 1e3, "unit": "s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)}


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=None,
                    help="BASELINE config (default: 1 on one GPU -- the global SRHT does not shard; "
                         "2, the row-sharded 1/2/4/8-GPU workload, for --gpus > 1)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--rho", type=float, default=0.125)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-tf32", action="store_true", help="fp32 Gaussian sketch on the FP32 pipe instead of TF32")
    ap.add_argument("--no-incremental", action="store_true", help="skip the incremental-growth variant")
    args = ap.parse_args()
    if args.config is None:
        args.config = 1 if args.gpus <= 1 else 2
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch this command under torchrun
        import socket
        import subprocess

        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
        s.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
        if "--config" not in sys.argv:
            cmd += ["--config", str(args.config)]
        sys.exit(subprocess.call(cmd))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
