"""Measure the FP64 (DMMA via cuBLAS DGEMM), TF32 and FP32 dense GEMM peaks on
this box, the way MEASURED_PEAKS.json measures bf16: torch.matmul at 8192^3,
best of 10 (burst) and back to back for ~4 s (sustained), CUDA events, with
nvidia-smi clocks sampled during the sustained loop.

    python tools/measure_peaks.py > profiles/r02_peaks.json

These are roofline denominators for the fp64 Gram / Cholesky units and the
TF32 Gaussian sketch and Gram (BASELINE.md section 2 "to be measured").
"""
from __future__ import annotations

import json
import subprocess
import time

import torch


def _clocks_start():
    q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    try:
        return subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits", "-lms", "100"],
                                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
    except OSError:
        return None


def _clocks_stop(p):
    if p is None:
        return {}
    p.terminate()
    out, _ = p.communicate(timeout=10)
    rows = [r.split(", ") for r in out.strip().splitlines() if r.strip()]
    mhz = sorted(float(r[1]) for r in rows if len(r) > 2)
    reasons = set()
    for r in rows:
        for name, v in zip(("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"), r[5:9]):
            if v.strip() == "Active":
                reasons.add(name)
    return {"samples": len(rows), "sm_mhz_median": mhz[len(mhz) // 2] if mhz else None,
            "sm_max_mhz": float(rows[0][2]) if rows else None, "reasons": sorted(reasons)}


def measure(dtype, tf32: bool, n: int = 8192, sustain_s: float = 4.0):
    torch.backends.cuda.matmul.allow_tf32 = tf32
    torch.backends.cudnn.allow_tf32 = tf32
    a = torch.randn(n, n, device="cuda", dtype=dtype)
    b = torch.randn(n, n, device="cuda", dtype=dtype)
    c = torch.empty(n, n, device="cuda", dtype=dtype)
    flops = 2.0 * n ** 3
    for _ in range(3):
        torch.matmul(a, b, out=c)
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b, out=c)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    # sustained: back to back for sustain_s
    reps = max(1, int(sustain_s / best))
    clk = _clocks_start()
    time.sleep(0.3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        torch.matmul(a, b, out=c)
    e1.record()
    torch.cuda.synchronize()
    clocks = _clocks_stop(clk)
    sus = e0.elapsed_time(e1) / 1e3 / reps
    return {"burst_tflops": flops / best / 1e12, "sustained_tflops": flops / sus / 1e12,
            "n": n, "reps": reps, "clocks_sustained": clocks}


def main():
    torch.cuda.init()
    out = {"gpu": torch.cuda.get_device_name(0), "torch": torch.__version__,
           "how": "torch.matmul n^3 (2n^3 flops), best of 10 (burst) and back-to-back ~4 s (sustained), CUDA events"}
    out["fp64"] = measure(torch.float64, False)
    out["tf32"] = measure(torch.float32, True)
    out["fp32_ffma"] = measure(torch.float32, False)
    out["bf16"] = measure(torch.bfloat16, False)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
