"""Dev probe: pipelined FWHT passes vs the tile kernels (bitwise) and timings."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2104_14101_b200.embeddings import srht_dev


def run(A, m, seed, pipe):
    os.environ["ADASK_FWHT_PIPE"] = "2" if pipe else "0"
    return srht_dev(A, m, seed)


def t(fn, k=5):
    fn()
    fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k


if os.environ.get("PARITY", "1") == "1":
    g = torch.Generator(device="cuda").manual_seed(0)
    cases = [(4096, 24, 40, torch.float64), (5000, 100, 300, torch.float64), (4097, 33, 4096, torch.float64),
             (1 << 14, 64, 1 << 14, torch.float64), (20000, 17, 999, torch.float32), (1 << 16, 1024, 4096, torch.float64),
             (70000, 40, 4096, torch.float32), ((1 << 21) - 5, 20, 32768, torch.float32),
             ((1 << 21), 24, 64, torch.float32), ((1 << 22), 16, 5000, torch.float32), ((1 << 20) + 1, 8, 100, torch.float64),
             ((1 << 21), 64, 32768, torch.float32), ((1 << 21) - 32, 40, 3000, torch.float64), ((1 << 20) + 64, 36, 1 << 20, torch.float32)]
    for n, d, m, dt in cases:
        A = torch.randn(n, d, dtype=dt, device="cuda", generator=g)
        a = run(A, m, 3, False)
        b = run(A, m, 3, True)
        torch.cuda.synchronize()
        same = torch.equal(a, b)
        diff = (a - b).abs().max().item()
        print(f"n={n} d={d} m={m} {dt}: bitwise {'OK' if same else 'DIFF'} maxdiff {diff:.3e}", flush=True)

if os.environ.get("TIME", "1") == "1":
    n, d = 1 << 16, 1024
    A = torch.randn(n, d, dtype=torch.float64, device="cuda")
    for m in (32, 256, 1024, 4096):
        for pipe in (False, True, 2):
            os.environ["ADASK_FWHT_LDG"] = "0" if pipe == 2 else "1"
            ms = t(lambda: run(A, m, 7, pipe))
            print(f"srht{(" ldg" if pipe is True else " tma") if pipe else ' tile'} n={n} d={d} m={m}: {ms*1e3:.1f} us  "
                  f"{(n+m)*d*8/ms/1e6:.0f} GB/s", flush=True)
    del A
    n, d = 1 << 21, 1024
    A = torch.randn(n, d, dtype=torch.float32, device="cuda")
    for m in (64, 1024, 4096, 32768):
        for pipe in (False, True, 2):
            os.environ["ADASK_FWHT_LDG"] = "0" if pipe == 2 else "1"
            ms = t(lambda: run(A, m, 7, pipe), 3)
            print(f"srht{(" ldg" if pipe is True else " tma") if pipe else ' tile'} fp32 n={n} d={d} m={m}: {ms*1e3:.1f} us  "
                  f"{(n+m)*d*4/ms/1e6:.0f} GB/s", flush=True)

if os.environ.get("B1SWEEP", "0") == "1":
    n, d = 1 << 21, 1024
    A = torch.randn(n, d, dtype=torch.float32, device="cuda")
    for b1 in (10, 11):
        os.environ["ADASK_FWHT_B1"] = str(b1)
        for m in (64, 1024, 4096, 32768):
            ms = t(lambda: run(A, m, 7, True), 3)
            print(f"srht pipe b1={b1} fp32 n={n} d={d} m={m}: {ms*1e3:.1f} us  {(n+m)*d*4/ms/1e6:.0f} GB/s", flush=True)
    del os.environ["ADASK_FWHT_B1"]
