"""Dev: host-side cost of one SRHT sketch call (GPU kept busy so the host time is all host work)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2104_14101_b200.embeddings import srht_dev
A = torch.randn(1 << 16, 1024, dtype=torch.float64, device="cuda")
W = torch.randn(8192, 8192, device="cuda")
for m in (32, 256, 1024, 4096):
    srht_dev(A, m, 7); torch.cuda.synchronize()
    ts = []
    for rep in range(5):
        for _ in range(20): W @ W          # ~ms of queued GPU work
        t0 = time.perf_counter()
        srht_dev(A, m, 7 + rep)
        ts.append((time.perf_counter() - t0) * 1e6)
        torch.cuda.synchronize()
    print(f"m={m}: host time per srht_dev call {min(ts):.0f} us (median {sorted(ts)[2]:.0f})", flush=True)
A4 = torch.randn(1 << 21, 1024, dtype=torch.float32, device="cuda")
for m in (64, 4096, 32768):
    ts = []
    for rep in range(5):
        for _ in range(40): W @ W
        t0 = time.perf_counter()
        srht_dev(A4, m, 7 + rep)
        ts.append((time.perf_counter() - t0) * 1e6)
        torch.cuda.synchronize()
    print(f"2^21 block m={m}: host time {min(ts):.0f} us (median {sorted(ts)[2]:.0f})", flush=True)
