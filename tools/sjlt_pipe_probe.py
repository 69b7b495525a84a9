"""Dev probe: bulk-copy streamed SJLT accumulation vs k_bucket_accumulate (bitwise) and timings."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2104_14101_b200.embeddings import sjlt_dev
def run(A, m, seed, pipe, s=1):
    os.environ["ADASK_SJLT_PIPE"] = "1" if pipe else "0"
    return sjlt_dev(A, m, seed, s) if s != 1 else sjlt_dev(A, m, seed)
def t(fn, k=3):
    fn(); fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k
g = torch.Generator(device="cuda").manual_seed(0)
for n, d, m, dt, s in [(1000, 16, 7, torch.float64, 1), (5000, 34, 300, torch.float64, 1), (70000, 2048, 64, torch.float64, 1),
                       (70000, 2048, 4096, torch.float64, 1), (30000, 512, 999, torch.float32, 1), (20000, 4096, 100, torch.float32, 1),
                       (3000, 48, 40, torch.float64, 3)]:
    A = torch.randn(n, d, dtype=dt, device="cuda", generator=g)
    a = run(A, m, 5, False, s); b = run(A, m, 5, True, s); torch.cuda.synchronize()
    print(f"n={n} d={d} m={m} {dt} s={s}: bitwise {'OK' if torch.equal(a, b) else 'DIFF'}", flush=True)
n, d = 1 << 20, 2048
A = torch.empty(n, d, dtype=torch.float64, device="cuda").normal_()
for m in (64, 128, 256, 512, 2048, 65536):
    for pipe in (False, True):
        ms = t(lambda: run(A, m, 7, pipe))
        print(f"sjlt {'pipe' if pipe else 'old '} n={n} d={d} m={m}: {ms*1e3:.1f} us  {(n+m)*d*8/ms/1e6:.0f} GB/s", flush=True)
