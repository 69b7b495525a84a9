"""Dev probe: SRHT / SJLT / Gaussian sketch time for config shapes."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2104_14101_b200.embeddings import srht_dev, sjlt_dev, gaussian_dev
def t(fn, k=5):
    fn(); fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k
which = os.environ.get("WHICH", "srht")
if which == "srht":
    n, d = 1 << 16, 1024
    A = torch.randn(n, d, dtype=torch.float64, device="cuda")
    for m in (32, 256, 1024, 4096):
        ms = t(lambda: srht_dev(A, m, 7))
        print(f"srht n={n} d={d} m={m}: {ms*1e3:.1f} us  {(n+m)*d*8/ms/1e6:.0f} GB/s", flush=True)
if which == "srht4":
    n, d = 1 << 21, 1024
    A = torch.randn(n, d, dtype=torch.float32, device="cuda")
    for m in (64, 1024, 4096, 32768):
        ms = t(lambda: srht_dev(A, m, 7), 3)
        print(f"srht fp32 n={n} d={d} m={m}: {ms*1e3:.1f} us  {(n+m)*d*4/ms/1e6:.0f} GB/s", flush=True)
if which == "sjlt":
    n, d = 1 << 20, 2048
    A = torch.empty(n, d, dtype=torch.float64, device="cuda").normal_()
    for m in [int(x) for x in os.environ.get("MS", "64,2048,65536").split(",")]:
        ms = t(lambda: sjlt_dev(A, m, 7))
        print(f"sjlt n={n} d={d} m={m}: {ms*1e3:.1f} us  {(n+m)*d*8/ms/1e6:.0f} GB/s", flush=True)
if which == "gauss":
    n, d = 4096, 256
    A = torch.randn(n, d, dtype=torch.float64, device="cuda")
    for m in (16, 256):
        ms = t(lambda: gaussian_dev(A, m, 7))
        print(f"gauss n={n} d={d} m={m}: {ms*1e3:.1f} us", flush=True)
