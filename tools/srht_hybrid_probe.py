"""Dev: fp64 SRHT at 2^16 x 1024, tile kernels vs pipelined vs hybrid (pipe pass 1 + tile pass 2)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2104_14101_b200.embeddings import srht_dev
def t(fn, k=10):
    fn(); fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k * 1e3
A = torch.randn(1 << 16, 1024, dtype=torch.float64, device="cuda")
for m in (256, 512, 1024, 2048, 4096):
    r = []
    for mode in ("0", "2", "3"):
        os.environ["ADASK_FWHT_PIPE"] = mode
        r.append(f"{ {'0': 'tile', '2': 'pipe', '3': 'hybrid'}[mode]} {t(lambda: srht_dev(A, m, 7)):6.1f}")
    print(f"m={m}: " + "  ".join(r) + " us", flush=True)
