"""Dev: A/B of an env toggle on the fp32 2^21 x 1024 block SRHT (interleaved)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2104_14101_b200.embeddings import srht_dev
var = os.environ.get("VAR", "ADASK_FWHT_NOMASK")
def t(fn, k=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k
A = torch.randn(1 << 21, 1024, dtype=torch.float32, device="cuda")
for m in (64, 1024, 4096, 32768):
    res = {"on": [], "off": []}
    for rep in range(3):
        for mode in ("on", "off"):
            if mode == "on": os.environ.pop(var, None)
            else: os.environ[var] = "1"
            res[mode].append(t(lambda: srht_dev(A, m, 7)))
    print(f"m={m}: default {min(res['on']):.3f} ms  {var}=1 {min(res['off']):.3f} ms", flush=True)
