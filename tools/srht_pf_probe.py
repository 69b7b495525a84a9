"""Dev: SRHT pipe timing vs L2 prefetch distance and in-place/scratch variant."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2104_14101_b200.embeddings import srht_dev
def t(fn, k=3):
    fn(); fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k
for (n, d, dt, ms_) in ((1 << 16, 1024, torch.float64, (32, 4096)), (1 << 21, 1024, torch.float32, (64, 32768))):
    A = torch.randn(n, d, dtype=dt, device="cuda")
    for ip in ("0", "1"):
        for pf in ("0", "1", "2", "4", "8"):
            os.environ["ADASK_FWHT_IP"] = ip; os.environ["ADASK_FWHT_PF"] = pf
            r = []
            for m in ms_:
                ms = t(lambda: srht_dev(A, m, 7))
                r.append(f"m={m}: {ms*1e3:8.1f} us {(n+m)*d*A.element_size()/ms/1e6:5.0f} GB/s")
            print(f"n={n} {dt} ip={ip} pf={pf}: " + " | ".join(r), flush=True)
    del A
