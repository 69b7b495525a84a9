"""Per-role cycle accounting of the tcgen05 Gaussian kernel (ADASK_TC_DEBUG |= 128),
first CTA pair, cycles per pipeline stage."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_14101_b200.embeddings import gaussian_dev  # noqa: E402

n, d, m = 1 << 21, 4096, int(os.environ.get("M", 2048))
A = torch.randn(n, d, device="cuda")
for v in [int(x) for x in os.environ.get("VARS", "128,136,132,140").split(",")]:
    os.environ["ADASK_TC_DEBUG"] = str(v)
    out = torch.zeros(m, d, device="cuda")
    gaussian_dev(A, m, 7, tf32=True, out=out)
    torch.cuda.synchronize()
    o = out.reshape(-1)[:32].cpu().tolist()
    for c in (0, 1):
        b = o[16 * c:16 * c + 16]
        nk = max(b[6], 1)
        print(f"dbg={v} cta{c}: stages={nk:.0f} loop {b[4]/nk:.0f} cyc/stage, total {b[5]/nk:.0f} | producer wait-empty "
              f"{b[0]/nk:.0f} | mma wait-full {b[1]/nk:.0f} | gen wait-empty {b[2]/nk:.0f} named-bar {b[3]/nk:.0f}")
