"""Dev: per-item phase times of the fused SRHT from a -DFUSED_TRACE build.

    ADASK_NVCC_EXTRA=-DFUSED_TRACE python -m paper_2104_14101_b200.buildlib --force
    M=4096 python tools/srht_trace.py          # GPU: runs one sketch, prints the phase table
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_14101_b200.embeddings import srht_dev  # noqa: E402

m = int(os.environ.get("M", 4096))
A = torch.randn(1 << 16, 1024, dtype=torch.float64, device="cuda")
for _ in range(3):
    srht_dev(A, m, 7)
torch.cuda.synchronize()
path = "/tmp/srht_trace.bin"
os.environ["ADASK_SRHT_FUSED_TRACE"] = path
srht_dev(A, m, 7)
torch.cuda.synchronize()
del os.environ["ADASK_SRHT_FUSED_TRACE"]
t = np.fromfile(path, dtype=np.uint64).reshape(148, 2, -1, 12).astype(np.int64)
kind = t[..., 0]
for kd, name in ((1, "pass 1"), (2, "pass 2")):
    sel = kind == kd
    if not sel.any():
        continue
    r = t[sel]
    ph = {"wait full": r[:, 2] - r[:, 1], "load+bfly5": r[:, 3] - r[:, 2], "wait xdone": r[:, 4] - r[:, 3],
          "exchange": r[:, 5] - r[:, 4] if kd == 1 else None, "tail": r[:, 6] - (r[:, 5] if kd == 1 else r[:, 4]),
          "item": r[:, 6] - r[:, 1]}
    if kd == 1:
        ph.update({" bfly4": r[:, 10] - r[:, 5], " z stores": r[:, 7] - r[:, 10], " proxy fence": r[:, 8] - r[:, 7],
                   " group barrier": r[:, 9] - r[:, 8], " threadfence+atomic": r[:, 6] - r[:, 9]})
    print(f"{name}: {sel.sum()} items")
    for k, v in ph.items():
        if v is None:
            continue
        print(f"   {k:12s} mean {v.mean():8.0f} ns  p50 {np.median(v):8.0f}  p90 {np.percentile(v, 90):8.0f}")
t0 = t[..., 1][kind > 0].min()
t1 = t[..., 6].max()
print(f"kernel span (traced items) {t1 - t0} ns; items per group: {np.count_nonzero(kind, axis=2).mean():.1f}")
# idle between items of a group
gaps = []
for b in range(148):
    for g in range(2):
        k = np.count_nonzero(kind[b, g])
        if k > 1:
            gaps.append(t[b, g, 1:k, 1] - t[b, g, :k - 1, 6])
gaps = np.concatenate(gaps)
print(f"gap between a group's items: mean {gaps.mean():.0f} ns")
