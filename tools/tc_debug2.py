"""Dump of pipeline stage 0 (S tile + A tile) of the tcgen05 Gaussian kernel."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_14101_b200.embeddings import gaussian_dev  # noqa: E402

np.set_printoptions(linewidth=220)
m, n, d = 128, 128, 256
A = (np.arange(n)[:, None] + 1000.0 * np.arange(d)[None, :]).astype(np.float32)
os.environ["ADASK_TC_DEBUG"] = "2"
out = gaussian_dev(torch.from_numpy(A).cuda(), m, 1, tf32=True).cpu().numpy().reshape(-1)
S = out[:2048].reshape(16, 128)  # byte offset / 4
B = out[2048:2048 + 4096]
print("S stage raw (first rows of 128B = 32 floats):")
for r in range(0, 20):
    print(r, S.reshape(-1)[r * 32:(r + 1) * 32].astype(int))
print("B stage raw, first 20 128B rows:")
for r in range(20):
    print(r, B[r * 32:(r + 1) * 32].astype(int))
print("nonzero in B:", np.count_nonzero(B), "of", B.size)
