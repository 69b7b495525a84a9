"""Layout debugging for the tcgen05 Gaussian kernel (ADASK_TC_DEBUG=1 makes
S[r, k] = [r == k mod 128]; the sketch then equals sum of A rows)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_14101_b200.embeddings import gaussian_dev  # noqa: E402

np.set_printoptions(linewidth=200)
m, n, d = 128, 128, 256
scale = np.sqrt(m)
# 1) A = row ids encoded: A[k, j] = k + 1000 * j  -> SA[r, j] should be r + 1000 j
A = (np.arange(n)[:, None] + 1000.0 * np.arange(d)[None, :]).astype(np.float32)
Ad = torch.from_numpy(A).cuda()
os.environ["ADASK_TC_DEBUG"] = "1"
got = gaussian_dev(Ad, m, 1, tf32=True).cpu().numpy() * scale
print("case1 max err", np.abs(got - A[:m]).max())
bad = np.argwhere(np.abs(got - A[:m]) > 0.5)
print("bad count", len(bad))
for r, j in bad[:40]:
    v = got[r, j]
    print(f"SA[{r},{j}] = {v:.1f}  want {A[r, j]:.1f}")
# 2) small integers, check decode of which (k, j) contributed
A2 = np.zeros((n, d), np.float32)
A2[np.arange(n), np.arange(n) % d] = 1.0
got2 = gaussian_dev(torch.from_numpy(A2).cuda(), m, 1, tf32=True).cpu().numpy() * scale
print("case2 nonzeros per row (want 1 at col r):")
for r in range(0, 128, 9):
    print(r, np.nonzero(np.abs(got2[r]) > 0.5)[0][:8], got2[r][np.abs(got2[r]) > 0.5][:8])
