"""Dev: repeated launches of the kernels changed in round 2 against CPU results
(rare-race / stale-flag hunting): random-size dataflow Cholesky factorizations
and inverses, fused SRHT sketches (all three row-count ranges), fp64 Gaussian."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_14101_b200 as ak  # noqa: E402
from oracle import adasketch_oracle as O  # noqa: E402
from paper_2104_14101_b200.embeddings import srht_dev  # noqa: E402

rng = np.random.default_rng(int(os.environ.get("SEED", 0)))
t0 = time.time()
nchol = nsrht = 0
worst = 0.0
while time.time() - t0 < float(os.environ.get("SECONDS", 60)):
    k = int(rng.choice([33, 64, 100, 256, 300, 512, 777, 1024, 1500]))
    dt = rng.choice(["float64", "float32"])
    X = rng.standard_normal((k + 8, k))
    M = X.T @ X / k + np.eye(k)
    L = ak.cholesky(M if dt == "float64" else M.astype(np.float32))
    Lo = np.linalg.cholesky(M)
    err = np.linalg.norm(np.asarray(L, dtype=np.float64) - Lo) / np.linalg.norm(Lo)
    tol = 1e-11 if dt == "float64" else 2e-5
    assert err <= tol, (k, dt, err)
    worst = max(worst, err / tol)
    nchol += 1
    if nchol % 4 == 0:
        n = int(rng.choice([2048, 5024, 1 << 15, 1 << 16]))
        d = int(rng.choice([8, 17, 40]))
        m = int(rng.choice([16, 300, 2000]))
        A = rng.standard_normal((n, d))
        got = srht_dev(torch.from_numpy(A).cuda(), m, nchol).cpu().numpy()
        assert np.array_equal(got, O.sketch_srht(A, m, nchol)), (n, d, m)
        nsrht += 1
print(f"stress ok: {nchol} factorizations (worst err/tol {worst:.2f}), {nsrht} fused SRHT sketches bitwise, {time.time() - t0:.0f} s")
