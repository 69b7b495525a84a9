"""Dev: native adaptive PCG-SRHT on the config-1 instance, fused SRHT on/off,
with and without a prior Python-path SRHT call in the same context."""
import os, sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests/golden")
import numpy as np, torch
import paper_2104_14101_b200 as ak
from recipes import baseline_instance
from paper_2104_14101_b200.embeddings import srht_dev
mode = sys.argv[1]
A, b, lam = baseline_instance(1, 65536)
p = ak.RegularizedProblem(torch.from_numpy(A), b, 1e-2, lam)
if mode == "warm":
    srht_dev(p.A_dev, 64, 1)
acfg = ak.AdaptiveConfig.for_method("pcg", 0.125, 32, 11, "srht", 1)
try:
    x, tr = ak.adaptive_run(p, np.zeros(1024), acfg, method="pcg", native=True)
    print(mode, os.environ.get("ADASK_SRHT_FUSED"), "ok", tr.schedule())
except Exception as e:
    print(mode, os.environ.get("ADASK_SRHT_FUSED"), "FAIL", e)
