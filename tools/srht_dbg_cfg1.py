import os, sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests/golden")
import numpy as np, torch
from recipes import baseline_instance
from paper_2104_14101_b200.embeddings import srht_dev
A, b, lam = baseline_instance(1, 65536)
Ad = torch.from_numpy(A).cuda()
print("A", A.dtype, A.flags["C_CONTIGUOUS"], Ad.stride(), Ad.data_ptr() % 256)
for m in [32, 64, 128, 256, 512, 1024, 2048, 4096]:
    os.environ["ADASK_SRHT_FUSED"] = "0"; r = srht_dev(Ad, m, 12345)
    os.environ["ADASK_SRHT_FUSED"] = "1"; f = srht_dev(Ad, m, 12345)
    bad = (r != f)
    print(m, int(bad.sum()), bad.any(1).nonzero().flatten()[:5].tolist(), bad.any(0).nonzero().flatten()[:10].tolist(), float((r-f).abs().max()))
