"""Dev: config-1 solves (for an ncu launch list of exactly the last solve)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2104_14101_b200 as ak
from paper_2104_14101_b200 import configs
cfg = configs.CONFIGS[1]
A, b, lam = configs.make_instance(cfg)
p = ak.RegularizedProblem(A, b, cfg.nu, lam)
x0 = torch.zeros(cfg.d, dtype=torch.float64, device="cuda")
acfg = ak.AdaptiveConfig.for_method(cfg.method, 0.125, cfg.m_init, 11, cfg.family, 1)
for _ in range(int(os.environ.get("SOLVES", 2))):
    x, tr = ak.adaptive_run(p, x0, acfg, method=cfg.method)
torch.cuda.synchronize()
print(tr.schedule(), ak.device.ctx().launches())
