import sys, os, dataclasses
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch
from paper_1905_10574_b200 import api
from paper_1905_10574_b200.configs import CONFIGS, device_system
for name, m in [("c5", 2048), ("c5", 4096), ("c5", 8192), ("c5", 16384), ("c2", 8000), ("c5", 40000)]:
    cfg = CONFIGS[name].scaled(m) if m != CONFIGS[name].m else CONFIGS[name]
    A, ac, B, bc, C = device_system(cfg, torch)
    Y = torch.empty((cfg.n, cfg.m), dtype=torch.float64, device="cuda").T
    for sched in (0, 1):
        st, res = api.solve_tiled_robust_device(A, ac, B, bc, C, Y, cfg.tile, scheduler=sched, raise_underflow=False)
        bad = ~torch.isfinite(Y)
        nb = int(bad.sum())
        where = None
        if nb:
            idx = bad.nonzero()[:3].tolist()
            where = idx
        print(name, m, "sched", sched, "alpha_exp", res.alpha_exp, "nonfinite", nb, where, flush=True)
