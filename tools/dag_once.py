"""One DAG solve of a (scaled) config, for ncu captures (development tool).
    python tools/dag_once.py c5 16000   -> c5 distributions at 16000^2 (hot tiles kept)"""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch
from paper_1905_10574_b200 import api
from paper_1905_10574_b200.configs import CONFIGS, device_system
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c5"]
if len(sys.argv) > 2:
    cfg = cfg.scaled(int(sys.argv[2]))
A, ac, B, bc, Cm = device_system(cfg, torch)
Y = torch.empty((cfg.n, cfg.m), dtype=torch.float64, device="cuda").T
reps = int(os.environ.get("REPS", "1"))
for _ in range(reps):
    st, res = api.solve_tiled_robust_device(A, ac, B, bc, Cm, Y, cfg.tile, raise_underflow=False)
    print(cfg.name, "status", st, "dag_ms %.2f" % res.dag_ms, "GF/s %.0f" % (cfg.flops() / res.dag_ms / 1e6),
          "alpha_exp", res.alpha_exp, "events", res.scaling_events)
