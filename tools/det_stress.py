"""Repeated device-resident solves of one config, compared bitwise on the device (development
tool: the persistent DAG's race detector at scale).  python tools/det_stress.py c5 [size] [reps]"""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch
from paper_1905_10574_b200 import api
from paper_1905_10574_b200.configs import CONFIGS, device_system
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c5"]
if len(sys.argv) > 2 and int(sys.argv[2]) > 0:
    cfg = cfg.scaled(int(sys.argv[2]))
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 8
A, ac, B, bc, C = device_system(cfg, torch)
Y0 = torch.empty((cfg.n, cfg.m), dtype=torch.float64, device="cuda").T
st0, r0 = api.solve_tiled_robust_device(A, ac, B, bc, C, Y0, cfg.tile, raise_underflow=False)
Y1 = torch.empty_like(Y0)
bad = 0
for k in range(reps):
    Y1.fill_(float("nan"))
    st, r = api.solve_tiled_robust_device(A, ac, B, bc, C, Y1, cfg.tile, raise_underflow=False)
    ne = int((Y1.view(torch.int64) != Y0.view(torch.int64)).sum().item())
    if ne or st != st0 or r.alpha_exp != r0.alpha_exp or r.scaling_events != r0.scaling_events:
        bad += 1
        d = (Y1 - Y0).abs()
        rel = float((d / Y0.abs().clamp_min(1e-300)).nan_to_num(0.0).max().item())
        print(f"  run {k}: {ne} entries differ (max rel {rel:.2e}), events {r.scaling_events} vs {r0.scaling_events}, alpha_exp {r.alpha_exp} vs {r0.alpha_exp}")
print(f"{cfg.name} {cfg.m}x{cfg.n}: {bad} of {reps} repeat solves differ from the first; dag_ms {r.dag_ms:.1f}")
