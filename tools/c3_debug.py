import sys, os, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "oracle"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np, pyoracle as po, bigrange as br
import paper_1905_10574_b200 as rs
from paper_1905_10574_b200.configs import CONFIGS, host_system
for name, n, t in [("c3", 16, 256), ("c3", 40, 8), ("c3", 64, 256), ("c3", 64, 16), ("c3", 64, 5), ("c3", 96, 32),
                   ("c3", 128, 40), ("c3", 128, 256), ("c2", 96, 16), ("c5", 96, 24), ("c5", 128, 64)]:
    cfg = CONFIGS[name].scaled(n, tile=t)
    a, ac, b, bc, c = host_system(cfg)
    A = rs.QuasiTriangular.from_codes(a, ac); B = rs.QuasiTriangular.from_codes(b, bc)
    for sched in (0, 1):
        try:
            r = rs.solve_tiled_robust(A, B, c, t, scheduler=sched); st = "ok"
        except rs.ScaleUnderflowError as e:
            r = e.result; st = "underflow"
        fin = bool(np.isfinite(r.y).all())
        res = po.relative_residual_safe(a, b, c, r.y, 1.0, r.alpha_exp) if fin else None
        Y = br.solve(a, ac, b, bc, c)
        d = br.rel_inf_diff_exp(r.y, r.alpha_exp, Y) if fin else None
        print(name, n, t, "sched", sched, st, "alpha_exp", r.alpha_exp, "finite", fin, "resid", res,
              "vs_bigrange", d, "log10max", round(br.log10_max_abs(Y), 1), "ev", r.scaling_events, flush=True)
cfg = CONFIGS["c3"]
import torch
from paper_1905_10574_b200 import api
from paper_1905_10574_b200.configs import device_system
A, ac, B, bc, Cm = device_system(cfg, torch)
Yd = torch.empty((cfg.n, cfg.m), dtype=torch.float64, device="cuda").T
for sched in (0, 1):
    st, res = api.solve_tiled_robust_device(A, ac, B, bc, Cm, Yd, cfg.tile, scheduler=sched, raise_underflow=False)
    print("c3 full sched", sched, "status", st, "alpha_exp", res.alpha_exp, "finite", bool(torch.isfinite(Yd).all()),
          "nonfinite", int((~torch.isfinite(Yd)).sum()), "dag_ms", res.dag_ms, flush=True)
