import sys, numpy as np
sys.path.insert(0, '.')
from paper_1905_10574_b200 import api, _native as nat
from paper_1905_10574_b200.configs import CONFIGS, host_system
cfg = CONFIGS["c1"].scaled(256, 256, 32)
a, ac, b, bc, c0 = host_system(cfg)
for (ri, ci) in [(100, 3), (100, 200), (10, 250), (250, 10)]:
    c = c0.copy(order="F"); c[ri, ci] = 1e7
    out = []
    for hp in (-1, 1):
        try:
            r = api.solve_tiled_robust(api.QuasiTriangular.from_codes(a, ac), api.QuasiTriangular.from_codes(b, bc), c, 32, api.OverflowConfig(omega=1e6), host_pipeline=hp)
            out.append(f"ok a={r.alpha_exp}")
        except Exception as e:
            out.append(f"EXC {e}")
    print((ri, ci), out, flush=True)
