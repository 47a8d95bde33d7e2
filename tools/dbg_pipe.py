import sys, time, numpy as np
sys.path.insert(0, '.')
from paper_1905_10574_b200 import api, testgen as tg, _native as nat
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100
a, ac = tg.generate_quasi_triangular(n, 1e-3, tg.mixed_pattern(n))
b, bc = tg.generate_quasi_triangular(n, 1e-2, tg.mixed_pattern(n))
c = tg.generate_rhs(n, n)
for hp, use_probe in [(1, False), (1, False), (1, True), (1, False), (-1, False), (1, False)]:
    ev = []
    t0 = time.time()
    try:
        r = api.solve_tiled_robust(api.QuasiTriangular.from_codes(a, ac), api.QuasiTriangular.from_codes(b, bc), c, 8,
                                   api.OverflowConfig(omega=1e4), probe=(lambda *x: ev.append(x)) if use_probe else None, host_pipeline=hp)
        print(hp, use_probe, "ok", r.alpha_exp, len(ev), round(time.time() - t0, 2), flush=True)
    except Exception as e:
        print(hp, use_probe, "EXC", e, round(time.time() - t0, 2), flush=True)
