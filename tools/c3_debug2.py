import sys, os, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "oracle"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np, pyoracle as po, bigrange as br
from decimal import Decimal
import paper_1905_10574_b200 as rs
from paper_1905_10574_b200.configs import CONFIGS, host_system

def tile_report(n, t):
    cfg = CONFIGS["c3"].scaled(n, tile=t)
    a, ac, b, bc, c = host_system(cfg)
    A = rs.QuasiTriangular.from_codes(a, ac); B = rs.QuasiTriangular.from_codes(b, bc)
    ev = []
    try:
        r = rs.solve_tiled_robust(A, B, c, t, probe=lambda k, l, s, nr: ev.append((k, l, s, nr)))
    except rs.ScaleUnderflowError as e:
        r = e.result
    Y = br.solve(a, ac, b, bc, c)
    M = -(-n // t)
    print(f"n={n} t={t} alpha_exp={r.alpha_exp}")
    for k in range(M):
        row = []
        for l in range(M):
            r0, r1, c0, c1 = k * t, min(n, (k + 1) * t), l * t, min(n, (l + 1) * t)
            yt = r.y[r0:r1, c0:c1]
            Yt = [row_[c0:c1] for row_ in Y[r0:r1]]
            mx = br.log10_max_abs(Yt)
            err = br.rel_inf_diff_exp(yt, r.alpha_exp, Yt)
            row.append(f"{mx:7.0f}:{err:7.1e}")
        print(" ".join(row))
tile_report(64, 16)
tile_report(48, 16)
for n in (256, 512, 1024, 2048, 4096):
    cfg = CONFIGS["c3"].scaled(n, tile=256)
    a, ac, b, bc, c = host_system(cfg)
    A = rs.QuasiTriangular.from_codes(a, ac); B = rs.QuasiTriangular.from_codes(b, bc)
    try:
        r = rs.solve_tiled_robust(A, B, c, 256)
    except rs.ScaleUnderflowError as e:
        r = e.result
    fin = np.isfinite(r.y)
    print("c3", n, "alpha_exp", r.alpha_exp, "nonfinite", int((~fin).sum()), "first", np.argwhere(~fin)[:2].tolist(), flush=True)
