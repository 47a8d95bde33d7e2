"""Quick GPU-vs-oracle shakeout used during development (not the test suite)."""
import sys, time, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "oracle"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import pyoracle as po
import paper_1905_10574_b200 as rs

WIDE = np.finfo(np.float64).max

def rel(a, b):
    d = np.abs(a - b).sum(axis=1).max(); r = np.abs(b).sum(axis=1).max()
    return d / r if r else d

def run(a, ab, b, bb, c, ts, omega, sched, label):
    A = rs.QuasiTriangular.from_codes(a, ab); B = rs.QuasiTriangular.from_codes(b, bb)
    ref = po.solve_tiled(a, ab, b, bb, c, ts, omega=omega, impl="ref", workers=8)
    cfg = rs.OverflowConfig(omega=omega)
    t0 = time.time()
    try:
        r = rs.solve_tiled_robust(A, B, c, ts, cfg, scheduler=sched)
        st = 0
    except rs.ScaleUnderflowError as e:
        r = e.result; st = 3
    except Exception as e:
        print(label, "GPU EXC", type(e).__name__, e); return
    dt = time.time() - t0
    if ref.status != 0:
        print(label, "ref status", ref.status, "gpu st", st, "alpha_exp", r.alpha_exp if r else None); return
    yg = r.y / r.alpha if r.alpha > 0 else None
    yr = ref.y / ref.alpha
    print(f"{label}: sched={sched} ts={ts} gpu_alpha=2^{r.alpha_exp} ref_alpha={ref.alpha:.3e} "
          f"rel={rel(yg, yr) if yg is not None else 'n/a'} maxnorm={r.max_tile_norm:.3e} "
          f"ev={r.scaling_events} dev_ms={r.device_ms:.2f} wall={dt:.2f}s finite={np.isfinite(r.y).all()}")

for sched in (1, 0):
    a, ab, b, bb, c = po.ref_random_system(71, 40, 37)
    for ts in (2, 3, 5, 8, 40):
        run(a, ab, b, bb, c, ts, WIDE, sched, "rand40x37")
    a, ab = po.ref_generate_quasi_triangular(100, 1e-3); b, bb = po.ref_generate_quasi_triangular(100, 1e-2)
    c = np.ones((100, 100))
    run(a, ab, b, bb, c, 25, 1e4, sched, "growth100")
    for seed in (1, 2):
        a, ab, b, bb, c = po.ref_random_system(seed, 300, 260)
        run(a, ab, b, bb, c, 64, WIDE, sched, "rand300")
        run(a, ab, b, bb, c, 128, 0.0, sched, "rand300d")
# robust update
rng = np.random.default_rng(5)
for (m, k, n) in [(2, 2, 2), (3, 5, 7), (128, 128, 128), (100, 120, 90)]:
    C = rng.uniform(-1, 1, (m, n)); A = rng.uniform(-1, 1, (m, k)); B = rng.uniform(-1, 1, (k, n))
    out, e, nrm, ev = rs.robust_update(C, 0, A, B, 0)
    want = C - A @ B
    print("robust_update", m, k, n, "exp", e, "rel", rel(out, want), "norm", nrm)
out, e, nrm, ev = rs.robust_update(np.zeros((2, 2)), 0, np.eye(2), np.eye(2), -1, omega=1e4)
print("eta case:", out, e)
