"""Generates tests/golden/*.npz from the UNMODIFIED reference library (oracle/_ref, built from
/root/reference/proj/src by oracle/Makefile). Run in the dev container (where /root/reference
exists):  python tests/golden/make_golden.py

Each fixture re-creates an input of the reference's own test suites (same generators, seeds,
omegas and tile sizes; file:line cited in the `origin` field) or a BASELINE-config twin, and
stores the reference outputs: status, alpha, scaling events, Y.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, ROOT)
import pyoracle as po  # noqa: E402
from paper_1905_10574_b200.configs import CONFIGS, host_system  # noqa: E402

WIDE = float(np.finfo(np.float64).max)
cases = {}


def add(name, origin, a, ab, b, bb, c, tile, omega, workers=0):
    r = po.solve_tiled(a, ab, b, bb, c, tile, omega=omega, impl="ref", workers=workers)
    cases[name] = dict(origin=origin, a=a, ab=ab, b=b, bb=bb, c=c, tile=tile, omega=omega,
                       status=r.status, alpha=r.alpha, events=r.events,
                       y=r.y if r.y is not None else np.zeros(0), pivot=r.pivot)
    print(f"{name:28s} status={po.STATUS_NAMES[r.status]:22s} alpha={r.alpha:.4e} ev={r.events}")


# test_tiled_solve.cpp:62-74 -- random 40x37 system, tiles {2,3,5,8,40}, omega = DBL_MAX
a, ab, b, bb, c = po.ref_random_system(71, 40, 37)
for ts in (2, 3, 5, 8, 40):
    add(f"oracle_tiles_t{ts}", "test_tiled_solve.cpp:62-74", a, ab, b, bb, c, ts, WIDE)
# test_tiled_solve.cpp:30-43 -- single tile, mixed pattern, omega 1e6
for n, mu, nu in ((7, 0.5, 0.8), (12, 0.5, 0.8), (20, 0.5, 0.8)):
    a, ab = po.ref_generate_quasi_triangular(n, mu)
    b, bb = po.ref_generate_quasi_triangular(n, nu)
    add(f"single_tile_n{n}", "test_tiled_solve.cpp:30-43", a, ab, b, bb, np.ones((n, n)), 2 * n, 1e6)
# test_tiled_solve.cpp:45-60 -- single tile under growth, omega 1e4
a, ab = po.ref_generate_quasi_triangular(30, 1e-3)
b, bb = po.ref_generate_quasi_triangular(30, 1e-2)
add("single_tile_growth_n30", "test_tiled_solve.cpp:45-60", a, ab, b, bb, np.ones((30, 30)), 30, 1e4)
# test_tiled_solve.cpp:94-111 -- growth system n=100, tile 25, omega 1e4
a, ab = po.ref_generate_quasi_triangular(100, 1e-3)
b, bb = po.ref_generate_quasi_triangular(100, 1e-2)
add("growth_n100_t25", "test_tiled_solve.cpp:94-111", a, ab, b, bb, np.ones((100, 100)), 25, 1e4)
# test_tiled_solve.cpp:113-135 -- at-rest bounded tiles n=64, tile 16
a, ab = po.ref_generate_quasi_triangular(64, 1e-3)
b, bb = po.ref_generate_quasi_triangular(64, 1e-2)
add("atrest_n64_t16", "test_tiled_solve.cpp:113-135", a, ab, b, bb, np.ones((64, 64)), 16, 1e4)
# acceptance_main.cpp:154-184 -- criterion 3 supplementary (n=100, tile 64, omega 1e4)
for mu in (1e-3, 1e-7):
    a, ab = po.ref_generate_quasi_triangular(100, mu)
    b, bb = po.ref_generate_quasi_triangular(100, 1e-2)
    add(f"crit3supp_mu{mu:g}", "acceptance_main.cpp:154-184", a, ab, b, bb, np.ones((100, 100)),
        64, 1e4)
# test_tiled_solve.cpp:218-226 -- ScaleUnderflowError at n=200 (ones pattern, tile 64)
a, ab = po.ref_generate_quasi_triangular(200, 1e-3, "ones")
b, bb = po.ref_generate_quasi_triangular(200, 1e-2, "ones")
add("underflow_n200", "test_tiled_solve.cpp:218-226", a, ab, b, bb, np.ones((200, 200)), 64, 1e4)
# test_tiled_solve.cpp:228-239 -- singular system (b_55 = -1)
a = np.eye(8)
b = np.eye(8)
b[5, 5] = -1.0
add("singular_n8", "test_tiled_solve.cpp:228-239", a, None, b, None, np.ones((8, 8)), 4, 0.0)
# test_tiled_solve.cpp:241-248 -- rhs tile above omega rejected
add("rhs_above_omega", "test_tiled_solve.cpp:241-248", np.eye(4), None, np.eye(4), None,
    np.ones((4, 4)), 4, 2.0)
# acceptance_main.cpp:188-211 -- criterion 4 benign regime (mu = m)
for (m, n) in ((100, 100), (80, 60)):
    a, ab = po.ref_generate_quasi_triangular(m, float(m))
    b, bb = po.ref_generate_quasi_triangular(n, float(n))
    add(f"crit4_{m}x{n}", "acceptance_main.cpp:188-211", a, ab, b, bb, np.ones((m, n)),
        max(m, n), 0.0)
# acceptance_main.cpp:57-81 -- criterion 1 (first 10 of the 50 systems, tile 8, DBL_MAX)
import ctypes  # noqa: E402
for s in range(10):
    a, ab, b, bb, c = po.ref_random_system(1001 + s, 3 + (7 * s) % 38, 3 + (11 * s) % 38)
    add(f"crit1_sys{s}", "acceptance_main.cpp:57-81 (seeded variant)", a, ab, b, bb, c, 8, WIDE)
# BASELINE-config twins at small sizes (configs.py generators)
for name, n, t in (("c1", 160, 32), ("c2", 160, 32), ("c4", 192, 32), ("c5", 192, 64),
                   ("c3", 16, 256)):
    cfg = CONFIGS[name].scaled(n if name != "c4" else n, n if name != "c4" else n // 4, t)
    a, ab, b, bb, c = host_system(cfg)
    add(f"twin_{name}_{cfg.m}x{cfg.n}_t{t}", f"BASELINE config {name} distributions", a, ab, b,
        bb, c, t, 0.0)

np.savez_compressed(os.path.join(HERE, "reference_solves.npz"),
                    **{f"{k}__{f}": (np.asarray(v) if v is not None else np.zeros(0))
                       for k, d in cases.items() for f, v in d.items()})

# guard known answers (test_overflow.cpp:31-66) + randomized guard pairs (crit. 8 style)
rng = np.random.default_rng(8008)
pu = [(0.0, 2.0, 100.0, 100.0), (1e4, 1e4, 1e4, 1e4), (0.0, 0.0, 0.0, 1e4)]
pu += [(float(x), float(y), float(z), 1e4) for x, y, z in rng.uniform(0, 1e4, (200, 3))]
pd = [(1e4, 1e-2, 1e4), (1.0, 0.5, 1e4)]
pd += [(float(x), float(10.0 ** e) * (1 if s else -1), 1e4)
       for x, e, s in zip(rng.uniform(0, 1e4, 200), rng.uniform(-300, 300, 200), rng.integers(0, 2, 200))]
zu = np.array([po.protect_update(*t, impl="ref")[1] for t in pu])
zd = np.array([po.protect_division(*t, impl="ref")[1] for t in pd])
np.savez_compressed(os.path.join(HERE, "guards.npz"), pu=np.array(pu), zu=zu, pd=np.array(pd), zd=zd)

# robust_update cases (test_robust_update.cpp:110-135 style): random tiles, scales 2^-k
ru = {}
rng = np.random.default_rng(53)
for t in range(60):
    m, k, n = rng.integers(1, 5, 3)
    g, al, be = 2.0 ** -rng.integers(0, 4, 3)
    c = rng.uniform(-2, 2, (m, n))
    a = rng.uniform(-2, 2, (m, k))
    b = rng.uniform(-2, 2, (k, n))
    st, y, s, nr, ev = po.robust_update(c, g, po.inf_norm(c), a, al, po.inf_norm(a), b, be,
                                        po.inf_norm(b), omega=50.0, impl="ref")
    ru[f"{t}"] = np.concatenate([[m, k, n, g, al, be, st, s, nr], c.ravel("F"), a.ravel("F"),
                                 b.ravel("F"), y.ravel("F")])
np.savez_compressed(os.path.join(HERE, "robust_update.npz"), **ru)
print("written", len(cases), "solve fixtures")
