"""Host pipeline of rsylv_b200_solve (inputs streamed in shells while the DAG runs -- tile row of
A from its diagonal on, tile column of B, the matching L-shaped piece of C;
include/rsylv_b200.h host_pipeline): results are bitwise those of the upfront path, and the
argument checks keep the reference's order and reason codes."""
import numpy as np
import pytest

import golden
import pyoracle as po
from paper_1905_10574_b200 import api
from paper_1905_10574_b200.configs import CONFIGS, host_system

pytestmark = pytest.mark.gpu


def qt(a, codes):
    return api.QuasiTriangular.from_codes(a, codes) if codes is not None else api.QuasiTriangular(a)


def _both(a, ac, b, bc, c, tile, cfg=None):
    out = []
    for hp in (-1, 1):
        out.append(api.solve_tiled_robust(qt(a, ac), qt(b, bc), c, tile, cfg, host_pipeline=hp))
    return out


@pytest.mark.parametrize("group", [None, "1", "3"])
@pytest.mark.parametrize("m,n,tile", [(300, 260, 32), (700, 650, 128), (129, 1000, 64), (1000, 129, 64),
                                      (520, 40, 8)])
def test_pipeline_bitwise_equals_upfront(m, n, tile, group, monkeypatch):
    # (group: shells whose copies are issued together, runtime.cpp RSYLV_B200_SHELL_GROUP;
    #  default 8, here also 1 and a size that does not divide the shell count)
    if group is not None:
        monkeypatch.setenv("RSYLV_B200_SHELL_GROUP", group)
    cfg = CONFIGS["c5"].scaled(m, n, tile)
    a, ac, b, bc, c = host_system(cfg)
    r0, r1 = _both(a, ac, b, bc, c, tile)
    assert r0.alpha_exp == r1.alpha_exp and r0.scaling_events == r1.scaling_events
    assert np.array_equal(r0.y, r1.y)


def test_pipeline_growth_system_matches_reference():
    d = golden.solves()["growth_n100_t25"]
    cfg = api.OverflowConfig(omega=d["omega"])
    r = api.solve_tiled_robust(qt(d["a"], d["ab"]), qt(d["b"], d["bb"]), d["c"], 8, cfg,
                               host_pipeline=1)
    mant, ex = np.frexp(d["alpha"])
    got = np.ldexp(r.y * mant, int(ex) - r.alpha_exp)
    assert golden.rel_inf_diff(got, d["y"]) <= 1e-12


@pytest.mark.parametrize("pos", [(250, 3), (3, 250), (3, 100), (130, 130)])
def test_pipeline_c_check_in_every_shell_piece(pos):
    """A C entry above omega is caught wherever its tile travels: the column piece of an early
    shell (bottom left), of the last shell (top right), a row strip, the corner tile."""
    cfg = CONFIGS["c1"].scaled(256, 256, 32)
    a, ac, b, bc, c = host_system(cfg)
    c = c.copy(order="F")
    c[pos] = 1e7
    om = api.OverflowConfig(omega=1e6)
    msgs = []
    for hp in (1, -1):
        with pytest.raises(ValueError) as e:
            api.solve_tiled_robust(qt(a, ac), qt(b, bc), c, 32, om, host_pipeline=hp)
        msgs.append(str(e.value))
    assert "norm of C" in msgs[0] and msgs[0] == msgs[1]


@pytest.mark.parametrize("which,reason", [("a", "norm of A"), ("b", "norm of B"), ("c", "norm of C")])
def test_pipeline_argument_checks_in_reference_order(which, reason):
    cfg = CONFIGS["c1"].scaled(256, 256, 32)
    a, ac, b, bc, c = host_system(cfg)
    om = api.OverflowConfig(omega=1e6)
    a, b, c = a.copy(order="F"), b.copy(order="F"), c.copy(order="F")
    if which == "a":
        a[0, 200] = 1e7
        c[5, 5] = 1e7  # an A violation is reported first even when C also fails
    elif which == "b":
        b[10, 250] = 1e7
        c[5, 5] = 1e7
    else:
        c[100, 3] = 1e7
    with pytest.raises(ValueError) as e:
        api.solve_tiled_robust(qt(a, ac), qt(b, bc), c, 32, om, host_pipeline=1)
    assert reason in str(e.value)
    with pytest.raises(ValueError) as e2:
        api.solve_tiled_robust(qt(a, ac), qt(b, bc), c, 32, om, host_pipeline=-1)
    assert str(e.value) == str(e2.value)


def test_pipeline_singular_like_upfront():
    d = golden.solves()["singular_n8"]
    for hp in (-1, 1):
        with pytest.raises(api.SingularEquationError) as e:
            api.solve_tiled_robust(qt(d["a"], None), qt(d["b"], None), d["c"], 2, host_pipeline=hp)
        assert e.value.pivot == d["pivot"]


def test_pipeline_reuse_after_failure():
    """A failed (aborted) pipelined solve leaves the context usable."""
    cfg = CONFIGS["c5"].scaled(400, 400, 64)
    a, ac, b, bc, c = host_system(cfg)
    bad = c.copy(order="F")
    bad[7, 300] = np.inf
    with pytest.raises(ValueError):
        api.solve_tiled_robust(qt(a, ac), qt(b, bc), bad, 64, host_pipeline=1)
    r0, r1 = _both(a, ac, b, bc, c, 64)
    assert np.array_equal(r0.y, r1.y)


@pytest.mark.parametrize("hp", [1, -1])
def test_probe_log_complete_with_pipeline(hp):
    """TileProbe (tiled_solve.hpp:24-27) completeness, also for the DAG CTAs the host pipeline
    launches on its side stream (>= 64 tiles). The reference probes after every robust update
    and after the tile solve (tiled_solve.cpp:49,60,71); the left-looking GPU task probes the
    tile once after its whole update phase and once at rest, so every tile appears exactly
    twice, the update event first."""
    cfg = CONFIGS["c5"].scaled(1100, 1030, 128)
    a, ac, b, bc, c = host_system(cfg)
    ev = []
    r = api.solve_tiled_robust(qt(a, ac), qt(b, bc), c, 128, host_pipeline=hp,
                               probe=lambda k, l, s, nr: ev.append((k, l, s, nr)))
    rc, cc = api.tile_cuts(ac, cfg.m, 128), api.tile_cuts(bc, cfg.n, 128)
    M, N = len(rc) - 1, len(cc) - 1
    assert M * N >= 64
    keys = sorted((k, l) for k, l, _, _ in ev)
    assert keys == sorted(2 * [(k, l) for k in range(M) for l in range(N)]), "missing/extra tiles"
    assert all(0.0 <= nr <= api.default_omega() and 0.0 <= s <= 1.0 for _, _, s, nr in ev)


def test_pipeline_survives_serialized_launches():
    """CUDA_LAUNCH_BLOCKING=1 serializes the streams: the host pipeline enqueues every producer
    before the spinning DAG kernel, so the solve still completes (no watchdog) and is bitwise
    the concurrent result."""
    import os
    import subprocess
    import sys
    code = r'''
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
from paper_1905_10574_b200 import api
from paper_1905_10574_b200.configs import CONFIGS, host_system
cfg = CONFIGS["c5"].scaled(1100, 1030, 128)
a, ac, b, bc, c = host_system(cfg)
r = api.solve_tiled_robust(api.QuasiTriangular.from_codes(a, ac), api.QuasiTriangular.from_codes(b, bc), c, 128, host_pipeline=1)
np.save(sys.argv[2], r.y)
print(r.alpha_exp)
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = os.path.join(root, "gpurun_out", "serialized_y.npy")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    env = dict(os.environ, CUDA_LAUNCH_BLOCKING="1")
    p = subprocess.run([sys.executable, "-c", code, root, out], env=env, capture_output=True,
                       text=True, timeout=300)
    assert p.returncode == 0, p.stderr[-3000:]
    cfg = CONFIGS["c5"].scaled(1100, 1030, 128)
    a, ac, b, bc, c = host_system(cfg)
    r = api.solve_tiled_robust(qt(a, ac), qt(b, bc), c, 128, host_pipeline=1)
    assert int(p.stdout.split()[-1]) == r.alpha_exp
    assert np.array_equal(np.load(out), r.y)
    os.remove(out)


def test_pageable_buffers_page_locked_for_the_call(monkeypatch):
    """The reference's DenseMatrix storage is pageable: with RSYLV_B200_HOST_REGISTER=1
    rsylv_b200_solve page-locks buffers of >= 64 MB for the call (so the host pipeline's
    per-column copies stay asynchronous) and unregisters them afterwards; bitwise the same
    result as without registration (the default: pinning per call is not profitable)."""
    cfg = CONFIGS["c1"].scaled(3000, 3000, 128)
    a, ac, b, bc, c = host_system(cfg)
    assert a.nbytes >= 64 << 20
    monkeypatch.setenv("RSYLV_B200_HOST_REGISTER", "1")
    r1 = api.solve_tiled_robust(qt(a, ac), qt(b, bc), c, 128)
    monkeypatch.setenv("RSYLV_B200_HOST_REGISTER", "0")
    r0 = api.solve_tiled_robust(qt(a, ac), qt(b, bc), c, 128)
    assert r1.alpha_exp == r0.alpha_exp and np.array_equal(r1.y, r0.y)
    # registration is released: the same buffers can be registered again by the next call
    monkeypatch.setenv("RSYLV_B200_HOST_REGISTER", "1")
    r2 = api.solve_tiled_robust(qt(a, ac), qt(b, bc), c, 128)
    assert np.array_equal(r2.y, r0.y)
