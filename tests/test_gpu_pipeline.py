"""Host pipeline of rsylv_b200_solve (inputs streamed tile column by tile column while the DAG
runs; include/rsylv_b200.h host_pipeline): results are bitwise those of the upfront path, and
the argument checks keep the reference's order and reason codes."""
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


@pytest.mark.parametrize("m,n,tile", [(300, 260, 32), (700, 650, 128), (129, 1000, 64)])
def test_pipeline_bitwise_equals_upfront(m, n, tile):
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
