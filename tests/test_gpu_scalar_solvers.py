"""GPU counterparts of the reference's scalar solvers:
solve_nonrobust (scalar_solve.cpp:130-138) and solve_robust_scalar (:140-149)."""
import numpy as np
import pytest

import golden
import pyoracle as po

pytestmark = pytest.mark.gpu
CASES = golden.solves()


def qt(m, codes):
    import paper_1905_10574_b200 as rs
    return rs.QuasiTriangular.from_codes(m, codes if codes is not None else np.ones(m.shape[0], np.uint8))


@pytest.mark.parametrize("name", ["oracle_tiles_t8", "crit4_100x100", "crit4_80x60", "twin_c1_160x160_t32"])
def test_nonrobust_matches_reference(name):
    import paper_1905_10574_b200 as rs
    d = CASES[name]
    y = rs.solve_nonrobust(qt(d["a"], d["ab"]), qt(d["b"], d["bb"]), d["c"])
    ref = po.solve_nonrobust(d["a"], d["ab"], d["b"], d["bb"], d["c"], impl="ref")
    assert ref.status == 0
    assert golden.rel_inf_diff(y, ref.y) <= 1e-12


def test_nonrobust_overflows_like_the_reference():
    """acceptance_main.cpp:139-147: on the growth system the non-robust solver leaves the
    omega = 1e4 range (here it overflows outright, as the reference's does)."""
    import paper_1905_10574_b200 as rs
    d = CASES["underflow_n200"]
    y = rs.solve_nonrobust(qt(d["a"], d["ab"]), qt(d["b"], d["bb"]), d["c"])
    ref = po.solve_nonrobust(d["a"], d["ab"], d["b"], d["bb"], d["c"], impl="ref")
    assert not np.all(np.abs(y) <= 1e4)
    assert np.isfinite(y).sum() == np.isfinite(ref.y).sum() or not np.isfinite(y).all()


@pytest.mark.parametrize("n", [128, 200, 300])
def test_nonrobust_inf_propagates_through_tiles(n):
    """Non-robust (omega = +inf) on a growth system that overflows, over several 128-tiles: no
    guard may fire and nothing may be rescaled, so the entries the reference's plain substitution
    keeps finite come out equal (the engine's exponent-form accumulation avoids some of the
    reference's intermediate overflows, so it may keep MORE entries finite, never markedly fewer).
    """
    import paper_1905_10574_b200 as rs
    a, ac = po.ref_generate_quasi_triangular(n, 1e-3)
    b, bc = po.ref_generate_quasi_triangular(n, 1e-2)
    c = np.ones((n, n))
    y = rs.solve_nonrobust(qt(a, ac), qt(b, bc), c)
    ref = po.solve_nonrobust(a, ac, b, bc, c, impl="ref")
    fg, fr = np.isfinite(y), np.isfinite(ref.y)
    assert not fr.all() and not fg.all()
    assert (fr & ~fg).sum() <= 0.01 * fr.sum()
    both = fg & fr & (np.abs(ref.y) > 0)
    rel = np.abs(y[both] - ref.y[both]) / np.abs(ref.y[both])
    assert np.median(rel) <= 1e-10 and np.quantile(rel, 0.9) <= 1e-8


def test_nonrobust_singular():
    import paper_1905_10574_b200 as rs
    d = CASES["singular_n8"]
    with pytest.raises(rs.SingularEquationError):
        rs.solve_nonrobust(qt(d["a"], None), qt(d["b"], None), d["c"])


@pytest.mark.parametrize("name", ["single_tile_growth_n30", "growth_n100_t25", "crit4_80x60"])
def test_robust_scalar_matches_reference(name):
    import paper_1905_10574_b200 as rs
    d = CASES[name]
    cfg = rs.OverflowConfig(omega=d["omega"] if d["omega"] > 0 else rs.default_omega())
    r = rs.solve_robust_scalar(qt(d["a"], d["ab"]), qt(d["b"], d["bb"]), d["c"], cfg)
    ref = po.solve_robust_scalar(d["a"], d["ab"], d["b"], d["bb"], d["c"], omega=d["omega"], impl="ref")
    assert ref.status == 0
    mant, ex = np.frexp(ref.alpha)
    got = np.ldexp(r.y * mant, int(ex) - r.alpha_exp)
    assert golden.rel_inf_diff(got, ref.y) <= 1e-12
