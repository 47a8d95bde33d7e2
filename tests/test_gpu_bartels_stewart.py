"""Bartels–Stewart wrapper: general A X + X B = alpha C through real
Schur forms, GPU transforms and the robust triangular engine; checked against LAPACK's
scipy.linalg.solve_sylvester and by residual."""
import numpy as np
import pytest

from paper_1905_10574_b200 import bartels_stewart as bs

pytestmark = pytest.mark.gpu


def _system(m, n, seed, rot=False):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((m, m)) / np.sqrt(m) + 3.0 * np.eye(m)
    b = rng.standard_normal((n, n)) / np.sqrt(n) + 2.0 * np.eye(n)
    if rot:  # strongly complex spectra: many 2x2 Schur blocks
        for k in range(0, m - 1, 2):
            a[k, k + 1] += 2.0
            a[k + 1, k] -= 2.0
        for k in range(0, n - 1, 2):
            b[k, k + 1] += 1.5
            b[k + 1, k] -= 1.5
    c = rng.standard_normal((m, n))
    return a, b, c


@pytest.mark.parametrize("m,n,rot,tile", [(150, 120, False, 128), (97, 203, True, 64),
                                          (256, 256, True, 128), (5, 3, True, 2)])
def test_matches_lapack_solve_sylvester(m, n, rot, tile):
    import scipy.linalg
    a, b, c = _system(m, n, m * 7 + n, rot)
    x, ae = bs.solve_sylvester(a, b, c, tile_size=tile)
    assert ae == 0
    ref = scipy.linalg.solve_sylvester(a, b, c)
    assert np.abs(x - ref).max() <= 1e-10 * np.abs(ref).max()
    assert bs.residual(a, b, c, x, ae) <= 1e-14


def test_reuses_schur_factorizations():
    a, b, c = _system(64, 48, 3, True)
    sa, sb = bs.schur_real(a), bs.schur_real(b)
    x1, _ = bs.solve_sylvester(a, b, c, schur_a=sa, schur_b=sb)
    x2, _ = bs.solve_sylvester(a, b, 2.0 * c, schur_a=sa, schur_b=sb)
    assert np.allclose(x2, 2.0 * x1, rtol=1e-13, atol=0)


def test_scaling_path_keeps_x_finite():
    from paper_1905_10574_b200 import OverflowConfig
    a, b, c = _system(80, 80, 11)
    # shift the spectra so A + B is nearly singular in many directions: large solutions
    a = a - 3.0 * np.eye(80) + 1e-3 * np.eye(80)
    b = b - 2.0 * np.eye(80) + 1e-3 * np.eye(80)
    cfg = OverflowConfig(omega=1e4)
    x, ae = bs.solve_sylvester(a, b, c, tile_size=16, cfg=cfg)
    assert np.isfinite(x).all()
    assert bs.residual(a, b, c, x, ae) <= 1e-12
