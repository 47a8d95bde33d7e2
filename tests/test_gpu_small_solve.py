"""Direct GPU tests of the diagonal-tile solver's pieces, ported from the reference's unit suites:
* the exact block solve (complete-pivoting Kronecker solve + division guard; the path every
  sub-block takes when the fast closed forms refuse) -- tests/test_small_solve.cpp:39-123,
  compared with the reference's solve_small_sylvester (oracle/_ref) on the same inputs;
* the exponent-form guards -- tests/test_overflow.cpp:68-99 (contract and idempotence over
  random inputs incl. the boundary values 0, 1, omega/2, omega).
Scale factors are powers of two here (2^-dz) where the reference uses Omega(1-2^-30)/growth:
the solutions agree as Z / scale, and the scale agrees to within one binade."""
import math

import numpy as np
import pytest

import pyoracle as po

pytestmark = pytest.mark.gpu
EPS = 2.0 ** -53


def api():
    from paper_1905_10574_b200 import api as a
    return a


def rot2(re, im):
    return np.array([[re, im], [-im, re]])


def s1(v):
    return np.array([[float(v)]])


def small_residual(a, b, c, z, dz):
    return np.abs(math.ldexp(1.0, -dz) * c - a @ z - z @ b).sum(axis=1).max()


def test_one_by_one_exact():  # test_small_solve.cpp:39-45
    (st, z, dz, _), = api().debug_small_solve([(s1(1), s1(1), s1(2))])
    assert st == 0 and dz == 0 and z[0, 0] == 1.0


def test_opposite_eigenvalues_are_singular():  # :47-52
    (st, z, dz, piv), = api().debug_small_solve([(s1(1), s1(-1), s1(1))])
    rst, _, _, rpiv = po.small_sylvester(s1(1), s1(-1), s1(1), impl="ref")
    assert st == 2 and rst == po.SINGULAR and piv == rpiv == 0.0


def test_two_by_two_pair_vs_reference():  # :54-76
    a, b, c = rot2(1, 1), rot2(1, 1), np.ones((2, 2))
    (st, z, dz, _), = api().debug_small_solve([(a, b, c)])
    rst, zr, beta, _ = po.small_sylvester(a, b, c, impl="ref")
    assert st == 0 and dz == 0 and beta == 1.0
    assert np.abs(z - zr).max() <= 1e-14 * np.abs(zr).max()


def test_tiny_eigenvalue_pair_scales():  # :78-87
    (st, z, dz, _), = api().debug_small_solve([(s1(1e-8), s1(1e-8), s1(1))], omega=1e4)
    rst, zr, beta, _ = po.small_sylvester(s1(1e-8), s1(1e-8), s1(1), omega=1e4, impl="ref")
    assert st == 0 and dz > 0 and beta < 1.0
    assert abs(z[0, 0]) <= 1e4
    assert 2e-8 * z[0, 0] == pytest.approx(math.ldexp(1.0, -dz), rel=1e-15)
    # same solution up to the scale: z / 2^-dz == zr / beta
    assert math.ldexp(z[0, 0], dz) == pytest.approx(zr[0, 0] / beta, rel=1e-14)
    assert abs(-dz - math.log2(beta)) <= 1.0


def test_backward_stable_random_blocks_vs_reference():  # :89-109 (500 cases)
    rng = np.random.default_rng(37)
    cases = []
    for _ in range(500):
        a2, b2 = rng.integers(0, 2, 2)
        mag = lambda: rng.uniform(0.5, 1.5)  # noqa: E731
        a = rot2(mag(), mag()) if a2 else s1(mag())
        b = rot2(mag(), mag()) if b2 else s1(mag())
        c = rng.uniform(-1, 1, (a.shape[0], b.shape[0]))
        cases.append((a, b, c))
    out = api().debug_small_solve(cases)
    for (a, b, c), (st, z, dz, _) in zip(cases, out):
        assert st == 0 and dz == 0
        nrm = lambda x: np.abs(x).sum(axis=1).max()  # noqa: E731
        bound = 50 * EPS * ((nrm(a) + nrm(b)) * nrm(z)) + 50 * EPS * nrm(c)
        assert small_residual(a, b, c, z, dz) <= bound
        rst, zr, beta, _ = po.small_sylvester(a, b, c, impl="ref")
        assert rst == 0 and beta == 1.0
        assert np.abs(z - zr).max() <= 1e-13 * max(1.0, np.abs(zr).max())


def test_two_column_blocks_never_exceed_omega():  # :111-123 (200 cases)
    rng = np.random.default_rng(41)
    cases = []
    for _ in range(200):
        a = rot2(rng.uniform(1e-4, 2e-4), rng.uniform(1e-4, 2e-4))
        b = rot2(rng.uniform(1e-4, 2e-4), rng.uniform(1e-4, 2e-4))
        c = np.ones((2, 2))
        c[0, 1] = -1.0
        cases.append((a, b, c))
    out = api().debug_small_solve(cases, omega=10.0)
    for (a, b, c), (st, z, dz, _) in zip(cases, out):
        assert st == 0
        assert np.abs(z).sum(axis=1).max() <= 10.0
        assert dz > 0  # beta < 1
        rst, zr, beta, _ = po.small_sylvester(a, b, c, omega=10.0, impl="ref")
        assert rst == 0 and beta < 1.0
        assert np.abs(np.ldexp(z, dz) - zr / beta).max() <= 1e-12 * np.abs(zr / beta).max()
        assert abs(-dz - math.log2(beta)) <= 1.0


@pytest.mark.parametrize("omega", [1e4, float(np.finfo(float).max / 2)])
def test_guards_contract_and_idempotence(omega):  # test_overflow.cpp:68-99
    rng = np.random.default_rng(31)
    boundary = np.array([0.0, 1.0, omega, omega / 2])
    n = 20000
    draw = lambda lane: np.where(np.arange(n) % 5 == lane,  # noqa: E731
                                 boundary[rng.integers(0, 4, n)], rng.uniform(0, 1, n) * omega)
    c, a, b = draw(0), draw(1), draw(2)
    bnd = np.where(np.arange(n) % 7 == 0, boundary[rng.integers(0, 4, n)], rng.uniform(0, 1, n) * omega)
    t = 10.0 ** rng.uniform(-300, 300, n) * np.where(rng.integers(0, 2, n) == 1, -1.0, 1.0)
    dq, df, dd = api().debug_guards(c, a, b, bnd, t, omega)
    target = omega * (1 - 2.0 ** -30)
    for d in (dq, df):
        assert (d >= 0).all()
        # contract: zeta * growth <= omega with zeta = 2^-d, evaluated exactly in log2 form
        with np.errstate(all="ignore"):  # log2 of the growth c + a b without overflow
            lg = np.logaddexp2(np.log2(c), np.log2(a) + np.log2(b))
        zero = np.isneginf(lg)
        ok = (lg - d <= math.log2(omega) + 1e-12) | zero
        assert ok.all()
        # no scaling when none is required
        assert (d[(lg <= math.log2(omega) - 1e-12) | zero] == 0).all()
        # the scale is within one binade of the least power of two meeting the target
        need = lg > math.log2(omega) + 1e-12
        assert (lg[need] - d[need] <= math.log2(target) + 1e-12).all()
        assert (lg[need] - (d[need] - 1) > math.log2(target) - 1.0).all()
    # the integer (xq) form fires no later than the exact (xf) form, at most one binade earlier
    assert ((dq - df >= 0) & (dq - df <= 1)).all()
    # division guard: bnd / |t| scaled below omega, none when not needed
    q = np.log2(bnd.astype(np.float64)) - np.log2(np.abs(t))
    pos = bnd > 0
    assert (q[pos] - dd[pos] <= math.log2(omega) + 1e-12).all()
    assert (dd[pos & (q <= math.log2(omega) - 1e-12)] == 0).all()
