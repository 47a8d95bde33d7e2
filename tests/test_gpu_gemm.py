"""The FP64 DMMA GEMM (rsylv_b200_dgemm) and the device residual (rsylv_b200_relative_residual)
against torch / numpy FP64 references."""
import numpy as np
import pytest

import pyoracle as po

pytestmark = pytest.mark.gpu


def colmajor(torch, x):
    return torch.as_tensor(np.asfortranarray(x), device="cuda").T.contiguous().T


@pytest.mark.parametrize("m,n,k", [(1, 1, 1), (7, 5, 3), (128, 128, 128), (129, 257, 33),
                                   (300, 200, 500), (1000, 64, 700)])
@pytest.mark.parametrize("ta,tb", [(0, 0), (1, 0), (0, 1), (1, 1)])
def test_dgemm_vs_numpy(m, n, k, ta, tb):
    import torch
    from paper_1905_10574_b200 import api
    rng = np.random.default_rng(m * 1000 + n * 10 + k + 7 * ta + 3 * tb)
    a = rng.standard_normal((k, m) if ta else (m, k))
    b = rng.standard_normal((n, k) if tb else (k, n))
    c = rng.standard_normal((m, n))
    A, B, Cd = colmajor(torch, a), colmajor(torch, b), colmajor(torch, c)
    api.dgemm(A, B, Cd, alpha=-1.5, beta=0.25, ta=bool(ta), tb=bool(tb))
    want = -1.5 * (a.T if ta else a) @ (b.T if tb else b) + 0.25 * c
    got = Cd.cpu().numpy()
    scale = (np.abs(a).max() * np.abs(b).max() * k + np.abs(c).max())
    assert np.abs(got - want).max() <= 8 * k * np.finfo(float).eps * scale


@pytest.mark.parametrize("m,n", [(250, 130), (129, 300)])
def test_dgemm_skips_structural_zeros_exactly(m, n):
    """a_upper / b_upper only skip K ranges that are zero in an upper quasi-triangular operand:
    the result equals the dense product."""
    import torch
    from paper_1905_10574_b200 import api
    rng = np.random.default_rng(5)
    a = np.triu(rng.standard_normal((m, m)), -1)
    y = rng.standard_normal((m, n))
    b = np.triu(rng.standard_normal((n, n)), -1)
    A, Y, B = colmajor(torch, a), colmajor(torch, y), colmajor(torch, b)
    R0 = colmajor(torch, np.zeros((m, n)))
    R1 = colmajor(torch, np.zeros((m, n)))
    api.dgemm(A, Y, R0)
    api.dgemm(A, Y, R1, a_upper=True)
    assert torch.equal(R0, R1)
    api.dgemm(Y, B, R0)
    api.dgemm(Y, B, R1, b_upper=True)
    assert torch.equal(R0, R1)


def test_relative_residual_matches_host():
    import torch
    from paper_1905_10574_b200 import api
    from paper_1905_10574_b200.configs import CONFIGS, host_system
    cfg = CONFIGS["c2"].scaled(300, 260, 64)
    a, ac, b, bc, c = host_system(cfg)
    r = api.solve_tiled_robust(api.QuasiTriangular.from_codes(a, ac),
                               api.QuasiTriangular.from_codes(b, bc), c, 64)
    dev = api.relative_residual_device(colmajor(torch, a), colmajor(torch, b), colmajor(torch, c),
                                       colmajor(torch, r.y), r.alpha_exp)
    host = po.relative_residual_safe(a, b, c, r.y, 1.0, r.alpha_exp)
    assert dev["relres"] <= 16 * 300 * 260 * np.finfo(float).eps
    assert abs(dev["relres"] - host) <= 0.05 * host + 1e-18
    # a wrong solution is seen
    yb = np.asfortranarray(r.y.copy())
    yb[np.unravel_index(np.argmax(np.abs(yb)), yb.shape)] *= 1.001  # where it is visible
    bad = api.relative_residual_device(colmajor(torch, a), colmajor(torch, b), colmajor(torch, c),
                                       colmajor(torch, yb), r.alpha_exp)
    assert bad["relres"] > 1e3 * dev["relres"]


def test_relative_residual_near_omega_and_tiny_alpha():
    """Tiles near omega and alpha far below DBL_MIN: the prescaled frame keeps the residual
    finite (the reference's plain evaluation would overflow)."""
    import torch
    from paper_1905_10574_b200 import api
    from paper_1905_10574_b200.configs import CONFIGS, host_system
    cfg = CONFIGS["c3"].scaled(96, tile=32)
    a, ac, b, bc, c = host_system(cfg)
    try:
        r = api.solve_tiled_robust(api.QuasiTriangular.from_codes(a, ac),
                                   api.QuasiTriangular.from_codes(b, bc), c, 32)
    except api.ScaleUnderflowError as e:
        r = e.result
    assert r.alpha_exp < -1022
    dev = api.relative_residual_device(colmajor(torch, a), colmajor(torch, b), colmajor(torch, c),
                                       colmajor(torch, r.y), r.alpha_exp)
    assert np.isfinite(dev["relres"]) and dev["relres"] <= 16 * 96 * 96 * np.finfo(float).eps
