"""Multi-GPU exchange validated on one GPU: tile columns block-cyclic over R virtual ranks, each
with its own workspace, solved tiles pushed into the consuming ranks' workspaces, one
cooperative persistent kernel (the device code of the one-process-per-GPU path with peer
pointers into the same device). Every tile sees the same sources in the same order, so the result
must be bitwise identical to the single-rank solve."""
import numpy as np
import pytest

import golden
import pyoracle as po

pytestmark = pytest.mark.gpu
CASES = golden.solves()


def solve(d, R, tile=None):
    import paper_1905_10574_b200 as m
    A = m.QuasiTriangular.from_codes(d["a"], d["ab"] if d["ab"] is not None else np.ones(d["a"].shape[0], np.uint8))
    B = m.QuasiTriangular.from_codes(d["b"], d["bb"] if d["bb"] is not None else np.ones(d["b"].shape[0], np.uint8))
    cfg = m.OverflowConfig(omega=d["omega"] if d["omega"] > 0 else m.default_omega())
    try:
        return 0, m.solve_tiled_robust(A, B, d["c"], tile or d["tile"], cfg, virtual_ranks=R)
    except m.ScaleUnderflowError as e:
        return 3, e.result
    except m.SingularEquationError as e:
        return 2, e


@pytest.mark.parametrize("R", [2, 3, 8])
@pytest.mark.parametrize("name", ["growth_n100_t25", "atrest_n64_t16", "oracle_tiles_t5",
                                  "underflow_n200", "twin_c2_160x160_t32", "twin_c5_192x192_t64",
                                  "twin_c4_192x48_t32"])
def test_virtual_ranks_bitwise_equal_single_rank(name, R):
    d = CASES[name]
    s1, r1 = solve(d, 1)
    sR, rR = solve(d, R)
    assert s1 == sR
    assert r1.alpha_exp == rR.alpha_exp
    assert np.array_equal(r1.y, rR.y)


def test_virtual_ranks_singular_stops_every_rank():
    d = CASES["singular_n8"]
    s, e = solve(d, 4, tile=2)
    assert s == 2 and e.pivot == d["pivot"]


def test_virtual_ranks_larger_system():
    from paper_1905_10574_b200.configs import CONFIGS, host_system
    cfg = CONFIGS["c5"].scaled(700, 650, 128)
    a, ac, b, bc, c = host_system(cfg)
    d = dict(a=a, ab=ac, b=b, bb=bc, c=c, tile=128, omega=0.0)
    s1, r1 = solve(d, 1)
    for R in (2, 4):
        sR, rR = solve(d, R)
        assert sR == s1 and np.array_equal(r1.y, rR.y)
    ref = po.solve_tiled(a, ac, b, bc, c, 128, impl="ref", workers=8)
    if ref.status == 0:
        mant, ex = np.frexp(ref.alpha)
        got = np.ldexp(r1.y * mant, int(ex) - r1.alpha_exp)
        assert golden.rel_inf_diff(got, ref.y) <= 1e-10


@pytest.mark.parametrize("name", ["growth_n100_t25", "twin_c5_192x192_t64", "singular_n8"])
def test_virtual_ranks_with_system_scope(name, monkeypatch):
    """RSYLV_B200_SYS_SCOPE=1: the one-rank-per-GPU memory model (ld.acquire.sys /
    st.release.sys flags, __threadfence_system before every push and publish, system-scope
    atomics on the peers' error words) on virtual ranks of one GPU -- the device code of the
    multi-GPU push path, bitwise equal to the single-rank solve."""
    monkeypatch.setenv("RSYLV_B200_SYS_SCOPE", "1")
    d = CASES[name]
    s1, r1 = solve(d, 1)
    for R in (2, 4):
        sR, rR = solve(d, R)
        assert s1 == sR
        if s1 == 2:
            assert rR.pivot == r1.pivot
            continue
        assert r1.alpha_exp == rR.alpha_exp and np.array_equal(r1.y, rR.y)


@pytest.mark.parametrize("w", [2, 4, 8])
def test_execution_mode_workers_map_to_ranks(w, monkeypatch):
    """ExecutionMode::parallel(w) (tiled_solve.hpp:16-22) reaches the multi-GPU path: with one
    visible GPU and RSYLV_B200_VIRTUAL_RANKS=1 it runs min(w, 8) virtual ranks; results are
    bitwise those of sequential() (acceptance criterion 5, acceptance_main.cpp:213-236)."""
    import paper_1905_10574_b200 as m
    monkeypatch.setenv("RSYLV_B200_VIRTUAL_RANKS", "1")
    d = CASES["twin_c2_160x160_t32"]
    A = m.QuasiTriangular.from_codes(d["a"], d["ab"])
    B = m.QuasiTriangular.from_codes(d["b"], d["bb"])
    r0 = m.solve_tiled_robust(A, B, d["c"], 32, mode=m.ExecutionMode.sequential())
    rw = m.solve_tiled_robust(A, B, d["c"], 32, mode=m.ExecutionMode.parallel(w))
    assert r0.alpha_exp == rw.alpha_exp and np.array_equal(r0.y, rw.y)


def test_group_solve_api_contract():
    """rsylv_b200_solve_group: R = 1 is the single-GPU solve; contexts must be distinct GPUs."""
    import ctypes as C
    import paper_1905_10574_b200 as m
    from paper_1905_10574_b200 import _native as nat
    d = CASES["twin_c2_160x160_t32"]
    A = m.QuasiTriangular.from_codes(d["a"], d["ab"])
    B = m.QuasiTriangular.from_codes(d["b"], d["bb"])
    ref = m.solve_tiled_robust(A, B, d["c"], 32)
    mm, nn = d["c"].shape
    cf = np.asfortranarray(d["c"])
    y = np.zeros((mm, nn), order="F")
    opt = nat.Options(m.default_omega(), m.default_small_num(), 32, 0, 0, 0, 0)
    res = nat.Result()
    dp = lambda x: x.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731
    up = lambda x: x.ctypes.data_as(C.POINTER(C.c_ubyte))  # noqa: E731
    am, bm = A.matrix(), B.matrix()
    L = nat.lib()
    one = (C.c_void_p * 1)(nat.context(0))
    st = L.rsylv_b200_solve_group(one, 1, mm, nn, dp(am), mm, up(A.codes), dp(bm), nn,
                                  up(B.codes), dp(cf), mm, dp(y), mm, C.byref(opt), C.byref(res))
    assert st == nat.RSYLV_OK and res.alpha_exp == ref.alpha_exp and np.array_equal(y, ref.y)
    two = (C.c_void_p * 2)(nat.context(0), nat.context(0))
    st = L.rsylv_b200_solve_group(two, 2, mm, nn, dp(am), mm, up(A.codes), dp(bm), nn,
                                  up(B.codes), dp(cf), mm, dp(y), mm, C.byref(opt), C.byref(res))
    assert st == nat.RSYLV_INVALID_ARGUMENT
    assert L.rsylv_b200_device_count() >= 1
