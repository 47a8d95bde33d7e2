"""CPU tests of the rsylv-bench restatements: the number format and
CSV records (records.py, run_record.cpp / matrix_io.cpp), the generators and the mt19937_64
stream of the verification suites (testgen.py, testgen.cpp / verify.cpp), pinned to the
unmodified reference through tests/golden/cli_golden.json (make_cli_golden.py) and, when
oracle/_ref is built, live; plus the CLI argument surface and its no-device behaviour."""
import ctypes as C
import io
import json
import os
import struct

import numpy as np
import pytest

from paper_1905_10574_b200 import cli
from paper_1905_10574_b200 import records as rec
from paper_1905_10574_b200 import testgen as tg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "cli_golden.json")))
REF_SO = os.path.join(ROOT, "oracle", "_ref", "librsylv_ref.so")


def _f(bits):
    return struct.unpack("<d", struct.pack("<Q", bits))[0]


def test_format_double_matches_reference_golden():
    bad = [(s, rec.format_double(_f(b))) for b, s in GOLD["format_double"]
           if rec.format_double(_f(b)) != s]
    assert not bad, bad[:5]


@pytest.mark.skipif(not os.path.exists(REF_SO), reason="oracle/_ref not built")
def test_format_double_matches_reference_live():
    L = C.CDLL(REF_SO)
    L.ref_format_double.argtypes = [C.c_double, C.c_char_p, C.c_size_t]
    buf = C.create_string_buffer(64)
    rng = np.random.default_rng(7)
    vals = list(rng.integers(0, 2 ** 63, 20000, dtype=np.uint64).view(np.float64))
    vals += list(rng.uniform(-1e9, 1e9, 5000)) + [2.0 ** e for e in range(-1074, 1024, 7)]
    for v in vals:
        if v != v:
            continue
        L.ref_format_double(float(v), buf, 64)
        assert rec.format_double(float(v)) == buf.value.decode(), v


def test_format_double_round_trips_and_special_values():
    for v in [0.0, -0.0, 1e-300, 5e-324, 1.7976931348623157e308, 0.1, 2 / 3, -12345.678]:
        assert rec.parse_double(rec.format_double(v)) == v
    assert rec.format_double(float("inf")) == "inf" and rec.format_double(-float("inf")) == "-inf"
    assert rec.format_double(100.0) == "100" and rec.format_double(1e5) == "1e+05"
    for bad in ["", " 1", "1 ", "+1", "1,0", "abc"]:
        with pytest.raises(ValueError):
            rec.parse_double(bad)


def test_csv_round_trip_bitwise_and_header():
    rows = [rec.RunRecord("robust-tiled", 1024, 512, 256, 8, 1024.0, 512.0, 1.7976931348623157e308,
                          2.0 ** -30, 0.123456789, 3.3e-17, 2.0 ** -31, 17, True, 1),
            rec.RunRecord("nonrobust", 8, 8, 256, 0, 0.001, 0.01, 1e4, 1.0, 1e-5, 0.0, 1.0, 0,
                          False, 1)]
    for g in (False, True):
        fh = io.StringIO()
        rec.write_csv(fh, rows, gpus=g)
        text = fh.getvalue()
        assert text.splitlines()[0] == rec.csv_header(g)
        back = rec.read_csv(io.StringIO(text))
        assert back == rows
    # the reference's exact 14-column header (run_record.cpp:35-38)
    assert rec.csv_header() == ("solver,m,n,tile_size,workers,mu,nu,omega,alpha,"
                                "wall_time_seconds,residual,min_local_alpha,scaling_events,median")
    with pytest.raises(ValueError):
        rec.read_csv(io.StringIO("solver,m\n"))
    with pytest.raises(ValueError):
        rec.parse_csv_row("a,b,c")


def test_matrix_file_round_trip(tmp_path):
    a = np.asfortranarray(np.random.default_rng(1).standard_normal((5, 3)) * 1e200)
    p = str(tmp_path / "a.txt")
    rec.write_matrix_file(p, a)
    assert open(p).readline() == "5 3\n"
    assert np.array_equal(rec.read_matrix_file(p), a)
    with pytest.raises(ValueError):
        rec.read_matrix(io.StringIO("2 2\n1 2 3\n"))


def test_mt19937_64_known_answer():
    r = tg.MT19937_64()
    for _ in range(9999):
        r()
    assert r() == 9981545732273789042  # C++ standard [rand.predef]


def test_random_system_matches_reference_golden():
    g = GOLD["random_system"]
    rng = tg.MT19937_64(g["seed"])
    a, ac = tg.random_quasi_triangular(rng, g["m"])
    b, bc = tg.random_quasi_triangular(rng, g["n"])
    c = tg.random_dense(rng, g["m"], g["n"])
    u = lambda x: [int(v) for v in x.reshape(-1, order="F").view(np.uint64)]  # noqa: E731
    assert u(a) == g["a"] and u(b) == g["b"] and u(c) == g["c"]
    assert ac.tolist() == g["ab"] and bc.tolist() == g["bb"]


@pytest.mark.skipif(not os.path.exists(REF_SO), reason="oracle/_ref not built")
@pytest.mark.parametrize("seed,m,n", [(1, 2, 3), (42, 40, 20), (99, 33, 17)])
def test_random_system_matches_reference_live(seed, m, n):
    L = C.CDLL(REF_SO)
    a = np.zeros((m, m), order="F"); b = np.zeros((n, n), order="F"); c = np.zeros((m, n), order="F")
    ab = np.zeros(m, np.uint8); bb = np.zeros(n, np.uint8)
    dp = lambda x: x.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731
    up = lambda x: x.ctypes.data_as(C.POINTER(C.c_ubyte))  # noqa: E731
    assert L.ref_random_system(C.c_uint64(seed), C.c_size_t(m), C.c_size_t(n), dp(a), up(ab),
                               dp(b), up(bb), dp(c)) == 0
    rng = tg.MT19937_64(seed)
    A, ac = tg.random_quasi_triangular(rng, m)
    B, bc = tg.random_quasi_triangular(rng, n)
    Cm = tg.random_dense(rng, m, n)
    assert np.array_equal(A, a) and np.array_equal(B, b) and np.array_equal(Cm, c)
    assert np.array_equal(ac, ab) and np.array_equal(bc, bb)


@pytest.mark.skipif(not os.path.exists(REF_SO), reason="oracle/_ref not built")
@pytest.mark.parametrize("n,pattern", [(1, 0), (2, 0), (9, 0), (9, 1), (64, 0)])
def test_generators_match_reference(n, pattern):
    L = C.CDLL(REF_SO)
    out = np.zeros((n, n), order="F")
    blk = np.zeros(n, np.uint8)
    assert L.ref_generate_quasi_triangular(C.c_size_t(n), C.c_double(2.5), pattern,
                                           out.ctypes.data_as(C.POINTER(C.c_double)),
                                           blk.ctypes.data_as(C.POINTER(C.c_ubyte))) == 0
    a, codes = tg.generate_quasi_triangular(n, 2.5, tg.mixed_pattern(n) if pattern == 0
                                            else tg.ones_pattern(n))
    assert np.array_equal(a, out) and np.array_equal(codes, blk)


def test_generator_patterns_and_errors():
    assert tg.mixed_pattern(5) == [1, 2, 1, 1] and tg.mixed_pattern(6) == [1, 2, 1, 2]
    assert tg.ones_pattern(3) == [1, 1, 1]
    with pytest.raises(ValueError):
        tg.generate_quasi_triangular(3, 0.0, [1, 1, 1])
    with pytest.raises(ValueError):
        tg.generate_quasi_triangular(3, 1.0, [1, 1])
    with pytest.raises(ValueError):
        tg.generate_rhs(0, 3)
    assert np.array_equal(tg.generate_rhs(2, 3), np.ones((2, 3)))


def test_cli_surface_defaults():
    p = cli.build_parser()
    a = p.parse_args(["bench"])
    assert (a.solver, a.m, a.n, a.tile_size, a.workers, a.reps, a.pattern) == \
        ("robust-tiled", 1024, 1024, 256, [0], 3, "mixed")
    a = p.parse_args(["bench", "--mu", "1,2.5", "--workers", "0,8", "--solver", "nonrobust"])
    assert a.mu == [1.0, 2.5] and a.workers == [0, 8]
    a = p.parse_args(["tune"])
    assert (a.tile_min, a.tile_max, a.tile_step) == (32, 256, 32)
    a = p.parse_args(["verify", "--sizes", "6,10"])
    assert a.sizes == [6, 10] and a.count == 3 and a.seed == 42 and a.tolerance == 1e-11
    with pytest.raises(SystemExit):
        p.parse_args(["bench", "--solver", "cholesky"])


def test_cli_bad_tune_range_is_an_error(capsys):
    assert cli.main(["tune", "--tile-min", "1"]) == 2
    assert "error: tune: bad tile range" in capsys.readouterr().err


def test_cli_without_device_fails_loudly(capsys):
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    assert cli.main(["verify", "--sizes", "6", "--count", "1"]) == 2
    assert "no_device" in capsys.readouterr().err


def test_bartels_stewart_host_parts():
    from paper_1905_10574_b200 import bartels_stewart as bs
    rng = np.random.default_rng(0)
    a = rng.standard_normal((9, 9))
    t, u = bs.schur_real(a)
    assert np.allclose(u @ t @ u.T, a, atol=1e-12)
    assert np.allclose(np.tril(t, -2), 0.0)
    with pytest.raises(ValueError):
        bs.solve_sylvester(np.eye(3), np.eye(2), np.ones((3, 3)))
