"""rsylv-bench on the GPU engine: the verify suite passes with the
reference's defaults and fails its negative control, bench/tune emit the reference's CSV
records, and the device residual agrees with the reference's relative_residual."""
import io
import os

import numpy as np
import pytest

from paper_1905_10574_b200 import cli
from paper_1905_10574_b200 import records as rec
from paper_1905_10574_b200 import testgen as tg
from paper_1905_10574_b200 import verify as vf

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SO = os.path.join(ROOT, "oracle", "_ref", "librsylv_ref.so")


def test_verify_default_suite_passes(capsys):
    assert cli.main(["verify"]) == 0
    out = capsys.readouterr().out
    assert out.rstrip().endswith("OK") and "verification passed" in out
    assert "min-local-alpha" in out
    # the three sections of verify.cpp in order
    assert out.index("oracle equivalence") < out.index("generator residuals") < \
        out.index("bounded tiles")


def test_verify_negative_control_fails(capsys):
    assert cli.main(["verify", "--sizes", "6,10", "--count", "1", "--inject-bug", "--quiet"]) == 1
    out = capsys.readouterr().out
    assert out.rstrip().endswith("FAILED") and "oracle equivalence" not in out


def test_bench_csv_records(tmp_path, capsys):
    path = str(tmp_path / "runs.csv")
    assert cli.main(["bench", "--m", "96", "--n", "80", "--tile-size", "32", "--reps", "3",
                     "--mu", "96,0.001", "--nu", "0.01", "--omega", "1e4", "--workers", "0,4",
                     "--csv", path, "--gpus-column"]) == 0
    assert "wrote 12 rows to" in capsys.readouterr().out
    rows = rec.read_csv(open(path))
    assert len(rows) == 12 and all(r.gpus == 1 and r.solver == "robust-tiled" for r in rows)
    for g in range(4):  # one lower-median row per repetition group
        grp = rows[3 * g:3 * g + 3]
        assert sum(r.median for r in grp) == 1
        med = [r for r in grp if r.median][0]
        assert sorted(r.wall_time_seconds for r in grp)[1] == med.wall_time_seconds
    benign = [r for r in rows if r.mu == 96.0]
    assert all(r.alpha == 1.0 and r.residual < 1e-14 for r in benign)
    growth = [r for r in rows if r.mu == 0.001]
    assert all(0 < r.alpha < 1.0 and r.scaling_events > 0 and r.residual < 1e-12 for r in growth)
    assert [r.workers for r in rows[:6]] == [0, 0, 0, 4, 4, 4]


@pytest.mark.parametrize("solver", ["nonrobust", "robust-scalar"])
def test_bench_scalar_solvers_stdout(solver, capsys):
    assert cli.main(["bench", "--solver", solver, "--m", "40", "--n", "24", "--reps", "1",
                     "--pattern", "ones"]) == 0
    rows = rec.read_csv(io.StringIO(capsys.readouterr().out))
    assert len(rows) == 1 and rows[0].solver == solver and rows[0].workers == 0
    assert rows[0].residual < 1e-14


def test_bench_dump_matrix_files(tmp_path, capsys):
    pre = str(tmp_path / "sys")
    assert cli.main(["bench", "--m", "12", "--n", "10", "--reps", "1", "--tile-size", "4",
                     "--dump", pre]) == 0
    a = rec.read_matrix_file(pre + "_mu12_a.txt")
    y = rec.read_matrix_file(pre + "_mu12_y.txt")
    b = rec.read_matrix_file(pre + "_mu12_b.txt")
    c = rec.read_matrix_file(pre + "_mu12_c.txt")
    assert a.shape == (12, 12) and y.shape == (12, 10)
    assert np.abs(a @ y + y @ b - c).max() < 1e-12 * np.abs(c).max() * 100


def test_tune_reports_best_tile(capsys):
    assert cli.main(["tune", "--m", "96", "--n", "96", "--tile-min", "32", "--tile-max", "96",
                     "--tile-step", "32", "--reps", "2"]) == 0
    out = capsys.readouterr().out
    rows = rec.read_csv(io.StringIO(out.split("best tile size")[0]))
    assert [r.tile_size for r in rows] == [32, 32, 64, 64, 96, 96]
    best = int(out.split("best tile size: ")[1].split()[0])
    med = {r.tile_size: r.wall_time_seconds for r in rows if r.median}
    assert best == min(med, key=lambda t: (med[t], t))


@pytest.mark.skipif(not os.path.exists(REF_SO), reason="oracle/_ref not built")
def test_device_residual_matches_reference():
    import pyoracle as po
    rng = tg.MT19937_64(5)
    a, ac = tg.random_quasi_triangular(rng, 30)
    b, bc = tg.random_quasi_triangular(rng, 20)
    c = tg.random_dense(rng, 30, 20)
    y = vf.dense_kron_solve(a, b, c) * (1 + 1e-9)
    ref = po.relative_residual(a, b, c, y, 1.0)
    got = vf.relative_residual(a, b, c, y, 0)
    assert abs(got - ref) <= 1e-6 * ref
    # scale invariance: Y * 2^-700 with alpha = 2^-700 gives the same residual
    got2 = vf.relative_residual(a, b, c, y * 2.0 ** -700, -700)
    assert abs(got2 - ref) <= 1e-6 * ref
