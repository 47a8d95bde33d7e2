"""tests/parity.py on synthetic pairs (CPU): a wrong small tile that the norm-wise bar misses is
caught per tile and elementwise; frames are exact power-of-two shifts."""
import numpy as np

import parity


def test_small_wrong_tile_is_caught_per_tile():
    rng = np.random.default_rng(0)
    want = rng.standard_normal((300, 260))
    want[:128, :128] *= 1e200  # one huge tile dominates the row sums
    got = want.copy()
    got[200:250, 140:200] *= 1 + 1e-6  # a small tile is wrong by 1e-6
    rep = parity.report(got, want, [0, 128, 256, 300], [0, 128, 256, 260])
    assert rep["normwise"] < 1e-12 < 1e-10 < rep["tile_max"]
    assert rep["tile_worst"] == [1, 1] and rep["tiles_above"] == 1
    assert rep["elem_above"] == 50 * 60 and rep["zero_mismatch"] == 0
    assert sum(rep["hist"]) == rep["elem_n"]


def test_frames_are_exact():
    y = np.array([[1.5, -3.0], [0.25, 2.0 ** -1000]])
    g = parity.in_ref_frame(y * 2.0 ** -7, -7, 1.0)
    assert np.array_equal(g, y)
    assert parity.alpha_binades(-10, 2.0 ** -12) == 2.0


def test_identical_is_clean():
    x = np.random.default_rng(1).standard_normal((50, 40))
    rep = parity.report(x, x, [0, 50], [0, 40])
    assert rep["tile_max"] == rep["normwise"] == rep["elem_max"] == 0.0
