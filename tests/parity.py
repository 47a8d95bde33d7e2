"""Per-tile and elementwise parity of Y/alpha between two solutions (test infrastructure).

The norm-wise bar of tests/support/oracles.cpp:75-81 (rel_inf_diff) is dominated by the largest
rows; on the BASELINE twins Y spans up to ~300 decades, so it cannot see a wrong small tile. The
report below adds, on the same pair of solutions:
* per tile (the solver's internal <= 128 partition): ||G_t - R_t||_inf / ||R_t||_inf, every tile
  normalized by its own norm;
* elementwise: |g - r| / |r| over the nonzero reference entries -- the fraction above a
  threshold, the maximum and a decade histogram -- plus the count of entries where exactly one
  side is zero;
* alpha: |alpha_exp_gpu - log2(alpha_ref)| in binades.
G is Y_gpu / 2^alpha_exp expressed in the reference's frame (multiplied by alpha_ref with an
exact power-of-two shift), so nothing overflows even when Y / alpha does.
"""
import math

import numpy as np

HIST_EDGES = [0.0, 1e-16, 1e-15, 1e-14, 1e-13, 1e-12, 1e-11, 1e-10, 1e-9, 1e-8, np.inf]


def in_ref_frame(y_gpu, alpha_exp_gpu, alpha_ref, alpha_exp_ref=None):
    """Y_gpu * alpha_ref / 2^alpha_exp_gpu (the GPU solution in the reference's alpha frame).
    alpha_exp_ref: use 2^alpha_exp_ref instead of alpha_ref (another exponent-form solution)."""
    if alpha_exp_ref is not None:
        mant, ex = 1.0, alpha_exp_ref
    else:
        mant, ex = math.frexp(alpha_ref)
    with np.errstate(all="ignore"):
        return np.ldexp(y_gpu * mant, ex - alpha_exp_gpu)


def report(got, want, rcuts, ccuts, thr=1e-10):
    """Parity of `got` against `want` (same frame). rcuts / ccuts: tile boundaries."""
    got = np.asarray(got)
    want = np.asarray(want)
    M, N = len(rcuts) - 1, len(ccuts) - 1
    worst, worst_t = 0.0, (0, 0)
    tiles_above = 0
    for i in range(M):
        for j in range(N):
            g = got[rcuts[i]:rcuts[i + 1], ccuts[j]:ccuts[j + 1]]
            w = want[rcuts[i]:rcuts[i + 1], ccuts[j]:ccuts[j + 1]]
            d = np.abs(g - w).sum(axis=1).max()
            nw = np.abs(w).sum(axis=1).max()
            e = d / nw if nw > 0 else d
            if not np.isfinite(e):
                e = np.inf
            if e > worst:
                worst, worst_t = e, (i, j)
            tiles_above += e > thr
    nz = want != 0
    with np.errstate(all="ignore"):
        rel = np.abs(got[nz] - want[nz]) / np.abs(want[nz])
    rel = np.where(np.isfinite(rel), rel, np.inf)
    zero_mismatch = int(np.count_nonzero((want == 0) != (got == 0)))
    hist = np.histogram(np.minimum(rel, 1e300), bins=HIST_EDGES)[0].tolist() if rel.size else []
    rd = np.abs(got - want).sum(axis=1).max() if got.size else 0.0
    rw = np.abs(want).sum(axis=1).max() if want.size else 0.0
    return dict(
        normwise=float(rd / rw if rw else rd),
        tile_max=float(worst), tile_worst=[int(worst_t[0]), int(worst_t[1])],
        tiles=M * N, tiles_above=int(tiles_above),
        elem_n=int(rel.size), elem_above=int(np.count_nonzero(rel > thr)),
        elem_frac_above=float(np.count_nonzero(rel > thr) / max(1, rel.size)),
        elem_max=float(rel.max()) if rel.size else 0.0,
        zero_mismatch=zero_mismatch, hist_edges=[float(x) for x in HIST_EDGES], hist=hist,
        thr=thr)


def alpha_binades(alpha_exp_gpu, alpha_ref):
    return abs(alpha_exp_gpu - math.log2(alpha_ref)) if alpha_ref > 0 else float("inf")
