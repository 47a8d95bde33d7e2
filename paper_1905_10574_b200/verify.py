"""Self-verification suites of the reference CLI on the GPU solvers.

Mirrors include/rsylv/verify.hpp + src/verify.cpp:108-199 (`rsylv-bench verify`):
1. oracle equivalence — the three GPU solvers (solve_nonrobust, solve_robust_scalar,
   solve_tiled_robust, Ω = DBL_MAX) against an independent dense Kronecker-system solve on the
   reference's own random systems (same std::mt19937_64 stream, testgen.py), norm-wise
   ≤ tolerance, and α = 1 on these benign systems;
2. generator residuals of the deterministic generator (μ = ν = n, mixed blocks, C = ones);
3. bounded tiles under an artificially small Ω (growth systems μ = 1e-3, ν = 1e-2): every
   tile at rest ≤ Ω (TileProbe), α < 1, scaled residual ≤ 1e-12.
`inject_bug` flips the sign of one reference entry (negative control). The dense Kronecker
solve (numpy/LAPACK LU with partial pivoting) is the suite's checker, never a solver path.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

from . import api
from . import testgen as tg
from .records import format_double


@dataclasses.dataclass
class VerifyOptions:
    """verify.hpp:16-28 (same defaults)."""
    sizes: list = dataclasses.field(default_factory=lambda: [6, 10, 16, 24, 32, 40])
    systems_per_size: int = 3
    seed: int = 42
    omegas: list = dataclasses.field(default_factory=lambda: [1e4])
    mu: float = 1e-3
    nu: float = 1e-2
    growth_size: int = 100
    tile_size: int = 8
    oracle_tol: float = 1e-11
    inject_bug: bool = False


@dataclasses.dataclass
class VerifyReport:
    text: str = ""
    ok: bool = False
    min_local_alpha: float = 1.0


def dense_kron_solve(a: np.ndarray, b: np.ndarray, c: np.ndarray) -> np.ndarray:
    """verify.cpp:58-95: the mn x mn system (I (x) A + B^T (x) I) vec(Y) = vec(C), solved by LU
    with partial pivoting. Never calls a solver kernel."""
    m, n = c.shape
    k = np.kron(np.eye(n), a) + np.kron(b.T, np.eye(m))
    y = np.linalg.solve(k, np.asarray(c, dtype=np.float64).reshape(-1, order="F"))
    return y.reshape((m, n), order="F")


def rel_inf_diff(got: np.ndarray, want: np.ndarray) -> float:
    """verify.cpp:99-106: ||got - want||_inf / ||want||_inf (absolute when want is zero)."""
    ref = np.abs(want).sum(axis=1).max() if want.size else 0.0
    d = np.abs(got - want).sum(axis=1).max() if want.size else 0.0
    return float(d if ref == 0.0 else d / ref)


def relative_residual(a, b, c, y, alpha_exp: int = 0, device: int = 0) -> float:
    """testgen.cpp:63-79, ||α C − A Y − Y B||_F / ((||A||_F + ||B||_F) ||Y||_F + ||α C||_F) with
    α = 2^alpha_exp, evaluated on the GPU (cuBLAS DGEMM via torch) after scaling Y by a power
    of two to max |Y| <= 1, so it stays finite where the reference's plain evaluation overflows
    (above ~1e154 it returns NaN); the ratio is scale-invariant, so it equals the reference's
    value wherever that one is finite (up to rounding)."""
    import torch
    dev = torch.device("cuda", device)
    t = lambda x: torch.as_tensor(np.asarray(x, dtype=np.float64), device=dev)  # noqa: E731
    A, B, C, Y = t(a), t(b), t(c), t(y)
    def p2(x, e):  # x * 2^e with exact power-of-two factors (at most two multiplies)
        if e < -2200:
            return torch.zeros_like(x)
        h = e // 2
        return x * math.ldexp(1.0, h) * math.ldexp(1.0, e - h)

    ymax = float(Y.abs().max().item()) if Y.numel() else 0.0
    k = math.frexp(ymax)[1] if ymax > 0 and math.isfinite(ymax) else 0
    Ys = p2(Y, -k)
    Cs = p2(C, alpha_exp - k)  # alpha * 2^-k * C
    R = Cs - A @ Ys - Ys @ B
    fro = lambda x: float(torch.linalg.vector_norm(x).item())  # noqa: E731
    den = (fro(A) + fro(B)) * fro(Ys) + fro(Cs)
    if den == 0.0:
        raise ZeroDivisionError("relative_residual: undefined (all norms zero)")
    return fro(R) / den


def run_verification(opt: VerifyOptions, device: int = 0) -> VerifyReport:
    """verify.cpp:108-199, with the GPU solvers; report text in the reference's format."""
    out = []
    ok = True

    def check(cond: bool, what: str):
        nonlocal ok
        if not cond:
            ok = False
            out.append(f"  FAILED: {what}")

    wide = lambda: api.OverflowConfig(omega=np.finfo(np.float64).max)  # noqa: E731

    out.append(f"oracle equivalence (tolerance {format_double(opt.oracle_tol)})")
    rng = tg.MT19937_64(opt.seed)
    for n in opt.sizes:
        for _ in range(opt.systems_per_size):
            nb = max(3, n // 2)
            a, ac = tg.random_quasi_triangular(rng, n)
            b, bc = tg.random_quasi_triangular(rng, nb)
            c = tg.random_dense(rng, n, nb)
            ref = dense_kron_solve(a, b, c)
            if opt.inject_bug:
                ref[0, 0] = -ref[0, 0]
            qa, qb = api.QuasiTriangular.from_codes(a, ac), api.QuasiTriangular.from_codes(b, bc)
            y0 = api.solve_nonrobust(qa, qb, c, device=device)
            y1 = api.solve_robust_scalar(qa, qb, c, wide(), device=device)
            y2 = api.solve_tiled_robust(qa, qb, c, opt.tile_size, wide(), device=device)
            d0, d1, d2 = rel_inf_diff(y0, ref), rel_inf_diff(y1.y, ref), rel_inf_diff(y2.y, ref)
            out.append(f"  m={n} n={nb} diff nonrobust={format_double(d0)} "
                       f"robust-scalar={format_double(d1)} robust-tiled={format_double(d2)}")
            check(d0 <= opt.oracle_tol, "nonrobust differs from the dense reference")
            check(d1 <= opt.oracle_tol, "robust-scalar differs from the dense reference")
            check(d2 <= opt.oracle_tol, "robust-tiled differs from the dense reference")
            check(y1.alpha == 1.0 and y2.alpha == 1.0, "robust solver scaled a benign system")

    out.append("generator residuals")
    for n in opt.sizes:
        a, ac = tg.generate_quasi_triangular(n, float(n), tg.mixed_pattern(n))
        b, bc = tg.generate_quasi_triangular(n, float(n), tg.mixed_pattern(n))
        c = tg.generate_rhs(n, n)
        r = api.solve_tiled_robust(api.QuasiTriangular.from_codes(a, ac),
                                   api.QuasiTriangular.from_codes(b, bc), c, opt.tile_size,
                                   wide(), device=device)
        res = relative_residual(a, b, c, r.y, r.alpha_exp, device)
        out.append(f"  n={n} residual={format_double(res)}")
        check(res <= opt.oracle_tol, "generator residual out of tolerance")

    min_alpha = 1.0
    out.append(f"bounded tiles (mu={format_double(opt.mu)} nu={format_double(opt.nu)})")
    for omega in opt.omegas:
        cfg = api.OverflowConfig(omega=omega)
        n = opt.growth_size
        a, ac = tg.generate_quasi_triangular(n, opt.mu, tg.mixed_pattern(n))
        b, bc = tg.generate_quasi_triangular(n, opt.nu, tg.mixed_pattern(n))
        c = tg.generate_rhs(n, n)
        state = {"bounded": True, "min": 1.0}

        def probe(k, l, al, norm, state=state, omega=omega):
            if not norm <= omega:
                state["bounded"] = False
            state["min"] = min(state["min"], al)

        r = api.solve_tiled_robust(api.QuasiTriangular.from_codes(a, ac),
                                   api.QuasiTriangular.from_codes(b, bc), c,
                                   max(opt.tile_size, 2), cfg, probe=probe, device=device)
        res = relative_residual(a, b, c, r.y, r.alpha_exp, device)
        alpha = math.ldexp(1.0, r.alpha_exp)
        min_alpha = min(min_alpha, state["min"], alpha)
        out.append(f"  omega={format_double(omega)} n={n} alpha={format_double(alpha)} "
                   f"min-local-alpha={format_double(state['min'])} residual={format_double(res)}")
        check(state["bounded"], "a tile norm exceeded omega at rest")
        check(alpha < 1.0, "growth system did not trigger scaling")
        check(res <= 1e-12, "scaled residual out of tolerance")

    out.append("verification passed" if ok else "verification FAILED")
    return VerifyReport("\n".join(out) + "\n", ok, min_alpha)
