"""The Bartels–Stewart wrapper around the triangular solve.

Solves the general real Sylvester equation A X + X B = α C (A m×m, B n×n, no structure) by
    A = U Ã Uᵀ, B = V B̃ Vᵀ          real Schur forms
    C̃ = Uᵀ C V                      two GEMMs on the GPU (this package's FP64 DMMA GEMM,
                                    rsylv_b200_dgemm)
    Ã Y + Y B̃ = α C̃                 the robust tiled solve (this package's CUDA engine)
    X = U Y Vᵀ                      two GEMMs on the GPU (rsylv_b200_dgemm)
The reference solves only the triangular inner problem; this is the wrapper a
user of the full equation needs. The Schur factorizations run on the host (LAPACK dgees via
scipy): there is no GPU real-Schur routine in this image, and they are preprocessing outside the
hot path. With orthogonal U, V the robustness carries over: ||X||_2 = ||Y||_2 <= sqrt(m n) Ω.
"""
from __future__ import annotations

import math
from typing import Optional

import numpy as np

from . import api


def schur_real(a: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """Real Schur form a = u t uᵀ with t upper quasi-triangular (standardized 2x2 blocks for
    complex conjugate pairs). Host LAPACK (scipy.linalg.schur, dgees)."""
    import scipy.linalg
    t, u = scipy.linalg.schur(np.asarray(a, dtype=np.float64), output="real")
    return t, u


def solve_sylvester(a, b, c, tile_size: int = 128, cfg: Optional[api.OverflowConfig] = None,
                    device: int = 0, schur_a=None, schur_b=None):
    """Returns (X, alpha_exp) with A X + X B = 2^alpha_exp C (alpha_exp <= 0; 0 when no scaling
    was needed). `schur_a` / `schur_b` may pass precomputed (t, u) factorizations to reuse them
    across right-hand sides. Raises like solve_tiled_robust (ValueError, SingularEquationError
    when A and -B share an eigenvalue to working precision)."""
    import torch
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    c = np.asarray(c, dtype=np.float64)
    m, n = c.shape
    if a.shape != (m, m) or b.shape != (n, n):
        raise ValueError("solve_sylvester: A, B, C do not conform")
    ta, ua = schur_a if schur_a is not None else schur_real(a)
    tb, ub = schur_b if schur_b is not None else schur_real(b)
    # exact zeros below the quasi-triangle (dgees leaves rounding noise of order eps there in
    # no case, but make the block structure explicit for the solver)
    ta = np.triu(ta, -1)
    tb = np.triu(tb, -1)
    qa, qb = api.QuasiTriangular(ta), api.QuasiTriangular(tb)
    dev = torch.device("cuda", device)
    # every device matrix is column-major (the C-ABI layout)
    cm = lambda x: torch.as_tensor(np.asfortranarray(x), device=dev).T.contiguous().T  # noqa: E731
    empty = lambda r, k: torch.empty((k, r), dtype=torch.float64, device=dev).T  # noqa: E731
    U, V, Cd = cm(ua), cm(ub), cm(c)
    T = empty(m, n)
    api.dgemm(U, Cd, T, ta=True, device=device)            # T = Uᵀ C
    C_d = empty(m, n)
    api.dgemm(T, V, C_d, device=device)                    # C̃ = T V
    A_d, B_d = cm(qa.matrix()), cm(qb.matrix())
    Y_d = empty(m, n)
    st, res = api.solve_tiled_robust_device(A_d, qa.codes, B_d, qb.codes, C_d, Y_d, tile_size,
                                            cfg, device=device, raise_underflow=False)
    api.dgemm(U, Y_d, T, device=device)                    # T = U Y
    X_d = empty(m, n)
    api.dgemm(T, V, X_d, tb=True, device=device)           # X = T Vᵀ
    torch.cuda.synchronize(dev)
    X = X_d.cpu().numpy()
    return X, int(res.alpha_exp)


def residual(a, b, c, x, alpha_exp: int = 0) -> float:
    """||A X + X B − 2^alpha_exp C||_F / ((||A||_F + ||B||_F) ||X||_F + ||2^alpha_exp C||_F)."""
    al = math.ldexp(1.0, alpha_exp)
    r = a @ x + x @ b - al * c
    den = (np.linalg.norm(a) + np.linalg.norm(b)) * np.linalg.norm(x) + al * np.linalg.norm(c)
    return float(np.linalg.norm(r) / den)
