"""TEST INFRASTRUCTURE ONLY: unbounded-exponent oracle for overflow-provoking systems.

The reference cannot return a solution once the required global scale drops below DBL_MIN
(it throws ScaleUnderflowError, overflow.cpp:42-46) — e.g. BASELINE config 3's distributions
for m = n >= 24. To still pin the GPU's exponent-form result (Y * 2^-alpha_exp), this module
restates the reference's non-robust block back substitution (scalar_solve.cpp:13-36:
column blocks left to right, row blocks bottom-up, 1x1/2x2 Kronecker solves) in Python
``decimal`` arithmetic with 40 significant digits and an exponent range of +-10^8, where no
intermediate can overflow. Cost is O(m n (m + n)) Decimal operations: small cases only.
"""
from __future__ import annotations

import decimal
from decimal import Decimal

import numpy as np

CTX = decimal.Context(prec=40, Emax=100_000_000, Emin=-100_000_000)


def _blocks(codes, n):
    out, i = [], 0
    while i < n:
        s = 2 if (codes is not None and codes[i] == 2) else 1
        out.append((i, s))
        i += s
    return out


def _solve_small(Ak, Bl, R):
    """Solves Ak Z + Z Bl = R for <= 2x2 blocks by Gaussian elimination (partial pivoting is
    enough at 40 digits)."""
    ma, nb = len(Ak), len(Bl)
    nk = ma * nb
    K = [[Decimal(0)] * nk for _ in range(nk)]
    v = [Decimal(0)] * nk
    for j in range(nb):
        for i in range(ma):
            row = j * ma + i
            v[row] = R[i][j]
            for p in range(ma):
                K[row][j * ma + p] = CTX.add(K[row][j * ma + p], Ak[i][p])
            for l in range(nb):
                K[row][l * ma + i] = CTX.add(K[row][l * ma + i], Bl[l][j])
    for s in range(nk):
        piv = max(range(s, nk), key=lambda r: abs(K[r][s]))
        K[s], K[piv] = K[piv], K[s]
        v[s], v[piv] = v[piv], v[s]
        if K[s][s] == 0:
            raise ZeroDivisionError("singular block")
        for r in range(s + 1, nk):
            f = CTX.divide(K[r][s], K[s][s])
            for c in range(s, nk):
                K[r][c] = CTX.subtract(K[r][c], CTX.multiply(f, K[s][c]))
            v[r] = CTX.subtract(v[r], CTX.multiply(f, v[s]))
    for s in range(nk - 1, -1, -1):
        acc = v[s]
        for c in range(s + 1, nk):
            acc = CTX.subtract(acc, CTX.multiply(K[s][c], v[c]))
        v[s] = CTX.divide(acc, K[s][s])
    return [[v[j * ma + i] for j in range(nb)] for i in range(ma)]


def solve(a, acodes, b, bcodes, c):
    """Exact-range solution of A Y + Y B = C as a nested list of Decimals (row-major)."""
    m, n = c.shape
    D = lambda x: Decimal(float(x))  # noqa: E731  (exact conversion of a double)
    A = [[D(a[i, j]) for j in range(m)] for i in range(m)]
    B = [[D(b[i, j]) for j in range(n)] for i in range(n)]
    Y = [[D(c[i, j]) for j in range(n)] for i in range(m)]
    ab, bb = _blocks(acodes, m), _blocks(bcodes, n)
    for (c0, cs) in bb:
        for (r0, rs) in reversed(ab):
            R = [[Y[r0 + i][c0 + j] for j in range(cs)] for i in range(rs)]
            for i in range(rs):
                for j in range(cs):
                    acc = R[i][j]
                    for p in range(r0 + rs, m):
                        if A[r0 + i][p] != 0:
                            acc = CTX.subtract(acc, CTX.multiply(A[r0 + i][p], Y[p][c0 + j]))
                    for q in range(0, c0):
                        if B[q][c0 + j] != 0:
                            acc = CTX.subtract(acc, CTX.multiply(Y[r0 + i][q], B[q][c0 + j]))
                    R[i][j] = acc
            Z = _solve_small([row[r0:r0 + rs] for row in A[r0:r0 + rs]],
                             [row[c0:c0 + cs] for row in B[c0:c0 + cs]], R)
            for i in range(rs):
                for j in range(cs):
                    Y[r0 + i][c0 + j] = Z[i][j]
    return Y


def rel_inf_diff_exp(y_gpu: np.ndarray, alpha_exp: int, Y) -> float:
    """||Y_gpu * 2^-alpha_exp - Y||_inf / ||Y||_inf computed in Decimal (oracles.cpp:75-81
    norm, exponent-form alpha)."""
    m, n = y_gpu.shape
    two = Decimal(2)
    scale = CTX.power(two, -alpha_exp)
    num = Decimal(0)
    den = Decimal(0)
    for i in range(m):
        sd = Decimal(0)
        sy = Decimal(0)
        for j in range(n):
            g = CTX.multiply(Decimal(float(y_gpu[i, j])), scale)
            sd = CTX.add(sd, abs(CTX.subtract(g, Y[i][j])))
            sy = CTX.add(sy, abs(Y[i][j]))
        num = max(num, sd)
        den = max(den, sy)
    return float(CTX.divide(num, den)) if den != 0 else float(num)


def log10_max_abs(Y) -> float:
    mx = max(abs(v) for row in Y for v in row)
    return float(mx.log10(CTX)) if mx != 0 else float("-inf")
