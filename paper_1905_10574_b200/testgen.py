"""System generators of the reference CLI and verification suites, restated bit-exactly.

* include/rsylv/testgen.hpp / src/testgen.cpp:9-61 — mixed_pattern, ones_pattern,
  generate_quasi_triangular (strict upper part 1, diagonal blocks mu / [[mu, mu], [-mu, mu]]),
  generate_rhs (all ones).
* src/verify.cpp:16-56 — random_quasi_triangular / random_dense driven by std::mt19937_64 and
  the libstdc++ distributions (uniform_real_distribution = generate_canonical<double, 53> * (b-a)
  + a with one 64-bit draw; bernoulli_distribution = generate_canonical < p). MT19937_64 is the
  standard engine (w=64, n=312, m=156, r=31); the C++ standard's known answer (10000th output of
  the default-seeded engine = 9981545732273789042) and the reference's own generators
  (oracle/_ref, tests/test_testgen.py) pin it.

Matrices are returned column-major (Fortran order) float64 with one block code per index
(1 = 1x1 block, 2 = start of a 2x2 block, 0 = its second index), the C-ABI convention.
"""
from __future__ import annotations

import numpy as np

_MASK = (1 << 64) - 1


class MT19937_64:
    """std::mt19937_64 (seed_seq-free integer seeding)."""

    def __init__(self, seed: int = 5489):
        mt = [0] * 312
        mt[0] = seed & _MASK
        for i in range(1, 312):
            mt[i] = (6364136223846793005 * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i) & _MASK
        self._mt, self._i = mt, 312

    def _twist(self):
        mt = self._mt
        for i in range(312):
            x = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % 312] & 0x7FFFFFFF)
            xa = x >> 1
            if x & 1:
                xa ^= 0xB5026F5AA96619E9
            mt[i] = mt[(i + 156) % 312] ^ xa
        self._i = 0

    def __call__(self) -> int:
        if self._i >= 312:
            self._twist()
        y = self._mt[self._i]
        self._i += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & _MASK


def canonical(rng: MT19937_64) -> float:
    """libstdc++ generate_canonical<double, 53> on a 64-bit engine: one draw, (double)u / 2^64,
    clamped below 1."""
    r = float(rng()) / 18446744073709551616.0
    return r if r < 1.0 else float(np.nextafter(1.0, 0.0))


def uniform(rng: MT19937_64, a: float, b: float) -> float:
    """std::uniform_real_distribution<double>(a, b)."""
    return canonical(rng) * (b - a) + a


def bernoulli(rng: MT19937_64, p: float) -> bool:
    """std::bernoulli_distribution(p)."""
    return canonical(rng) < p


def mixed_pattern(n: int) -> list[int]:
    """testgen.cpp:9-20: 1, 2, 1, 2, ... (a trailing 2 that does not fit becomes 1)."""
    p, pos, nxt = [], 0, 1
    while pos < n:
        s = nxt if pos + nxt <= n else 1
        p.append(s)
        pos += s
        nxt = 2 if nxt == 1 else 1
    return p


def ones_pattern(n: int) -> list[int]:
    """testgen.cpp:22-24."""
    return [1] * n


def _codes(pattern) -> np.ndarray:
    codes, pos = [], 0
    for s in pattern:
        codes += [2, 0] if s == 2 else [1]
        pos += s
    return np.array(codes, dtype=np.uint8)


def generate_quasi_triangular(n: int, mu: float, pattern) -> tuple[np.ndarray, np.ndarray]:
    """testgen.cpp:26-55: strict upper triangle 1, diagonal blocks mu (1x1) or
    [[mu, mu], [-mu, mu]] (2x2). Raises ValueError like the reference's invalid_argument."""
    if not mu > 0.0:
        raise ValueError("generate_quasi_triangular: mu must be positive")
    if any(s not in (1, 2) for s in pattern):
        raise ValueError("generate_quasi_triangular: block sizes must be 1 or 2")
    if sum(pattern) != n:
        raise ValueError("generate_quasi_triangular: block sizes must sum to n")
    m = np.triu(np.ones((n, n)), 1)
    pos = 0
    for s in pattern:
        m[pos, pos] = mu
        if s == 2:
            m[pos, pos + 1] = mu
            m[pos + 1, pos] = -mu
            m[pos + 1, pos + 1] = mu
        pos += s
    return np.asfortranarray(m), _codes(pattern)


def generate_rhs(m: int, n: int) -> np.ndarray:
    """testgen.cpp:57-61."""
    if m < 1 or n < 1:
        raise ValueError("generate_rhs: dimensions must be >= 1")
    return np.ones((m, n), order="F")


def random_quasi_triangular(rng: MT19937_64, n: int) -> tuple[np.ndarray, np.ndarray]:
    """verify.cpp:16-46: 2x2 block with probability 0.4 at each start (eigenvalue real parts and
    imaginary parts in [0.5, 1.5)), strict upper entries U(-1, 1) column by column, skipping the
    in-block (i, i+1) entry of each 2x2 block."""
    m = np.zeros((n, n))
    codes = np.zeros(n, dtype=np.uint8)
    pos = 0
    while pos < n:
        if pos + 1 < n and bernoulli(rng, 0.4):
            re = uniform(rng, 0.5, 1.5)
            im = uniform(rng, 0.5, 1.5)
            m[pos, pos] = re
            m[pos, pos + 1] = im
            m[pos + 1, pos] = -im
            m[pos + 1, pos + 1] = re
            codes[pos] = 2
            pos += 2
        else:
            m[pos, pos] = uniform(rng, 0.5, 1.5)
            codes[pos] = 1
            pos += 1
    for j in range(n):
        for i in range(j):
            if i + 1 != j or m[j, i] == 0.0:
                m[i, j] = uniform(rng, -1.0, 1.0)
    return np.asfortranarray(m), codes


def random_dense(rng: MT19937_64, m: int, n: int) -> np.ndarray:
    """verify.cpp:48-54 (column by column)."""
    out = np.zeros((m, n), order="F")
    for j in range(n):
        for i in range(m):
            out[i, j] = uniform(rng, -1.0, 1.0)
    return out
