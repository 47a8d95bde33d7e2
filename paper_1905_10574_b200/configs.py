"""BASELINE.json workloads and their seeded synthetic generators.

The reference has no dataset: the paper's matrices are synthetic and
BASELINE.json states the distributions. Two bit-identical generators exist for the uniform
distributions: a counter-based (splitmix64) one on the device (`rsylv_b200_generate_*` in the
extension) and the numpy restatement below (host), so the CPU reference and the GPU see the same
matrices. (The N(0,1) right-hand side of config 4 uses device libm and is not bit-identical on
the host.)

Interpretations (stated in DESIGN.md):
* "x% 2x2 blocks": each block start is a 2x2 block with probability x (Bernoulli per block start,
  the pattern of verify.cpp:19,25).
* 2x2 block [[a, b], [-c, a]]: a from the config's diagonal distribution, b, c ~ U(0.1, 1) (configs
  4/5 give no form; config 2's is reused).
* config 3 gives no tile size: 256.
* config 5's "1% of tiles scaled by 1e250": max(1, round(0.01 * #tiles)) tiles of the nominal
  t x t grid, chosen by a seeded permutation.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass(frozen=True)
class Config:
    name: str
    m: int
    n: int
    tile: int
    p2x2: float
    a_up: tuple
    a_diag: tuple
    b_up: tuple
    b_diag: tuple
    off: tuple = (0.1, 1.0)
    c_dist: int = 0  # 0 uniform(lo, hi), 1 normal * hi + lo
    c_range: tuple = (-1.0, 1.0)
    hot_frac: float = 0.0
    hot_factor: float = 1.0
    seed: int = 12345
    note: str = ""

    def flops(self) -> float:
        return float(self.m) * self.n * (self.m + self.n)

    def alg_bytes(self) -> float:
        """read the upper A and B, read C, write Y (8-byte doubles)."""
        return 8.0 * (self.m * self.m / 2 + self.n * self.n / 2 + 2.0 * self.m * self.n)

    def scaled(self, m: int, n: int | None = None, tile: int | None = None) -> "Config":
        d = dict(self.__dict__)
        d.update(m=m, n=n if n is not None else m, tile=tile or self.tile,
                 name=f"{self.name}@{m}x{n if n is not None else m}")
        return Config(**d)


CONFIGS = {
    "c1": Config("c1", 2000, 2000, 128, 0.0, (-1, 1), (1, 2), (-1, 1), (1, 2),
                 note="m=n=2000, 1x1 only, well conditioned (alpha=1)"),
    "c2": Config("c2", 8000, 8000, 256, 0.5, (-1, 1), (0.5, 2), (-1, 1), (0.5, 2),
                 note="m=n=8000, 50% 2x2 complex pairs"),
    "c3": Config("c3", 8000, 8000, 256, 0.0, (-1e3, 1e3), (1e-8, 2e-8), (-1, 1), (1e-8, 2e-8),
                 c_range=(-1e300, 1e300), note="overflow-provoking, tile 256 assumed"),
    "c4": Config("c4", 32000, 4000, 256, 0.3, (-1, 1), (1, 2), (-1, 1), (1, 2), c_dist=1,
                 c_range=(0.0, 1.0), note="rectangular, 30% 2x2, C ~ N(0,1)"),
    "c5": Config("c5", 40000, 40000, 512, 0.5, (-1, 1), (0.5, 2), (-1, 1), (0.5, 2),
                 hot_frac=0.01, hot_factor=1e250,
                 note="m=n=40000, 50% 2x2, 1% of tiles x 1e250"),
}

# ---------------------------------------------------------------- counter-based RNG (numpy)
_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _splitmix64(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        x = (x + np.uint64(0x9E3779B97F4A7C15))
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return x ^ (x >> np.uint64(31))


def u01(seed: int, stream: int, idx: np.ndarray) -> np.ndarray:
    """Same as the device u01(seed, stream, idx) in kernels.cu (exactly)."""
    idx = np.asarray(idx, dtype=np.uint64)
    with np.errstate(over="ignore"):
        inner = _splitmix64(np.uint64(stream) * np.uint64(0x632BE59BD9B4E019) + idx)
    h = _splitmix64(np.uint64(seed) ^ inner)
    return (h >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def uab(u, lo, hi):
    return lo + u * (hi - lo)


def block_codes(n: int, p2x2: float, seed: int, stream: int = 8) -> np.ndarray:
    """Bernoulli(p2x2) 2x2 block at each block start (1 = 1x1, 2 = 2x2 start, 0 = 2nd index)."""
    codes = np.zeros(n, dtype=np.uint8)
    if p2x2 <= 0:
        codes[:] = 1
        return codes
    u = u01(seed, stream, np.arange(n, dtype=np.uint64))
    pos = 0
    while pos < n:
        if pos + 1 < n and u[pos] < p2x2:
            codes[pos], codes[pos + 1] = 2, 0
            pos += 2
        else:
            codes[pos] = 1
            pos += 1
    return codes


def host_quasi_triangular(n, codes, seed, up, diag, off):
    """numpy restatement of kernels.cu k_gen_qt (bit-identical)."""
    j = np.arange(n, dtype=np.uint64)[None, :]
    i = np.arange(n, dtype=np.uint64)[:, None]
    a = np.zeros((n, n), order="F")
    upper = uab(u01(seed, 1, j * np.uint64(n) + i), up[0], up[1])
    iu = np.triu_indices(n, 1)
    a[iu] = upper[iu]
    dvals = uab(u01(seed, 2, np.arange(n, dtype=np.uint64)), diag[0], diag[1])
    for c in range(n):
        if codes[c] == 0:  # second index of a 2x2 block starting at c-1
            a[c, c] = dvals[c - 1]
            a[c - 1, c] = uab(u01(seed, 3, np.array([c - 1], dtype=np.uint64))[0], off[0], off[1])
        else:
            a[c, c] = dvals[c]
        if codes[c] == 2:
            a[c + 1, c] = -uab(u01(seed, 4, np.array([c], dtype=np.uint64))[0], off[0], off[1])
    return a


def hot_tiles(cfg: Config) -> np.ndarray:
    if cfg.hot_frac <= 0:
        return np.zeros((0, 2), dtype=np.int32)
    mt = -(-cfg.m // cfg.tile)
    nt = -(-cfg.n // cfg.tile)
    count = max(1, int(round(cfg.hot_frac * mt * nt)))
    perm = np.random.default_rng(cfg.seed).permutation(mt * nt)[:count]
    return np.stack([perm // nt, perm % nt], axis=1).astype(np.int32)


def host_rhs(cfg: Config) -> np.ndarray:
    m, n = cfg.m, cfg.n
    j = np.arange(n, dtype=np.uint64)[None, :]
    i = np.arange(m, dtype=np.uint64)[:, None]
    idx = j * np.uint64(m) + i
    if cfg.c_dist == 0:
        c = uab(u01(cfg.seed, 5, idx), cfg.c_range[0], cfg.c_range[1])
    else:
        u1 = np.maximum(u01(cfg.seed, 6, idx), 2.0 ** -60)
        u2 = u01(cfg.seed, 7, idx)
        c = np.sqrt(-2.0 * np.log(u1)) * np.cos(2 * np.pi * u2) * cfg.c_range[1] + cfg.c_range[0]
    for (ti, tj) in hot_tiles(cfg):
        c[ti * cfg.tile:(ti + 1) * cfg.tile, tj * cfg.tile:(tj + 1) * cfg.tile] *= cfg.hot_factor
    return np.asfortranarray(c)


def host_system(cfg: Config):
    """(A, A codes, B, B codes, C) on the host, bit-identical to the device generator for the
    uniform distributions."""
    ac = block_codes(cfg.m, cfg.p2x2, cfg.seed, stream=8)
    bc = block_codes(cfg.n, cfg.p2x2, cfg.seed + 1, stream=9)
    a = host_quasi_triangular(cfg.m, ac, cfg.seed, cfg.a_up, cfg.a_diag, cfg.off)
    b = host_quasi_triangular(cfg.n, bc, cfg.seed + 1, cfg.b_up, cfg.b_diag, cfg.off)
    return a, ac, b, bc, host_rhs(cfg)


def device_system(cfg: Config, torch, device="cuda", stream=None):
    """Same system generated directly in HBM (column-major torch tensors)."""
    import ctypes as C
    from . import _native as nat
    ac = block_codes(cfg.m, cfg.p2x2, cfg.seed, stream=8)
    bc = block_codes(cfg.n, cfg.p2x2, cfg.seed + 1, stream=9)
    A = torch.empty((cfg.m, cfg.m), dtype=torch.float64, device=device).T
    B = torch.empty((cfg.n, cfg.n), dtype=torch.float64, device=device).T
    Cm = torch.empty((cfg.n, cfg.m), dtype=torch.float64, device=device).T
    L = nat.lib()
    up = lambda x: x.ctypes.data_as(C.POINTER(C.c_ubyte))  # noqa: E731
    st = stream or torch.cuda.current_stream().cuda_stream
    r = L.rsylv_b200_generate_quasi_triangular(cfg.m, C.c_void_p(A.data_ptr()), cfg.m, up(ac),
                                               cfg.seed, cfg.a_up[0], cfg.a_up[1], cfg.a_diag[0],
                                               cfg.a_diag[1], cfg.off[0], cfg.off[1],
                                               C.c_void_p(st))
    r |= L.rsylv_b200_generate_quasi_triangular(cfg.n, C.c_void_p(B.data_ptr()), cfg.n, up(bc),
                                                cfg.seed + 1, cfg.b_up[0], cfg.b_up[1],
                                                cfg.b_diag[0], cfg.b_diag[1], cfg.off[0],
                                                cfg.off[1], C.c_void_p(st))
    hot = np.ascontiguousarray(hot_tiles(cfg), dtype=np.int32)
    r |= L.rsylv_b200_generate_rhs(cfg.m, cfg.n, C.c_void_p(Cm.data_ptr()), cfg.m, cfg.seed,
                                   cfg.c_dist, cfg.c_range[0], cfg.c_range[1],
                                   hot.ctypes.data_as(C.POINTER(C.c_int32)), len(hot), cfg.tile,
                                   cfg.hot_factor, C.c_void_p(st))
    if r:
        raise RuntimeError("device generator failed")
    return A, ac, B, bc, Cm
