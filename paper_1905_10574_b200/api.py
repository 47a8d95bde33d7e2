"""Python mirror of the reference's public API for the hot path.

Names, argument meaning and error behaviour follow /root/reference/proj/include/rsylv:

* ``QuasiTriangular``           partition.hpp:22-42 (explicit or detected 2x2 blocks, validated)
* ``OverflowConfig``            overflow.hpp:13-34 (omega, small_num, scaling_events counter)
* ``ExecutionMode``             tiled_solve.hpp:16-22 (workers -> GPU count; 0/1 = one GPU)
* ``solve_tiled_robust``        tiled_solve.hpp:36-40
* ``SolveResult``               scalar_solve.hpp:15-18 (+ ``alpha_exp``: alpha as 2^alpha_exp)
* ``SingularEquationError``,    errors.hpp:10-30
  ``ScaleUnderflowError``
* ``std::invalid_argument``  -> ``ValueError``

Everything runs on the CUDA extension; there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Callable, Optional, Sequence

import numpy as np

from . import _native as nat

DBL_MAX = np.finfo(np.float64).max
DBL_MIN = np.finfo(np.float64).tiny
DBL_EPS = np.finfo(np.float64).eps


def default_omega() -> float:
    return DBL_MAX / 2  # overflow.hpp:23-25


def default_small_num() -> float:
    return DBL_MIN / DBL_EPS  # overflow.hpp:27-29


class SingularEquationError(RuntimeError):
    """errors.hpp:10-21: an eigenvalue pair lambda_i(A) + lambda_j(B) is numerically zero."""

    def __init__(self, pivot: float):
        super().__init__(f"singular Sylvester equation: pivot magnitude {pivot!r} below the "
                         "tiny-divisor threshold")
        self.pivot = pivot


class ScaleUnderflowError(RuntimeError):
    """errors.hpp:25-30: the global scale factor falls below the smallest normal double.

    The GPU solve itself never underflows (exponents are int32); ``result`` carries the
    exponent-form solution (alpha = 2**alpha_exp) for callers that can use it."""

    def __init__(self, result: "SolveResult | None" = None):
        super().__init__("scaling factor underflow: accumulated scale fell below the smallest "
                         "normal double")
        self.result = result


@dataclass
class OverflowConfig:
    omega: float = field(default_factory=default_omega)
    small_num: float = field(default_factory=default_small_num)
    scaling_events: int = 0  # bumped by the number of guard activations of each solve


@dataclass
class ExecutionMode:
    workers: int = 0

    @staticmethod
    def sequential() -> "ExecutionMode":
        return ExecutionMode(0)

    @staticmethod
    def parallel(w: int) -> "ExecutionMode":
        return ExecutionMode(w)

    def is_parallel(self) -> bool:
        return self.workers > 0


@dataclass
class SolveResult:
    alpha: float
    y: np.ndarray
    alpha_exp: int = 0
    scaling_events: int = 0
    device_ms: float = 0.0
    max_tile_norm: float = 0.0


class QuasiTriangular:
    """Upper quasi-triangular matrix with its 1x1/2x2 diagonal block list (partition.hpp:22-42).

    ``blocks`` is a list of (start, size); when omitted, 2x2 blocks are detected from exactly
    nonzero subdiagonal entries (partition.cpp:8-23)."""

    def __init__(self, m, blocks: Optional[Sequence[tuple]] = None):
        m = np.asfortranarray(np.asarray(m, dtype=np.float64))
        if m.ndim != 2 or m.shape[0] != m.shape[1]:
            raise ValueError("QuasiTriangular: matrix must be square")
        n = m.shape[0]
        if blocks is None:
            blocks, i = [], 0
            while i < n:
                if i + 1 < n and m[i + 1, i] != 0.0:
                    blocks.append((i, 2))
                    i += 2
                else:
                    blocks.append((i, 1))
                    i += 1
        else:
            pos = 0
            for (s, z) in blocks:
                if s != pos or z not in (1, 2):
                    raise ValueError("QuasiTriangular: block list must cover the diagonal in order")
                pos += z
            if pos != n:
                raise ValueError("QuasiTriangular: block sizes must sum to the dimension")
        self._m = m
        self._blocks = [(int(s), int(z)) for (s, z) in blocks]
        self._validate()
        codes = np.zeros(n, dtype=np.uint8)
        for s, z in self._blocks:
            codes[s] = z
        self.codes = codes

    @classmethod
    def from_codes(cls, m, codes) -> "QuasiTriangular":
        codes = np.asarray(codes, dtype=np.uint8)
        blocks = [(i, int(c)) for i, c in enumerate(codes) if c in (1, 2)]
        return cls(m, blocks)

    def _validate(self):  # partition.cpp:40-54
        m, n = self._m, self._m.shape[0]
        if n > 2 and np.any(np.tril(m, -2) != 0.0):
            raise ValueError("QuasiTriangular: nonzero entry below the first subdiagonal")
        in_block = np.zeros(max(n - 1, 0), dtype=bool)
        for s, z in self._blocks:
            if z == 2:
                in_block[s] = True
        sub = np.diagonal(m, -1) if n > 1 else np.zeros(0)
        if np.any((sub != 0.0) & ~in_block):
            raise ValueError("QuasiTriangular: nonzero subdiagonal outside a declared 2x2 block")

    def dim(self) -> int:
        return self._m.shape[0]

    def matrix(self) -> np.ndarray:
        return self._m

    def view(self) -> np.ndarray:
        return self._m

    def diag_blocks(self):
        return list(self._blocks)


INTERNAL_TILE = 128  # largest internal tile edge (kTileMax in csrc/common.cuh)


def tile_cuts(codes, n: int, tile_size: int) -> list:
    """The B200 partition of an index range (mirror of partition() in csrc/runtime.cpp): cut at
    running multiples of min(tile_size, 128); a cut that would split a 2x2 block moves one index
    EARLIER (the reference moves it later, partition.cpp:74-91). alpha and the TileProbe
    indices refer to these tiles."""
    ts = min(max(2, int(tile_size)), INTERNAL_TILE)
    cuts, pos = [0], 0
    while pos < n:
        nx = pos + ts
        if nx >= n:
            nx = n
        elif codes is not None and codes[nx - 1] == 2:
            nx -= 1
        cuts.append(nx)
        pos = nx
    return cuts


def _status_to_exc(st: int, res: nat.Result, partial: "SolveResult | None" = None):
    if st == nat.RSYLV_INVALID_ARGUMENT:
        return ValueError("solve_tiled_robust: " + nat.REASONS.get(res.invalid_reason, "invalid"))
    if st == nat.RSYLV_SINGULAR:
        return SingularEquationError(res.pivot)
    if st == nat.RSYLV_SCALE_UNDERFLOW:
        return ScaleUnderflowError(partial)
    msg = nat.lib().rsylv_b200_last_error(nat.context()).decode()
    return RuntimeError(f"rsylv-b200: {nat.lib().rsylv_b200_status_string(st).decode()} {msg}")


def _replay_probe(res: nat.Result, buf, probe):
    if probe is None:
        return
    nc = min(res.probe_count, res.probe_cap)
    for t in range(nc):
        e = buf[t]
        probe(int(e.k), int(e.l), float(np.ldexp(1.0, e.scale_exp)) if e.scale_exp >= -1074 else 0.0,
              float(e.norm))


def solve_tiled_robust(a: QuasiTriangular, b: QuasiTriangular, c, tile_size: int,
                       cfg: Optional[OverflowConfig] = None,
                       mode: Optional[ExecutionMode] = None,
                       probe: Optional[Callable[[int, int, float, float], None]] = None,
                       scheduler: int = 0, device: int = 0,
                       probe_capacity: int = 1 << 20, virtual_ranks: int = 1,
                       host_pipeline: int = 0, fast_diag: bool = False) -> SolveResult:
    """Solves A*Y + Y*B = alpha*C with every tile of Y bounded by cfg.omega (tiled_solve.hpp:29-40).

    HOST arrays in, HOST array out (the reference calling convention). ``mode.workers`` is the
    reference's worker count and maps to GPUs like the C++ shim: w >= 2 solves on min(w, visible
    GPUs, 8) GPUs of this process (rsylv_b200_solve_group); with one visible GPU and
    RSYLV_B200_VIRTUAL_RANKS=1, min(w, 8) virtual ranks share it (a probe keeps one GPU).
    ``host_pipeline`` (0 auto, 1 on, -1 off) streams the inputs to the device tile column by tile
    column while the solve runs (rsylv_b200_options)."""
    cfg = cfg or OverflowConfig()
    c = np.asarray(c, dtype=np.float64)
    if c.ndim != 2 or c.shape[0] != a.dim() or c.shape[1] != b.dim():
        raise ValueError("solve_tiled_robust: C does not conform with A and B")
    m, n = c.shape
    cf = np.asfortranarray(c)
    y = np.zeros((m, n), order="F")
    opt = nat.Options(cfg.omega, cfg.small_num, int(tile_size), scheduler, int(virtual_ranks),
                      int(host_pipeline), int(bool(fast_diag)))
    res = nat.Result()
    pbuf = None
    if probe is not None:
        pbuf = (nat.ProbeEvent * probe_capacity)()
        res.probe_log = C.cast(pbuf, C.POINTER(nat.ProbeEvent))
        res.probe_cap = probe_capacity
    dp = lambda x: x.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731
    up = lambda x: x.ctypes.data_as(C.POINTER(C.c_ubyte))  # noqa: E731
    am, bm = a.matrix(), b.matrix()
    w = min(int(mode.workers), 8) if mode is not None else 0
    gpus = nat.lib().rsylv_b200_device_count() if (w >= 2 and probe is None) else 1
    if w >= 2 and probe is None and gpus >= 2:
        R = min(w, gpus)
        ctxs = (C.c_void_p * R)(*[nat.context(d) for d in range(R)])
        st = nat.lib().rsylv_b200_solve_group(ctxs, R, m, n, dp(am), m, up(a.codes), dp(bm), n,
                                              up(b.codes), dp(cf), m, dp(y), m, C.byref(opt),
                                              C.byref(res))
    else:
        if w >= 2 and probe is None and os.environ.get("RSYLV_B200_VIRTUAL_RANKS") == "1":
            opt.virtual_ranks = w
        st = nat.lib().rsylv_b200_solve(nat.context(device), m, n, dp(am), m, up(a.codes), dp(bm),
                                        n, up(b.codes), dp(cf), m, dp(y), m, C.byref(opt),
                                        C.byref(res))
    cfg.scaling_events += int(res.scaling_events)
    _replay_probe(res, pbuf, probe)
    out = SolveResult(res.alpha, y, int(res.alpha_exp), int(res.scaling_events), res.device_ms,
                      res.max_tile_norm)
    if st not in (nat.RSYLV_OK,):
        raise _status_to_exc(st, res, out if st == nat.RSYLV_SCALE_UNDERFLOW else None)
    return out


def solve_tiled_robust_device(a_dev, a_codes, b_dev, b_codes, c_dev, y_dev, tile_size: int,
                              cfg: Optional[OverflowConfig] = None, stream=None,
                              scheduler: int = 0, device: int = 0, raise_underflow=True,
                              virtual_ranks: int = 1, fast_diag: bool = False):
    """Device-resident variant: torch CUDA tensors (column-major, i.e. ``t.T.contiguous().T``
    or any tensor whose stride(0) == 1). Returns (status, nat.Result)."""
    cfg = cfg or OverflowConfig()
    m, n = c_dev.shape
    for t in (a_dev, b_dev, c_dev, y_dev):
        if t.stride(0) != 1:
            raise ValueError("device arrays must be column-major (stride(0) == 1)")
    opt = nat.Options(cfg.omega, cfg.small_num, int(tile_size), scheduler, int(virtual_ranks), 0,
                      int(bool(fast_diag)))
    res = nat.Result()
    up = lambda x: x.ctypes.data_as(C.POINTER(C.c_ubyte))  # noqa: E731
    st = nat.lib().rsylv_b200_solve_device(
        nat.context(device), m, n, C.c_void_p(a_dev.data_ptr()), a_dev.stride(1),
        up(np.ascontiguousarray(a_codes, dtype=np.uint8)), C.c_void_p(b_dev.data_ptr()),
        b_dev.stride(1), up(np.ascontiguousarray(b_codes, dtype=np.uint8)),
        C.c_void_p(c_dev.data_ptr()), c_dev.stride(1), C.c_void_p(y_dev.data_ptr()),
        y_dev.stride(1), C.byref(opt), C.c_void_p(stream) if stream else None, C.byref(res))
    cfg.scaling_events += int(res.scaling_events)
    if st != nat.RSYLV_OK and not (st == nat.RSYLV_SCALE_UNDERFLOW and not raise_underflow):
        raise _status_to_exc(st, res)
    return st, res


def solve_robust_scalar(a: QuasiTriangular, b: QuasiTriangular, c,
                        cfg: Optional[OverflowConfig] = None, device: int = 0) -> SolveResult:
    """rsylv::solve_robust_scalar (scalar_solve.hpp:27-32): A*Y + Y*B = alpha*C with one global
    scale. On the GPU this is the tiled robust solve with the whole matrix as the requested tile
    (served by 128-tiles); Y/alpha is the same solution."""
    c = np.asarray(c, dtype=np.float64)
    return solve_tiled_robust(a, b, c, max(2, c.shape[0], c.shape[1]), cfg, device=device)


def solve_nonrobust(a: QuasiTriangular, b: QuasiTriangular, c, device: int = 0) -> np.ndarray:
    """rsylv::solve_nonrobust (scalar_solve.hpp:24-25): plain block back substitution, entries
    may overflow to Inf. Runs the same GPU engine with omega = +Inf, so no guard ever fires and
    no input is rejected (the reference does not validate either); raises
    SingularEquationError like the reference."""
    cfg = OverflowConfig(omega=float("inf"))
    r = solve_tiled_robust(a, b, np.asarray(c, dtype=np.float64), 128, cfg, device=device)
    return r.y


def robust_update(c, c_exp: int, a, b, ab_exp: int, omega: float = 0.0, device: int = 0):
    """<gamma,C> <- <gamma,C> - <alpha,A><beta,B> (robust_update.hpp:25-33) on the GPU.

    Scales are powers of two: gamma = 2**c_exp, alpha*beta = 2**ab_exp. Returns
    (new C, new exponent, inf-norm, scaling events)."""
    c = np.asfortranarray(np.array(c, dtype=np.float64))
    a = np.asfortranarray(np.asarray(a, dtype=np.float64))
    b = np.asfortranarray(np.asarray(b, dtype=np.float64))
    m, n = c.shape
    k = a.shape[1]
    ce, cn, ev = C.c_int32(c_exp), C.c_double(0), C.c_uint64(0)
    dp = lambda x: x.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731
    st = nat.lib().rsylv_b200_robust_update(nat.context(device), m, k, n, dp(c), C.byref(ce),
                                            C.byref(cn), dp(a), dp(b), ab_exp, omega, C.byref(ev))
    if st != nat.RSYLV_OK:
        raise RuntimeError(f"robust_update failed: {st}")
    return c, int(ce.value), float(cn.value), int(ev.value)


def _colmajor(t, name):
    if t.stride(0) != 1:
        raise ValueError(f"{name}: device arrays must be column-major (stride(0) == 1)")
    return t.stride(1) if t.dim() == 2 and t.shape[1] > 1 else max(1, t.shape[0])


def dgemm(a_dev, b_dev, c_dev, alpha: float = 1.0, beta: float = 0.0, ta: bool = False,
          tb: bool = False, a_upper: bool = False, b_upper: bool = False, stream=None,
          device: int = 0):
    """C = alpha * op(A) op(B) + beta * C on the FP64 tensor path (rsylv_b200_dgemm), torch
    CUDA tensors in column-major layout; a_upper / b_upper skip the structural zeros of an
    upper quasi-triangular op(A) / op(B)."""
    m, n = c_dev.shape
    k = a_dev.shape[0] if ta else a_dev.shape[1]
    if (b_dev.shape[1] if tb else b_dev.shape[0]) != k or (a_dev.shape[1] if ta else a_dev.shape[0]) != m \
            or (b_dev.shape[0] if tb else b_dev.shape[1]) != n:
        raise ValueError("dgemm: shapes do not conform")
    st = nat.lib().rsylv_b200_dgemm(
        nat.context(device), int(ta), int(tb), m, n, k, float(alpha), C.c_void_p(a_dev.data_ptr()),
        _colmajor(a_dev, "A"), C.c_void_p(b_dev.data_ptr()), _colmajor(b_dev, "B"), float(beta),
        C.c_void_p(c_dev.data_ptr()), _colmajor(c_dev, "C"), int(a_upper), int(b_upper),
        C.c_void_p(stream) if stream is not None else None)
    if st != nat.RSYLV_OK:
        raise RuntimeError(f"rsylv_b200_dgemm: {nat.lib().rsylv_b200_status_string(st).decode()}")
    return c_dev


def relative_residual_device(a_dev, b_dev, c_dev, y_dev, alpha_exp: int, stream=None,
                             device: int = 0) -> dict:
    """Overflow-safe relative residual of A Y + Y B = 2^alpha_exp C on the device
    (src/testgen.cpp:64-79 in a power-of-two prescaled frame; rsylv_b200_relative_residual)."""
    m, n = c_dev.shape
    out = (C.c_double * 7)()
    st = nat.lib().rsylv_b200_relative_residual(
        nat.context(device), m, n, C.c_void_p(a_dev.data_ptr()), _colmajor(a_dev, "A"),
        C.c_void_p(b_dev.data_ptr()), _colmajor(b_dev, "B"), C.c_void_p(c_dev.data_ptr()),
        _colmajor(c_dev, "C"), C.c_void_p(y_dev.data_ptr()), _colmajor(y_dev, "Y"),
        int(alpha_exp), C.c_void_p(stream) if stream is not None else None, out)
    if st != nat.RSYLV_OK:
        raise RuntimeError(f"rsylv_b200_relative_residual: {nat.lib().rsylv_b200_status_string(st).decode()}")
    return dict(relres=out[0], norm_r=out[1], norm_a=out[2], norm_b=out[3], norm_y=out[4],
                norm_c=out[5], frame=int(out[6]))


def _dptr(x):
    return x.ctypes.data_as(C.POINTER(C.c_double))


def _iptr(x):
    return x.ctypes.data_as(C.POINTER(C.c_int32))


def debug_small_solve(cases, omega: float = 0.0, small_num: float = 0.0, device: int = 0):
    """The diagonal-tile solver's exact block solve (complete pivoting + division guard) on
    single blocks: cases = [(a, b, c)] with a rs x rs, b cs x cs, c rs x cs (rs, cs in {1, 2}).
    Returns [(status, z, dz, pivot)] with a z + z b = 2^-dz c (rsylv_b200_debug_small_solve)."""
    nat.context(device)
    n = len(cases)
    rs = np.array([np.shape(a)[0] for a, _, _ in cases], dtype=np.int32)
    cs = np.array([np.shape(b)[0] for _, b, _ in cases], dtype=np.int32)
    pack = lambda xs: np.stack([np.pad(np.asarray(x, float).reshape(np.shape(x)),  # noqa: E731
                                       ((0, 2 - np.shape(x)[0]), (0, 2 - np.shape(x)[1])))
                                .flatten(order="F") for x in xs])
    A, B, Cm = pack([a for a, _, _ in cases]), pack([b for _, b, _ in cases]), pack([c for _, _, c in cases])
    Z = np.zeros((n, 4))
    dz, stt = np.zeros(n, np.int32), np.zeros(n, np.int32)
    piv = np.zeros(n)
    st = nat.lib().rsylv_b200_debug_small_solve(n, _iptr(rs), _iptr(cs), _dptr(A), _dptr(B),
                                                _dptr(Cm), float(omega), float(small_num),
                                                _dptr(Z), _iptr(dz), _iptr(stt), _dptr(piv))
    if st != nat.RSYLV_OK:
        raise RuntimeError("rsylv_b200_debug_small_solve failed")
    out = []
    for t in range(n):
        z = Z[t].reshape((2, 2), order="F")[:rs[t], :cs[t]]
        out.append((int(stt[t]), z, int(dz[t]), float(piv[t])))
    return out


def debug_guards(c, a, b, bnd, t, omega: float, device: int = 0):
    """Exponent-form guards (rsylv_b200_debug_guards): returns (d_update_xq, d_update_xf,
    d_division) arrays; the scale factor is 2^-d (-1: division by zero)."""
    nat.context(device)
    arrs = [np.ascontiguousarray(x, dtype=np.float64) for x in (c, a, b, bnd, t)]
    n = len(arrs[0])
    o = [np.zeros(n, np.int32) for _ in range(3)]
    st = nat.lib().rsylv_b200_debug_guards(n, *[_dptr(x) for x in arrs], float(omega),
                                           *[_iptr(x) for x in o])
    if st != nat.RSYLV_OK:
        raise RuntimeError("rsylv_b200_debug_guards failed")
    return tuple(o)
