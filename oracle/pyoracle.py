"""TEST INFRASTRUCTURE ONLY: ctypes bindings for the CPU oracle.

Two libraries, both built by ``oracle/Makefile`` into ``oracle/_ref/``:

* ``librsylv_ref.so`` -- the UNMODIFIED reference library (rsylv, /root/reference/proj/src),
  reached through ``oracle/ref_capi.cpp``. Used to pin the restatement and as the CPU baseline.
* ``liboracle.so``    -- ``oracle/rsylv_oracle.c``, the plain-C restatement (the checker).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline leg import this module.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")

OK, INVALID, SINGULAR, UNDERFLOW = 0, 1, 2, 3
STATUS_NAMES = {0: "ok", 1: "invalid_argument", 2: "SingularEquationError",
                3: "ScaleUnderflowError", 4: "other"}

_dp = C.POINTER(C.c_double)
_up = C.POINTER(C.c_ubyte)
_sz = C.c_size_t
_u64p = C.POINTER(C.c_uint64)


def _d(a):
    return None if a is None else a.ctypes.data_as(_dp)


def _u(a):
    return None if a is None else a.ctypes.data_as(_up)


def _lib(name):
    path = os.path.join(REF_DIR, name)
    if not os.path.exists(path):
        raise FileNotFoundError(f"{path} missing: run `make -C oracle` (or __graft_entry__.build())")
    return C.CDLL(path)


_REF = None
_ORA = None


def host_has_avx512() -> bool:
    try:
        with open("/proc/cpuinfo") as f:
            flags = f.read()
        return all(x in flags for x in ("avx512f", "avx512bw", "avx512dq", "avx512vl", "avx512cd"))
    except OSError:
        return False


def ref_variant() -> str:
    """Which reference build ref_lib() loads: "v3" (x86-64-v3, the pinned test build) unless
    RSYLV_REF_VARIANT=native asks for the best build this host runs (x86-64-v4 / AVX-512 when
    available: the CPU baseline of bench.py, mirroring the reference's -march=native)."""
    want = os.environ.get("RSYLV_REF_VARIANT", "v3")
    if want == "native" and host_has_avx512() and os.path.exists(os.path.join(REF_DIR, "librsylv_ref_v4.so")):
        return "v4"
    return "v3"


def ref_lib():
    global _REF
    if _REF is None:
        lib = _lib("librsylv_ref_v4.so" if ref_variant() == "v4" else "librsylv_ref.so")
        lib.ref_solve_tiled.argtypes = [_sz, _sz, _dp, _sz, _up, _dp, _sz, _up, _dp, _sz, _sz,
                                        C.c_double, C.c_double, _sz, _dp, _sz, _dp, _u64p, _dp]
        lib.ref_solve_robust_scalar.argtypes = [_sz, _sz, _dp, _up, _dp, _up, _dp, C.c_double,
                                                C.c_double, _dp, _dp, _u64p, _dp]
        lib.ref_solve_nonrobust.argtypes = [_sz, _sz, _dp, _up, _dp, _up, _dp, _dp, _dp]
        lib.ref_robust_update.argtypes = [_sz, _sz, _sz, _dp, _dp, _dp, _dp, C.c_double,
                                          C.c_double, _dp, C.c_double, C.c_double, C.c_double,
                                          _u64p]
        lib.ref_small_sylvester.argtypes = [_sz, _sz, _dp, _dp, _dp, C.c_double, C.c_double,
                                            _dp, _dp, _dp]
        lib.ref_protect_update.argtypes = [C.c_double] * 4 + [_dp]
        lib.ref_protect_division.argtypes = [C.c_double] * 3 + [_dp, _dp]
        lib.ref_relative_residual.argtypes = [_sz, _sz, _dp, _dp, _dp, _dp, C.c_double, _dp]
        lib.ref_generate_quasi_triangular.argtypes = [_sz, C.c_double, C.c_int, _dp, _up]
        lib.ref_random_system.argtypes = [C.c_uint64, _sz, _sz, _dp, _up, _dp, _up, _dp]
        lib.ref_dense_kron_solve.argtypes = [_sz, _sz, _dp, _up, _dp, _up, _dp, _dp]
        _REF = lib
    return _REF


def oracle_lib():
    global _ORA
    if _ORA is None:
        lib = _lib("liboracle.so")
        lib.or_solve_tiled.argtypes = [_sz, _sz, _dp, _sz, _up, _dp, _sz, _up, _dp, _sz, _sz,
                                       C.c_double, C.c_double, _dp, _sz, _dp, _u64p, _dp,
                                       C.c_void_p, C.c_void_p]
        lib.or_solve_robust_scalar.argtypes = [_sz, _sz, _dp, _up, _dp, _up, _dp, C.c_double,
                                               C.c_double, _dp, _dp, _u64p, _dp]
        lib.or_solve_nonrobust.argtypes = [_sz, _sz, _dp, _up, _dp, _up, _dp, _dp, _dp]
        lib.or_robust_update.argtypes = [_sz, _sz, _sz, _dp, _dp, _dp, _dp, C.c_double,
                                         C.c_double, _dp, C.c_double, C.c_double, C.c_double,
                                         _u64p]
        lib.or_small_sylvester.argtypes = [_sz, _sz, _dp, _dp, _dp, C.c_double, C.c_double,
                                           _dp, _dp, _dp]
        lib.or_protect_update.argtypes = [C.c_double] * 4 + [_dp]
        lib.or_protect_division.argtypes = [C.c_double] * 3 + [_dp, _dp]
        lib.or_inf_norm.argtypes = [_dp, _sz, _sz, _sz]
        lib.or_inf_norm.restype = C.c_double
        lib.or_kron_solve.argtypes = [_sz, _sz, _dp, _dp, _dp, _dp]
        lib.or_relative_residual.argtypes = [_sz, _sz, _dp, _dp, _dp, _dp, C.c_double]
        lib.or_relative_residual.restype = C.c_double
        lib.or_relative_residual_safe.argtypes = [_sz, _sz, _dp, _sz, _dp, _sz, _dp, _sz, _dp,
                                                  _sz, C.c_double, C.c_int]
        lib.or_relative_residual_safe.restype = C.c_double
        _ORA = lib
    return _ORA


PROBE_FN = C.CFUNCTYPE(None, C.c_size_t, C.c_size_t, C.c_double, C.c_double, C.c_void_p)


@dataclass
class Solve:
    status: int
    y: np.ndarray | None
    alpha: float
    events: int
    pivot: float = 0.0


def _f(a):
    return np.asfortranarray(a, dtype=np.float64)


def _blk(b, n):
    if b is None:
        return None
    return np.ascontiguousarray(b, dtype=np.uint8)


def solve_tiled(a, ablk, b, bblk, c, tile, omega=0.0, small_num=0.0, workers=0, impl="oracle",
                probe=None):
    """Sequential (workers=0) or parallel tiled robust solve. impl: 'oracle' or 'ref'."""
    a, b, c = _f(a), _f(b), _f(c)
    m, n = c.shape
    ab, bb = _blk(ablk, m), _blk(bblk, n)
    y = np.zeros((m, n), order="F")
    alpha, ev, piv = C.c_double(0), C.c_uint64(0), C.c_double(0)
    if impl == "ref":
        st = ref_lib().ref_solve_tiled(m, n, _d(a), m, _u(ab), _d(b), n, _u(bb), _d(c), m, tile,
                                       omega, small_num, workers, _d(y), m, C.byref(alpha),
                                       C.byref(ev), C.byref(piv))
    else:
        cb = None
        if probe is not None:
            cb = PROBE_FN(lambda k, l, s, nr, u: probe(k, l, s, nr))
        st = oracle_lib().or_solve_tiled(m, n, _d(a), m, _u(ab), _d(b), n, _u(bb), _d(c), m,
                                         tile, omega, small_num, _d(y), m, C.byref(alpha),
                                         C.byref(ev), C.byref(piv),
                                         C.cast(cb, C.c_void_p) if cb else None, None)
    return Solve(st, y if st == 0 else None, alpha.value, ev.value, piv.value)


def solve_robust_scalar(a, ablk, b, bblk, c, omega=0.0, small_num=0.0, impl="oracle"):
    a, b, c = _f(a), _f(b), _f(c)
    m, n = c.shape
    y = np.zeros((m, n), order="F")
    alpha, ev, piv = C.c_double(0), C.c_uint64(0), C.c_double(0)
    fn = ref_lib().ref_solve_robust_scalar if impl == "ref" else oracle_lib().or_solve_robust_scalar
    st = fn(m, n, _d(a), _u(_blk(ablk, m)), _d(b), _u(_blk(bblk, n)), _d(c), omega, small_num,
            _d(y), C.byref(alpha), C.byref(ev), C.byref(piv))
    return Solve(st, y if st == 0 else None, alpha.value, ev.value, piv.value)


def solve_nonrobust(a, ablk, b, bblk, c, impl="oracle"):
    a, b, c = _f(a), _f(b), _f(c)
    m, n = c.shape
    y = np.zeros((m, n), order="F")
    piv = C.c_double(0)
    fn = ref_lib().ref_solve_nonrobust if impl == "ref" else oracle_lib().or_solve_nonrobust
    st = fn(m, n, _d(a), _u(_blk(ablk, m)), _d(b), _u(_blk(bblk, n)), _d(c), _d(y), C.byref(piv))
    return Solve(st, y if st == 0 else None, 1.0, 0, piv.value)


def robust_update(c, c_scale, c_norm, a, a_scale, a_norm, b, b_scale, b_norm, omega=0.0,
                  impl="oracle"):
    c = np.array(c, dtype=np.float64, order="F", copy=True)
    a, b = _f(a), _f(b)
    m, n = c.shape
    k = a.shape[1]
    cs, cn, ev = C.c_double(c_scale), C.c_double(c_norm), C.c_uint64(0)
    fn = ref_lib().ref_robust_update if impl == "ref" else oracle_lib().or_robust_update
    st = fn(m, k, n, _d(c), C.byref(cs), C.byref(cn), _d(a), a_scale, a_norm, _d(b), b_scale,
            b_norm, omega, C.byref(ev))
    return st, c, cs.value, cn.value, ev.value


def small_sylvester(a, b, c, omega=0.0, small_num=0.0, impl="oracle"):
    a, b, c = _f(a), _f(b), _f(c)
    z = c.copy(order="F")
    beta, piv = C.c_double(0), C.c_double(0)
    if impl == "ref":
        out = np.zeros_like(z)
        st = ref_lib().ref_small_sylvester(a.shape[0], b.shape[0], _d(a), _d(b), _d(c), omega,
                                           small_num, _d(out), C.byref(beta), C.byref(piv))
        z = out
    else:
        st = oracle_lib().or_small_sylvester(a.shape[0], b.shape[0], _d(a), _d(b), _d(z), omega,
                                             small_num, C.byref(beta), C.byref(piv))
    return st, z, beta.value, piv.value


def protect_update(cn, an, bn, omega, impl="oracle"):
    z = C.c_double(0)
    fn = ref_lib().ref_protect_update if impl == "ref" else oracle_lib().or_protect_update
    st = fn(cn, an, bn, omega, C.byref(z))
    return st, z.value


def protect_division(nb, d, omega, impl="oracle"):
    z, piv = C.c_double(0), C.c_double(0)
    fn = ref_lib().ref_protect_division if impl == "ref" else oracle_lib().or_protect_division
    st = fn(nb, d, omega, C.byref(z), C.byref(piv))
    return st, z.value


def inf_norm(x):
    x = _f(x)
    return oracle_lib().or_inf_norm(_d(x), x.shape[0], x.shape[1], x.shape[0])


def kron_solve(a, b, c):
    a, b, c = _f(a), _f(b), _f(c)
    m, n = c.shape
    y = np.zeros((m, n), order="F")
    st = oracle_lib().or_kron_solve(m, n, _d(a), _d(b), _d(c), _d(y))
    if st:
        raise RuntimeError("kron_solve: singular")
    return y


def relative_residual(a, b, c, y, alpha):
    a, b, c, y = _f(a), _f(b), _f(c), _f(y)
    m, n = c.shape
    return oracle_lib().or_relative_residual(m, n, _d(a), _d(b), _d(c), _d(y), alpha)


def relative_residual_safe(a, b, c, y, alpha_mant=1.0, alpha_exp=0):
    """Overflow-safe residual; alpha = alpha_mant * 2**alpha_exp (exponent form allowed)."""
    a, b, c, y = _f(a), _f(b), _f(c), _f(y)
    m, n = c.shape
    return oracle_lib().or_relative_residual_safe(m, n, _d(a), m, _d(b), n, _d(c), m, _d(y), m,
                                                  alpha_mant, alpha_exp)


# ---------- reference-suite input generators (through the unmodified reference) ----------

def ref_generate_quasi_triangular(n, mu, pattern="mixed"):
    out = np.zeros((n, n), order="F")
    blk = np.zeros(n, dtype=np.uint8)
    st = ref_lib().ref_generate_quasi_triangular(n, mu, 0 if pattern == "mixed" else 1, _d(out),
                                                 _u(blk))
    assert st == 0
    return out, blk


def ref_random_system(seed, m, n):
    a = np.zeros((m, m), order="F")
    b = np.zeros((n, n), order="F")
    c = np.zeros((m, n), order="F")
    ab = np.zeros(m, dtype=np.uint8)
    bb = np.zeros(n, dtype=np.uint8)
    st = ref_lib().ref_random_system(seed, m, n, _d(a), _u(ab), _d(b), _u(bb), _d(c))
    assert st == 0
    return a, ab, b, bb, c
