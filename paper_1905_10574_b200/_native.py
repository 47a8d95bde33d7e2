"""ctypes binding of the in-tree CUDA extension ``librsylv_b200.so`` (C-ABI: include/rsylv_b200.h).

There is no CPU fallback: if the extension is missing or no CUDA device is visible, every entry
point raises. Build with ``python -c "import __graft_entry__ as g; g.build()"`` or
``make -C paper_1905_10574_b200/csrc``.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "librsylv_b200.so")

RSYLV_OK, RSYLV_INVALID_ARGUMENT, RSYLV_SINGULAR, RSYLV_SCALE_UNDERFLOW = 0, 1, 2, 3
RSYLV_CUDA_ERROR, RSYLV_NO_DEVICE = 4, 5
DIST_HANDLE_BYTES = 320

REASONS = {0: "", 1: "C does not conform with A and B", 2: "tile size must be >= 2",
           3: "a tile norm of A exceeds omega", 4: "a tile norm of B exceeds omega",
           5: "a tile norm of C exceeds omega", 6: "bad options"}


class Options(C.Structure):
    _fields_ = [("omega", C.c_double), ("small_num", C.c_double), ("tile_size", C.c_size_t),
                ("scheduler", C.c_int), ("virtual_ranks", C.c_int), ("host_pipeline", C.c_int),
                ("fast_diag", C.c_int)]


class ProbeEvent(C.Structure):
    _fields_ = [("k", C.c_uint32), ("l", C.c_uint32), ("scale_exp", C.c_int32),
                ("pad", C.c_int32), ("norm", C.c_double)]


class Result(C.Structure):
    _fields_ = [("alpha", C.c_double), ("alpha_exp", C.c_int32), ("invalid_reason", C.c_int32),
                ("scaling_events", C.c_uint64), ("pivot", C.c_double),
                ("device_ms", C.c_double), ("max_tile_norm", C.c_double),
                ("row_tiles", C.c_size_t), ("col_tiles", C.c_size_t),
                ("probe_log", C.POINTER(ProbeEvent)), ("probe_cap", C.c_size_t),
                ("probe_count", C.c_size_t), ("pack_ms", C.c_double), ("dag_ms", C.c_double),
                ("unpack_ms", C.c_double), ("dag_launches", C.c_uint64),
                ("h2d_bytes", C.c_uint64), ("d2h_bytes", C.c_uint64)]


_dp = C.POINTER(C.c_double)
_up = C.POINTER(C.c_ubyte)
_sz = C.c_size_t
_lib = None


def lib():
    """Load the extension (raises if absent — the product never falls back to the CPU)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"CUDA extension missing: {LIB_PATH} (run __graft_entry__.build())")
        L = C.CDLL(LIB_PATH)
        L.rsylv_b200_create.argtypes = [C.c_int, C.POINTER(C.c_void_p)]
        L.rsylv_b200_destroy.argtypes = [C.c_void_p]
        L.rsylv_b200_status_string.argtypes = [C.c_int]
        L.rsylv_b200_status_string.restype = C.c_char_p
        L.rsylv_b200_last_error.argtypes = [C.c_void_p]
        L.rsylv_b200_last_error.restype = C.c_char_p
        L.rsylv_b200_solve.argtypes = [C.c_void_p, _sz, _sz, _dp, _sz, _up, _dp, _sz, _up, _dp,
                                       _sz, _dp, _sz, C.POINTER(Options), C.POINTER(Result)]
        L.rsylv_b200_solve_device.argtypes = [C.c_void_p, _sz, _sz, C.c_void_p, _sz, _up,
                                              C.c_void_p, _sz, _up, C.c_void_p, _sz, C.c_void_p,
                                              _sz, C.POINTER(Options), C.c_void_p,
                                              C.POINTER(Result)]
        L.rsylv_b200_robust_update.argtypes = [C.c_void_p, _sz, _sz, _sz, _dp,
                                               C.POINTER(C.c_int32), _dp, _dp, _dp, C.c_int32,
                                               C.c_double, C.POINTER(C.c_uint64)]
        L.rsylv_b200_dist_prepare.argtypes = [C.c_void_p, C.c_int, C.c_int, _sz, _sz, C.c_void_p,
                                              _sz, _up, C.c_void_p, _sz, _up, C.c_void_p, _sz,
                                              C.POINTER(Options), C.c_void_p, C.c_void_p,
                                              C.POINTER(Result)]
        L.rsylv_b200_dist_run.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(Result)]
        L.rsylv_b200_dist_finish.argtypes = [C.c_void_p, C.c_int, C.c_void_p, _sz, C.c_void_p,
                                             C.POINTER(Result)]
        L.rsylv_b200_generate_quasi_triangular.argtypes = [_sz, C.c_void_p, _sz, _up,
                                                           C.c_uint64] + [C.c_double] * 6 + [
                                                               C.c_void_p]
        L.rsylv_b200_generate_rhs.argtypes = [_sz, _sz, C.c_void_p, _sz, C.c_uint64, C.c_int,
                                              C.c_double, C.c_double, C.POINTER(C.c_int32), _sz,
                                              _sz, C.c_double, C.c_void_p]
        L.rsylv_b200_dgemm.argtypes = [C.c_void_p, C.c_int, C.c_int, _sz, _sz, _sz, C.c_double,
                                       C.c_void_p, _sz, C.c_void_p, _sz, C.c_double, C.c_void_p,
                                       _sz, C.c_int, C.c_int, C.c_void_p]
        L.rsylv_b200_relative_residual.argtypes = [C.c_void_p, _sz, _sz, C.c_void_p, _sz,
                                                   C.c_void_p, _sz, C.c_void_p, _sz, C.c_void_p,
                                                   _sz, C.c_int32, C.c_void_p, _dp]
        L.rsylv_b200_solve_group.argtypes = [C.POINTER(C.c_void_p), C.c_int, _sz, _sz, _dp, _sz,
                                             _up, _dp, _sz, _up, _dp, _sz, _dp, _sz,
                                             C.POINTER(Options), C.POINTER(Result)]
        L.rsylv_b200_device_count.argtypes = []
        L.rsylv_b200_has_fast_diag.argtypes = []
        _ip = C.POINTER(C.c_int32)
        L.rsylv_b200_debug_small_solve.argtypes = [_sz, _ip, _ip, _dp, _dp, _dp, C.c_double,
                                                   C.c_double, _dp, _ip, _ip, _dp]
        L.rsylv_b200_debug_guards.argtypes = [_sz, _dp, _dp, _dp, _dp, _dp, C.c_double, _ip, _ip,
                                              _ip]
        _lib = L
    return _lib


_ctx = {}


def context(device: int = 0):
    """Process-wide context per device (rsylv_b200_create)."""
    if device not in _ctx:
        h = C.c_void_p()
        st = lib().rsylv_b200_create(device, C.byref(h))
        if st != RSYLV_OK:
            raise RuntimeError(f"rsylv_b200_create failed: {lib().rsylv_b200_status_string(st).decode()}"
                               " (a CUDA device is required; there is no CPU fallback)")
        _ctx[device] = h
    return _ctx[device]
