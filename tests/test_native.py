"""CPU tests of the boundary: the C-ABI library loads and exports every symbol declared in
include/rsylv_b200.h; the Python mirror validates like the reference; the product never falls
back to the CPU."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_1905_10574_b200 import _native as nat, api
from paper_1905_10574_b200.configs import CONFIGS, block_codes, host_system, u01

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "rsylv_b200.h")).read()
    return sorted(set(re.findall(r"\b(rsylv_b200_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    assert os.path.exists(nat.LIB_PATH), "build the extension first (__graft_entry__.build())"
    lib = ctypes.CDLL(nat.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 9
    for s in syms:
        assert hasattr(lib, s), s


def test_library_is_sm100a_only():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", nat.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_status_strings():
    lib = nat.lib()
    assert lib.rsylv_b200_status_string(3) == b"ScaleUnderflowError"
    assert lib.rsylv_b200_status_string(2) == b"SingularEquationError"


def test_quasi_triangular_validation_mirrors_reference():
    m = np.triu(np.ones((5, 5)))
    assert api.QuasiTriangular(m).diag_blocks() == [(i, 1) for i in range(5)]
    m2 = m.copy()
    m2[2, 1] = 3.0
    q = api.QuasiTriangular(m2)  # detected 2x2 block (partition.cpp:8-23)
    assert (1, 2) in q.diag_blocks()
    bad = m.copy()
    bad[4, 1] = 1.0
    with pytest.raises(ValueError):
        api.QuasiTriangular(bad)  # below the first subdiagonal (partition.cpp:42-46)
    with pytest.raises(ValueError):
        api.QuasiTriangular(m2, [(0, 1), (1, 1), (2, 1), (3, 1), (4, 1)])  # undeclared 2x2
    with pytest.raises(ValueError):
        api.QuasiTriangular(np.ones((3, 4)))


def test_nonconforming_rhs_rejected_before_any_device_call():
    a = api.QuasiTriangular(np.eye(4))
    b = api.QuasiTriangular(np.eye(3))
    with pytest.raises(ValueError):
        api.solve_tiled_robust(a, b, np.ones((4, 4)), 2)


def test_no_cpu_fallback_without_device():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    a = api.QuasiTriangular(np.eye(4))
    with pytest.raises(RuntimeError):
        api.solve_tiled_robust(a, a, np.ones((4, 4)), 2)


def test_generators_deterministic_and_shaped():
    cfg = CONFIGS["c5"].scaled(64, tile=16)
    a1, ac1, b1, bc1, c1 = host_system(cfg)
    a2, ac2, b2, bc2, c2 = host_system(cfg)
    assert np.array_equal(a1, a2) and np.array_equal(c1, c2) and np.array_equal(ac1, ac2)
    assert np.all(np.tril(a1, -2) == 0)
    frac2 = np.mean(block_codes(40000, 0.5, 12345) == 2) * 2
    assert 0.6 < frac2 < 0.72  # 50% of block starts -> ~2/3 of indices in 2x2 blocks
    # 2x2 block form [[a, b], [-c, a]] (BASELINE config 2)
    i = int(np.argmax(ac1 == 2))
    assert a1[i, i] == a1[i + 1, i + 1] and a1[i + 1, i] < 0 < a1[i, i + 1]
    assert 0.0 <= u01(1, 2, np.arange(4, dtype=np.uint64)).min() < 1.0
