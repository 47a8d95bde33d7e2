"""Golden fixtures for the CLI restatements (records.py, testgen.py), produced by the
UNMODIFIED reference through oracle/_ref/librsylv_ref.so (test infrastructure):
* format_double strings (matrix_io.cpp:10-14) for a fixed set of doubles;
* the first values of random_quasi_triangular / random_dense (verify.cpp:16-56) for seed 42.
Run from the repo root after `make -C oracle`:  python tests/golden/make_cli_golden.py"""
import ctypes as C
import json
import os
import random
import struct

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
L = C.CDLL(os.path.join(ROOT, "oracle", "_ref", "librsylv_ref.so"))
L.ref_format_double.argtypes = [C.c_double, C.c_char_p, C.c_size_t]
buf = C.create_string_buffer(64)

rng = random.Random(20261020)
vals = [0.0, -0.0, 1.0, -1.0, 100.0, 123456.0, 1e5, 1e16, 1e21, 1e22, 1e-5, 1e-4, 0.1, 1 / 3,
        2.5, 5e-324, 2.2250738585072014e-308, 1.7976931348623157e308, 1234.5, 0.001,
        123456789012345678.0, 9.999999999999999e22, 4e-5, 0.00012, 1.5e-7, 1e4, 1e15, 65536.0]
for _ in range(400):
    vals.append(struct.unpack("<d", struct.pack("<Q", rng.getrandbits(64)))[0])
    vals.append(rng.uniform(-1e6, 1e6))
    vals.append(float(rng.randint(-10 ** 20, 10 ** 20)))
    vals.append(round(rng.uniform(0, 100), rng.randint(0, 6)))
vals = [v for v in vals if v == v]
fmt = []
for v in vals:
    L.ref_format_double(v, buf, 64)
    fmt.append([struct.unpack("<Q", struct.pack("<d", v))[0], buf.value.decode()])

m, n = 11, 6
a = np.zeros((m, m), order="F"); b = np.zeros((n, n), order="F"); c = np.zeros((m, n), order="F")
ab = np.zeros(m, np.uint8); bb = np.zeros(n, np.uint8)
dp = lambda x: x.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731
up = lambda x: x.ctypes.data_as(C.POINTER(C.c_ubyte))  # noqa: E731
assert L.ref_random_system(C.c_uint64(42), C.c_size_t(m), C.c_size_t(n), dp(a), up(ab), dp(b),
                           up(bb), dp(c)) == 0
bits = lambda x: [int(u) for u in np.asarray(x, dtype=np.float64).reshape(-1, order="F").view(np.uint64)]  # noqa: E731
out = {"origin": "oracle/_ref (matrix_io.cpp:10-14, verify.cpp:16-56)", "format_double": fmt,
       "random_system": {"seed": 42, "m": m, "n": n, "a": bits(a), "ab": ab.tolist(),
                         "b": bits(b), "bb": bb.tolist(), "c": bits(c)}}
with open(os.path.join(ROOT, "tests", "golden", "cli_golden.json"), "w") as fh:
    json.dump(out, fh)
print(len(fmt), "format cases")
