"""Single-warp latency of one 16x16 sub-block solve (development tool): mode bit 0 = mixed
1x1/2x2 blocks, bit 1 = force the exact (left-looking) solver instead of the column fast
path. Built with EXTRA=-DRSYLV_SUBPROF it also prints the exact solver's section split."""
import ctypes as C, sys, os
import numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_1905_10574_b200 import _native as nat
L = nat.lib(); nat.context()
L.rsylv_b200_debug_subsolve.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_longlong), C.POINTER(C.c_double)]
L.rsylv_b200_debug_counters.argtypes = [C.POINTER(C.c_uint64), C.c_int]
reps = 50
for mixed in (0, 1):
    outs = []
    for exact in (0, 1):
        cyc = C.c_longlong(0)
        out = np.zeros(256)
        cnt = (C.c_uint64 * 32)()
        L.rsylv_b200_debug_counters(cnt, 1)
        L.rsylv_b200_debug_subsolve(reps, mixed | (exact << 1), C.byref(cyc), out.ctypes.data_as(C.POINTER(C.c_double)))
        L.rsylv_b200_debug_counters(cnt, 0)
        outs.append(out)
        print("mixed" if mixed else "1x1  ", "exact-solver" if exact else "column-path",
              "cycles per 16x16 sub-block solve:", cyc.value, " per lane-step:", round(cyc.value / 31, 1))
        names = ["setup", "rhs", "solve", "vote+exact", "install"]
        if exact and any(cnt[8 + k] for k in range(5)):
            print("   per step:", " ".join(f"{names[k]}={cnt[8 + k] / reps / 31:.0f}" for k in range(1, 5)))
    d = np.abs(outs[0] - outs[1]).max() / np.abs(outs[1]).max()
    print("   column path vs exact solver: max rel diff", d)
