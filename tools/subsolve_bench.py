"""Single-warp latency of one 16x16 sub-block solve (development tool). Built with
EXTRA=-DRSYLV_SUBPROF, it also prints the per-section cycle split (g_prof[8..12])."""
import ctypes as C, sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_1905_10574_b200 import _native as nat
L = nat.lib(); nat.context()
L.rsylv_b200_debug_subsolve.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_longlong)]
L.rsylv_b200_debug_counters.argtypes = [C.POINTER(C.c_uint64), C.c_int]
reps = 50
for mixed in (0, 1):
    cyc = C.c_longlong(0)
    out = (C.c_uint64 * 16)()
    L.rsylv_b200_debug_counters(out, 1)
    L.rsylv_b200_debug_subsolve(reps, mixed, C.byref(cyc))
    L.rsylv_b200_debug_counters(out, 0)
    print("mixed" if mixed else "1x1  ", "cycles per 16x16 sub-block solve:", cyc.value, " per lane-step:", round(cyc.value / 31, 1))
    names = ["setup", "rhs", "solve", "vote+exact", "install+colupd"]
    if any(out[8 + k] for k in range(5)):
        print("   per solve:", " ".join(f"{names[k]}={out[8 + k] / reps:.0f}" for k in range(5)),
              " per step:", " ".join(f"{names[k]}={out[8 + k] / reps / 31:.0f}" for k in range(1, 5)))
