import ctypes as C, sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_1905_10574_b200 import _native as nat
L = nat.lib(); nat.context()
L.rsylv_b200_debug_subsolve.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_longlong)]
for mixed in (0, 1):
    cyc = C.c_longlong(0)
    L.rsylv_b200_debug_subsolve(50, mixed, C.byref(cyc))
    print("mixed" if mixed else "1x1  ", "cycles per 16x16 sub-block solve:", cyc.value, " per lane-step:", round(cyc.value / 31, 1))
