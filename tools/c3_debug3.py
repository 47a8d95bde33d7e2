import sys, os, math
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "oracle"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np, pyoracle as po, bigrange as br
import paper_1905_10574_b200 as rs
from paper_1905_10574_b200.configs import CONFIGS, host_system
n, t = 64, 16
cfg = CONFIGS["c3"].scaled(n, tile=t)
a, ac, b, bc, c = host_system(cfg)
A = rs.QuasiTriangular.from_codes(a, ac); B = rs.QuasiTriangular.from_codes(b, bc)
ev = []
def probe(k, l, s, nr):
    ev.append((k, l, s, nr))
import ctypes as C
from paper_1905_10574_b200 import _native as nat
opt = nat.Options(0, 0, t, 1, 0); res = nat.Result()
pb = (nat.ProbeEvent * 10000)(); res.probe_log = C.cast(pb, C.POINTER(nat.ProbeEvent)); res.probe_cap = 10000
y = np.zeros((n, n), order="F"); af = np.asfortranarray(a); bf = np.asfortranarray(b); cf = np.asfortranarray(c)
dp = lambda x: x.ctypes.data_as(C.POINTER(C.c_double)); up = lambda x: x.ctypes.data_as(C.POINTER(C.c_ubyte))
st = nat.lib().rsylv_b200_solve(nat.context(), n, n, dp(af), n, up(ac), dp(bf), n, up(bc), dp(cf), n, dp(y), n, C.byref(opt), C.byref(res))
Y = br.solve(a, ac, b, bc, c)
def true_norm_log2(k, l):
    rows = Y[k*t:(k+1)*t]
    mx = max(sum(abs(v) for v in r[l*t:(l+1)*t]) for r in rows)
    return float(mx.ln(br.CTX) / br.CTX.ln(2)) if mx else float('-inf')
print("status", st, "alpha_exp", res.alpha_exp, "events", res.probe_count)
for i in range(res.probe_count):
    e = pb[i]
    kind = "?"
    print(f"tile ({e.k},{e.l}) exp={e.scale_exp} norm=2^{math.log2(e.norm) if e.norm > 0 else float('-inf'):.2f} "
          f"-> true log2 norm est {math.log2(e.norm) - e.scale_exp if e.norm > 0 else float('nan'):.2f} ; bigrange {true_norm_log2(e.k, e.l):.2f}")
