"""Where the host-buffer call's time goes (development tool): wall time of rsylv_b200_solve with
pinned buffers against its device-side phases (prepare / DAG incl. waiting on the streamed
inputs / unpack) and the device-resident DAG of the same system.
    python tools/e2e_breakdown.py [config] [reps]"""
import ctypes as C, json, os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch
from paper_1905_10574_b200 import api, _native as nat
from paper_1905_10574_b200.configs import CONFIGS, device_system
name = sys.argv[1] if len(sys.argv) > 1 else "c5"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cfg = CONFIGS[name]
A, ac, B, bc, Cm = device_system(cfg, torch)
Y = torch.empty((cfg.n, cfg.m), dtype=torch.float64, device="cuda").T
for _ in range(2):
    st, res = api.solve_tiled_robust_device(A, ac, B, bc, Cm, Y, cfg.tile, raise_underflow=False)
print(json.dumps({"config": name, "path": "device-resident", "pack_ms": res.pack_ms, "dag_ms": res.dag_ms,
                  "unpack_ms": res.unpack_ms}), flush=True)
del Y
L = nat.lib(); ctx = nat.context(0)
up = lambda x: x.ctypes.data_as(C.POINTER(C.c_ubyte))
pa = torch.empty((cfg.m, cfg.m), dtype=torch.float64, pin_memory=True); pa.copy_(A.T)
pb = torch.empty((cfg.n, cfg.n), dtype=torch.float64, pin_memory=True); pb.copy_(B.T)
pc = torch.empty((cfg.n, cfg.m), dtype=torch.float64, pin_memory=True); pc.copy_(Cm.T)
py = torch.empty((cfg.n, cfg.m), dtype=torch.float64, pin_memory=True)
del A, B, Cm
torch.cuda.synchronize()
dp = lambda t: C.cast(C.c_void_p(t.data_ptr()), C.POINTER(C.c_double))
opt = nat.Options(0.0, 0.0, cfg.tile, 0, 0)
for it in range(reps + 1):
    r = nat.Result()
    t0 = time.perf_counter()
    st = L.rsylv_b200_solve(ctx, cfg.m, cfg.n, dp(pa), cfg.m, up(ac), dp(pb), cfg.n, up(bc), dp(pc), cfg.m,
                            dp(py), cfg.m, C.byref(opt), C.byref(r))
    wall = 1e3 * (time.perf_counter() - t0)
    if it:
        print(json.dumps({"config": name, "path": "host buffers (pinned)", "status": st, "wall_ms": wall,
                          "device_ms": r.device_ms, "pack_ms": r.pack_ms, "dag_ms": r.dag_ms, "unpack_ms": r.unpack_ms,
                          "after_device_ms": wall - r.device_ms, "h2d_GB": r.h2d_bytes / 1e9, "d2h_GB": r.d2h_bytes / 1e9}), flush=True)
