"""e2e through the host C-ABI (rsylv_b200_solve) with the reference's kind of buffers (ordinary
pageable numpy storage, what DenseMatrix holds) against pinned buffers, with and without the
automatic page-locking of the caller's buffers (development / evidence tool).
    python tools/e2e_pageable.py [config] [reps]  -> one JSON line per variant"""
import ctypes as C
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch  # noqa: E402
from paper_1905_10574_b200 import api, _native as nat  # noqa: E402
from paper_1905_10574_b200.configs import CONFIGS, device_system  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = CONFIGS[name]
A, ac, B, bc, Cm = device_system(cfg, torch)
torch.cuda.synchronize()
L = nat.lib()
ctx = nat.context(0)
up = lambda x: x.ctypes.data_as(C.POINTER(C.c_ubyte))  # noqa: E731


def run(bufs, label):
    a, b, c, y = bufs
    dp = lambda x: C.cast(C.c_void_p(x), C.POINTER(C.c_double))  # noqa: E731
    ptr = lambda t: t.data_ptr() if isinstance(t, torch.Tensor) else t.ctypes.data  # noqa: E731
    opt = nat.Options(0.0, 0.0, cfg.tile, 0, 0)
    ts = []
    for it in range(reps + 1):
        r = nat.Result()
        t0 = time.perf_counter()
        st = L.rsylv_b200_solve(ctx, cfg.m, cfg.n, dp(ptr(a)), cfg.m, up(ac), dp(ptr(b)), cfg.n,
                                up(bc), dp(ptr(c)), cfg.m, dp(ptr(y)), cfg.m, C.byref(opt), C.byref(r))
        dt = time.perf_counter() - t0
        if it:
            ts.append(dt)
    t = sum(ts) / len(ts)
    print(json.dumps({"config": name, "buffers": label, "status": st, "ms_per_solve": 1e3 * t,
                      "gflops": cfg.flops() / t / 1e9, "device_ms": r.device_ms,
                      "h2d_bytes": int(r.h2d_bytes), "d2h_bytes": int(r.d2h_bytes)}), flush=True)
    return y


# pinned (torch pin_memory) -- the bench.py e2e setting
pa = torch.empty((cfg.m, cfg.m), dtype=torch.float64, pin_memory=True); pa.copy_(A.T)
pb = torch.empty((cfg.n, cfg.n), dtype=torch.float64, pin_memory=True); pb.copy_(B.T)
pc = torch.empty((cfg.n, cfg.m), dtype=torch.float64, pin_memory=True); pc.copy_(Cm.T)
py = torch.empty((cfg.n, cfg.m), dtype=torch.float64, pin_memory=True)
torch.cuda.synchronize()
y1 = run((pa, pb, pc, py), "pinned").clone()
# pageable numpy copies (column-major storage = the transposed torch layout)
na, nb, nc = pa.numpy().copy(), pb.numpy().copy(), pc.numpy().copy()
ny = np.zeros_like(nc)
del pa, pb, pc
os.environ["RSYLV_B200_HOST_REGISTER"] = "0"
run((na, nb, nc, ny), "pageable, not registered (default)")
y2 = ny.copy()
os.environ["RSYLV_B200_HOST_REGISTER"] = "1"
ny[:] = 0
run((na, nb, nc, ny), "pageable, page-locked for the call (RSYLV_B200_HOST_REGISTER=1)")
assert np.array_equal(ny, y2) and np.array_equal(ny, y1.numpy()), "results differ"
print(json.dumps({"bitwise_equal": True}))
