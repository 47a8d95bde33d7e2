"""Update-phase throughput alone (development tool): scheduler 2 launches one tile task per SM
with the update GEMM only (~M + N source tiles per CTA, results are garbage) on the c5 system,
and reports the DMMA-equivalent TFLOP/s of the update mainloop."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch
from paper_1905_10574_b200 import api
from paper_1905_10574_b200.configs import CONFIGS, device_system
name = sys.argv[1] if len(sys.argv) > 1 else "c5"
cfg = CONFIGS[name]
A, ac, B, bc, Cm = device_system(cfg, torch)
Y = torch.empty((cfg.n, cfg.m), dtype=torch.float64, device="cuda").T
for rep in range(3):
    st, res = api.solve_tiled_robust_device(A, ac, B, bc, Cm, Y, cfg.tile, scheduler=2, raise_underflow=False)
    M, N = res.row_tiles, res.col_tiles
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    flops = 0
    for b in range(sms):
        i, j = (b % M, b % N) if os.environ.get("UB_DISTINCT") else (b % 8, max(0, N - 2 - (b // 8) % 4))
        nsrc = (M - 1 - i) + j
        flops += 2 * 128 * 128 * 128 * nsrc
    print(f"{name}: update-only {res.dag_ms:.2f} ms, {flops / res.dag_ms / 1e9:.2f} TFLOP/s "
          f"({100 * flops / res.dag_ms / 1e9 / 37.05:.1f}% of DMMA peak)")
