"""Per-phase cycle counters of the tile tasks (development tool)."""
import ctypes as C, sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch
from paper_1905_10574_b200 import api, _native as nat
from paper_1905_10574_b200.configs import CONFIGS, device_system
L = nat.lib()
L.rsylv_b200_debug_counters.argtypes = [C.POINTER(C.c_uint64), C.c_int]
for name in sys.argv[1:] or ["c1"]:
    cfg = CONFIGS[name]
    A, ac, B, bc, Cm = device_system(cfg, torch)
    Y = torch.empty((cfg.n, cfg.m), dtype=torch.float64, device="cuda").T
    api.solve_tiled_robust_device(A, ac, B, bc, Cm, Y, cfg.tile, raise_underflow=False)
    out = (C.c_uint64 * 32)()
    L.rsylv_b200_debug_counters(out, 1)
    st, res = api.solve_tiled_robust_device(A, ac, B, bc, Cm, Y, cfg.tile, raise_underflow=False)
    L.rsylv_b200_debug_counters(out, 0)
    ntiles = res.row_tiles * res.col_tiles
    names = ["update", "setup", "subsolve", "in-tile upd", "finalize"]
    tot = sum(out[i] for i in range(5))
    if out[6]:
        print("   per sub-block (per warp): solve %.2f us, norm %.2f us, count %d" % (out[5] / out[6] / 1965, out[7] / out[6] / 1965, out[6]))
    print("   column-path fallbacks to the exact sub-block solver: %d" % out[12])
    if out[22]:
        print("   fast path per solver-warp call: urgent updates %.2f us, sub-block solve(s) %.2f us (%d calls), immediate repeat %.2f us; deferred updates %.1f us/tile summed over warps" % (out[20] / out[22] / 1965, out[21] / out[22] / 1965, out[22], out[24] / out[22] / 1965, out[23] / ntiles / 1965))
    print("   fast diagonal-tile attempt: %.1f us/tile in its wavefront, %d of %d tiles fell back to the exact path" % (out[14] / ntiles / 1965, out[15], ntiles))
    print("   flag-wait=%.1f us/tile, metadata-arrival=%.1f us/tile, header=%.1f us/tile, chunks=%d prescaled=%d (%.1f%%)" % (out[9] / ntiles / 1965, out[14] / ntiles / 1965, out[13] / ntiles / 1965, out[10], out[11], 100.0 * out[11] / max(1, out[10])))
    nw = ntiles * 16 * 1965
    print("   chunks with an accumulator shift %d (%.1f%%), skipped (not live) %d" % (out[18], 100.0 * out[18] / max(1, out[10]), out[19]))
    print(name, "dag_ms", round(res.dag_ms, 2), "tiles", ntiles, " ".join(
        f"{names[i]}={out[i] / ntiles / 1965:.1f}us({100 * out[i] / tot:.0f}%)" for i in range(5)))
    print("   lookahead-ready sources %d, of which the flag was NOT set at the duty thread's own acquire: %d" % (out[26], out[25]))
    if out[28] and out[31]:
        print("   exact wavefront: urgent update %.2f us per solver warp and step; deferred updates %.2f us per idle warp and step (longest %.1f us)" % (out[30] / out[31] / 1965, out[27] / out[28] / 1965, out[29] / 1965))
    if out[22] and not out[14]:
        print("   in-tile update sections (all calls, per call): bounds + destination load %.2f us, column product %.2f us, row product %.2f us, store %.2f us (%d calls)" % tuple([out[k] / out[22] / 1965 for k in (16, 17, 20, 21)] + [out[22]]))
