"""Development patch: in-tile updates split into urgent (next anti-diagonal) and deferred
(later anti-diagonals, overlapped with the next step's sub-block solves on the idle warps)."""
import sys
p = sys.argv[1]
s = open(p).read()
a = s.index("    constexpr int kT8 = kSub / 8;\n    int nev_w = 0;\n    for (int w = 0; w < NP + NQ - 1; ++w) {")
b = s.index("    if (lane == 0 && nev_w) atomicAdd(&ss.events, nev_w);")
loop = s[a:b]
# the solver block
sa = loop.index("        for (int it = warp; it < nit; it += kWarps) {")
sb = loop.index("        __syncthreads();\n        PROF_ADD(2, t_0);")
solver = loop[sa:sb]
# the item body
ia = loop.index("            const int t = rem;\n")
ib = loop.index("        __syncthreads();\n        PROF_ADD(3, t_0);")
item = loop[ia + len("            const int t = rem;\n"):ib]
item = item.rstrip()
assert item.endswith("}")
item = item[:-1]  # drop the closing brace of the di loop
item = item.replace("            if (!hasc && !hasr) continue;", "            if (!hasc && !hasr) return;")
item_lines = [l[4:] if l.startswith("    ") else l for l in item.split("\n")]
item = "\n".join(item_lines)
new = """    constexpr int kT8 = kSub / 8;
    int nev_w = 0;
    const int nd = NP + NQ - 1;
    // Update of destination sub-block (r, t) by the sub-blocks solved on anti-diagonal w: at most
    // one column update  T(r,t) -= A(r,p_t) X(p_t,t)  and one row update  T(r,t) -= X(r,q_r) B(q_r,t),
    // under one exponent-form ProtectUpdate.
    auto upd = [&](int w, int r, int t) {
        const int qlo = max(0, w - (NP - 1)), qhi = min(NQ - 1, w);
""" + item + """    };
    // all such updates whose destination lies on anti-diagonals [dmin, dmax], over the warps
    // [w0, w0 + nw)
    auto upd_range = [&](int w, int dmin, int dmax, int w0, int nw) {
        if (warp < w0) return;
        int ndest = 0;
        for (int r = 0; r < NP; ++r) {
            const int base = NP - 1 - r;  // anti-diagonal of (r, t) = base + t
            ndest += max(0, min(NQ - 1, dmax - base) - max(0, dmin - base) + 1);
        }
        for (int di = warp - w0; di < ndest; di += nw) {
            int r = 0, rem = di, t = 0;
            for (;; ++r) {
                const int base = NP - 1 - r;
                const int tlo = max(0, dmin - base);
                const int cnt = max(0, min(NQ - 1, dmax - base) - tlo + 1);
                if (rem < cnt) {
                    t = tlo + rem;
                    break;
                }
                rem -= cnt;
            }
            upd(w, r, t);
        }
    };
    // Sub-block wavefront. Step w: the warps [0, nit) solve the sub-blocks on anti-diagonal w
    // while the idle warps apply the DEFERRED updates of step w-1 (destinations on anti-diagonals
    // >= w+1); after a barrier all warps apply the URGENT updates of step w (destinations on
    // w+1), which the next step's solves wait for. Each destination still receives its updates
    // in the order of the source anti-diagonals, so the arithmetic is that of a full right-looking
    // update after every step. xm/xe hold a norm bound of every sub-block, gx its exponent
    // relative to the tile.
    for (int w = 0; w < nd; ++w) {
        const int qlo = max(0, w - (NP - 1)), qhi = min(NQ - 1, w);
        const int nit = qhi - qlo + 1;
        const int nsolv = min(nit, kWarps);
""" + solver + """        if (w > 0 && nsolv < kWarps) upd_range(w - 1, w + 1, nd - 1, nsolv, kWarps - nsolv);
        __syncthreads();
        PROF_ADD(2, t_0);
        if (w == nd - 1) break;
        if (w > 0 && nsolv >= kWarps) {  // no idle warp during the solves (kSub = 8 only)
            upd_range(w - 1, w + 1, nd - 1, 0, kWarps);
            __syncthreads();
        }
        upd_range(w, w + 1, w + 1, 0, kWarps);
        __syncthreads();
        PROF_ADD(3, t_0);
    }
"""
s = s[:a] + new + s[b:]
open(p, 'w').write(s)
print("patched")
