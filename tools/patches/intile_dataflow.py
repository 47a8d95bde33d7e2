"""Development patch: the diagonal-tile sub-block wavefront as an in-CTA dataflow (shared-memory
flags instead of one CTA barrier per anti-diagonal step)."""
import sys
p = sys.argv[1]
s = open(p).read()
def rep(o, n):
    global s
    assert s.count(o) == 1, o[:80]
    s = s.replace(o, n)
rep("""    int rtab[kSolvers][kSub + 1], ctab[kSolvers][kSub + 1];""",
    """    int rtab[kSolvers][kSub + 1], ctab[kSolvers][kSub + 1];
    int sflag[kSubMax][kSubMax];         // 1 once a sub-block is solved (dataflow wavefront)
    int dcnt[kSubMax][kSubMax];          // deferred updates applied to a sub-block so far""")
a = s.index("    // Sub-block wavefront. Step w: the warps [0, nit) solve the sub-blocks on anti-diagonal w")
b = s.index("    if (lane == 0 && nev_w) atomicAdd(&ss.events, nev_w);")
old_loop = s[a:b]
sa = old_loop.index("        for (int it = warp; it < nit; it += kWarps) {")
sb = old_loop.index("        if (w > 0 && nsolv < kWarps) upd_range(w - 1, w + 1, nd - 1, nsolv, kWarps - nsolv);")
solver_body = old_loop[sa:sb]
# the body between the item header and the end of the for loop
ba = solver_body.index("            const int r0 = ss.rsub[pb]")
bb = solver_body.rindex("        }")
body = solver_body[ba:bb]
body = body.replace("""            // the URGENT updates of this sub-block (from its neighbours solved in step w-1),
            // applied by the warp that solves it: no separate update phase and barrier per step
            if (w > 0 && nsolv < kWarps) {
                upd(w - 1, pb, qb);
                __syncwarp();
            }""", """            // the URGENT update of this sub-block (from its neighbours on anti-diagonal w-1),
            // applied by the warp that solves it
            if (w > 0) {
                upd(w - 1, pb, qb);
                __syncwarp();
            }""")
body = "\n".join(("    " + l) if l.strip() else l for l in body.split("\n"))
new_loop = """    if (kSolvers < kWarps) {
        // Sub-block wavefront as an in-CTA dataflow. Warps [0, kSolvers) take the sub-blocks in
        // anti-diagonal order (round robin); each waits for its two neighbours (sflag) and for
        // its DEFERRED updates (dcnt), applies its URGENT update (from anti-diagonal w-1) and
        // solves. Warps [kSolvers, kWarps) apply the deferred updates -- destination (r, t) from
        // anti-diagonal w' <= d(r, t) - 2 -- in order of w' (round robin), each after its source
        // sub-blocks are solved and the destination's earlier deferred updates are in. Every
        // destination thus receives its updates in source order (the arithmetic of a full
        // right-looking update after every step) without a CTA barrier per step; the lists are
        // topologically ordered, so the round robin cannot deadlock.
        auto wait_ge = [&](int* f, int v) {
            if (lane == 0)
                while (*((volatile int*)f) < v) __nanosleep(20);
            __syncwarp();
            __threadfence_block();
        };
        auto post = [&](int* f, int v) {
            __syncwarp();
            __threadfence_block();
            if (lane == 0) *((volatile int*)f) = v;
        };
        auto wmin_of = [&](int r, int t) { return min(t, NP - 1 - r); };
        if (warp < kSolvers) {
            int k = 0;
            for (int w = 0; w < nd; ++w) {
                const int qlo = max(0, w - (NP - 1)), qhi = min(NQ - 1, w);
                for (int qb = qlo; qb <= qhi; ++qb, ++k) {
                    if (k % kSolvers != warp) continue;
                    const int pb = NP - 1 - (w - qb);
                    if (pb + 1 < NP) wait_ge(&ss.sflag[pb + 1][qb], 1);
                    if (qb >= 1) wait_ge(&ss.sflag[pb][qb - 1], 1);
                    wait_ge(&ss.dcnt[pb][qb], max(0, w - 1 - wmin_of(pb, qb)));
""" + body + """                    post(&ss.sflag[pb][qb], 1);
                }
            }
        } else {
            const int nw = kWarps - kSolvers, me = warp - kSolvers;
            int k = 0;
            for (int wp = 0; wp + 2 < nd; ++wp)
                for (int r = 0; r < NP; ++r) {
                    const int base = NP - 1 - r;  // anti-diagonal of (r, t) = base + t
                    for (int t = max(0, wp + 2 - base); t < NQ; ++t) {
                        if (wp < wmin_of(r, t)) continue;  // (r, t) receives nothing from wp
                        if (k++ % nw != me) continue;
                        if (wp >= t) wait_ge(&ss.sflag[NP - 1 - wp + t][t], 1);
                        if (wp >= base) wait_ge(&ss.sflag[r][wp - base], 1);
                        wait_ge(&ss.dcnt[r][t], wp - wmin_of(r, t));
                        upd(wp, r, t);
                        post(&ss.dcnt[r][t], wp - wmin_of(r, t) + 1);
                    }
                }
        }
        __syncthreads();
        PROF_ADD(2, t_0);
    } else {
""" + "\n".join(("    " + l) if l.strip() else l for l in old_loop.split("\n")) + """    }
"""
s = s[:a] + new_loop + s[b:]
# flags zeroed with the initial norms
rep("""        if (lane == 0) {
            const xf x = xf_from(v);
            ss.xm[pb][qb] = x.m;
            ss.xe[pb][qb] = x.e;
            ss.gx[pb][qb] = 0;
        }""", """        if (lane == 0) {
            const xf x = xf_from(v);
            ss.xm[pb][qb] = x.m;
            ss.xe[pb][qb] = x.e;
            ss.gx[pb][qb] = 0;
            ss.sflag[pb][qb] = 0;
            ss.dcnt[pb][qb] = 0;
        }""")
open(p, 'w').write(s)
print("patched")
