"""Development patch: the per-source header and the lookahead rotate over the warps."""
import sys
p = sys.argv[1]
s = open(p).read()
a = s.index("    // Lookahead (thread 0 only): while the chunks of `cur` stream")
b = s.index("    int loaded = 0;")
new = r'''    // Per-source duties rotate over the warps (lane 0 of warp nsrc % 16): that thread computes
    // the source's header (exponent-form ProtectUpdate on integer bounds, frame, pre-scale) and
    // publishes the header of each of its chunks; lane 0 of the NEXT source's warp runs the
    // lookahead during this source's later chunks: it polls the next source's ready flag
    // (relaxed load, consumed one call later), then issues the loads of its norms and exponents
    // and the L2 prefetch of its two tile slots. With the warps decoupled, each warp carries
    // 1/16 of this serial single-thread work instead of warp 0 carrying all of it.
    // Ordering: the producer releases a flag after its tile and metadata reached L2
    // (st.release); every read here is an L2 read (.cg / cp.async.cg) issued after the flag
    // value was observed. The shared running state (z.E, z.F, z.bound, z.nev) passes from one
    // duty thread to the next through the stage barriers (a duty's writes precede its empty
    // arrival for an earlier chunk, which the next duty's refill waited on).
    int la_flag = 0, la_esrc = 0, la_s = 0;  // (registers: loads in flight across calls)
    double la_nl = 0.0, la_nr = 0.0;
    int la_st = 0;         // lookahead state of this lane: 0 idle, 1 poll in flight, 2 meta in flight
    bool la_pre = false;   // this lane holds the metadata of the source it will head
    int nsrc = -1;         // sequence number of the current source (every thread)
    SrcCursor& la = sm.la[warp];  // lookahead cursor of this warp's lane 0
    UHdr& hc = sm.cur[warp];      // header of the source this warp's lane 0 heads
    auto la_meta = [&]() {
        // the static operand's stored (normalized) norm and exponent enter as
        // norm * 2^-s and esrc - s: the product bound is unchanged
        if (la.kind == 0) {
            la_nl = ld_cg_pin(&P.anorm[i * M + la.idx]);
            la_nr = ld_cg_pin(&P.ynorm[la.idx * N + j]);
            la_esrc = ld_cg_pin(&P.yexp[la.idx * N + j]);
            la_s = ld_cg_pin(&P.aexp[i * M + la.idx]);
        } else {
            la_nl = ld_cg_pin(&P.ynorm[i * N + la.idx]);
            la_nr = ld_cg_pin(&P.bnorm[la.idx * N + j]);
            la_esrc = ld_cg_pin(&P.yexp[i * N + la.idx]);
            la_s = ld_cg_pin(&P.bexp[la.idx * N + j]);
        }
    };
    // the next source's two tile slots into L2 while the current source streams
    auto la_prefetch = [&]() {
        if (!RSYLV_L2_PREFETCH) return;
        const long long slot = (long long)TSP * TSP;
        const double* L = la.kind == 0 ? a_slot(P, i, la.idx) : y_slot(P, i, la.idx);
        const double* R = la.kind == 0 ? y_slot(P, la.idx, j) : b_slot(P, la.idx, j);
        prefetch_l2(L, (unsigned)(slot * 8));
        prefetch_l2(R, (unsigned)(slot * 8));
    };
    auto la_poll = [&]() {
        la_flag = ld_relaxed(la.kind == 0 ? &P.state[la.idx * N + j] : &P.state[i * N + la.idx],
                             P.sys_scope != 0);
    };

    auto issue = [&](int stage) {
        bool fresh = false;
        if (cur.chunk == cur.nch) {
            next_src(cur, i, j, M);
            if (cur.kind == 0) {
                const int k = cur.idx;
                cur.nch = (P.rcut[k + 1] - P.rcut[k] + kKC - 1) / kKC;
            } else {
                const int l = cur.idx;
                cur.nch = (P.ccut[l + 1] - P.ccut[l] + kKC - 1) / kKC;
            }
            cur.chunk = 0;
            fresh = true;
            ++nsrc;
        }
        const bool duty = lane == 0 && warp == (nsrc & (kWarps - 1));
        const bool nduty = lane == 0 && warp == ((nsrc + 1) & (kWarps - 1));
        if (fresh) {
            // The source must be published before this warp's copies read it: the lookahead
            // thread records in sm.ready_src every flag it saw set; otherwise lane 0 spins on
            // the flag itself (no CTA barrier).
            const bool pre = duty && la_pre;
            PROF_T0(t_w);
            if (kWaitFlags && !RSYLV_EXPERIMENT_NOWAIT) {
                if (lane == 0 && !pre && *((volatile int*)&sm.ready_src) < nsrc) {
                    const int* flag = cur.kind == 0 ? &P.state[cur.idx * N + j]
                                                    : &P.state[i * N + cur.idx];
                    const unsigned long long t_start = globaltimer_ns();
                    while ((P.sys_scope ? ld_acquire_sys(flag) : ld_acquire(flag)) == 0) {
                        if (aborted(P, tile_pri(P, i, j))) break;
                        if (globaltimer_ns() - t_start > kWatchdogNs) {  // never hang the GPU
                            set_error(P, kErrWatchdog, 0.0);
                            break;
                        }
                        __nanosleep(128);
                    }
                }
                __syncwarp();
            }
            PROF_ADD(9, t_w);   // source-ready wait
            if (duty) {
                if (!pre) {
                    la = cur;
                    la_meta();
                }
                const xq nl = la.kind == 0 ? xq_shift(xq_from(la_nl), -la_s) : xq_from(la_nl);
                const xq nr = la.kind == 0 ? xq_from(la_nr) : xq_shift(xq_from(la_nr), -la_s);
                const int esrc = la_esrc - la_s;
                xq term = xq_shift(xq_mul(nl, nr), (z.e_d0 + z.E) - esrc);
                xq gsum = xq_add(z.bound, term);
                const int d = xq_guard(gsum, z.q_omega, z.q_target);
                if (d > 0) {
                    z.E -= d;
                    gsum = xq_shift(gsum, -d);
                    ++z.nev;
                }
                z.bound = gsum;
                const int p = (z.e_d0 + z.E) - esrc;
                const int Fn = gsum.m ? min(max(p, gsum.e - 1022), gsum.e + 900) : z.F;
                int pa, pb;
                const bool live = split_prescale(p - Fn, nl.m != 0, nl.e, nr.m != 0, nr.e, pa, pb);
                hc.acc_shift = -d + (z.F - Fn);
                hc.frame = Fn;
                z.F = Fn;
                hc.live = live;
                hc.sa = p2_factors(pa, hc.fa1, hc.fa2);
                hc.sb = p2_factors(pb, hc.fb1, hc.fb2);
                la_pre = false;
                la_st = 0;
            }
            PROF_ADD(13, t_w);  // source header
        }
        // lookahead for the next source, from this source's third chunk on (by then the
        // previous duty's shared-state writes are ordered before this call: see above)
        if (nduty && cur.chunk >= 2 && !la_pre) {
            if (la_st == 0) {
                la = cur;
                if (next_src(la, i, j, M)) {
                    if (kWaitFlags) {
                        la_poll();
                        la_st = 1;
                    } else {
                        la_meta();
                        la_prefetch();
                        la_pre = true;
                    }
                } else {
                    la_st = 3;  // no next source
                }
            } else if (la_st == 1) {
                if (la_flag != 0) {
                    *((volatile int*)&sm.ready_src) = nsrc + 1;
                    la_meta();  // consumed at the next source's first call, a chunk later
                    la_prefetch();
                    la_pre = true;
                } else {
                    la_poll();
                }
            }
        }
        const int k0 = cur.chunk * kKC;
        // the source's two slots (recomputed per call: fewer registers live across the loop)
        const double* cL = cur.kind == 0 ? a_slot(P, i, cur.idx) : y_slot(P, i, cur.idx);
        const double* cR = cur.kind == 0 ? y_slot(P, cur.idx, j) : b_slot(P, cur.idx, j);
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const int cidx = tid + t * kThreads;
            const int kk = cidx >> 6, r2 = (cidx & 63) * 2;
            cp_async16(&sm.A[stage][kk][r2], cL + r2 + (long long)(k0 + kk) * TSP);
        }
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const int cidx = tid + t * kThreads;
            const int col = cidx >> 4, k2 = (cidx & 15) * 2;
            cp_async16(&sm.B[stage][col][k2], cR + (k0 + k2) + (long long)col * TSP);
        }
        // the stage's full barrier completes when every thread's copies landed (asynchronous
        // arrivals) and the source's duty thread published the stage header (release)
        cp_async_arrive(&sfull[stage]);
        if (duty) {
            sm.hdr[stage] = hc;
            if (!fresh) sm.hdr[stage].acc_shift = 0;
            mbar_arrive(&sfull[stage]);
        }
        ++cur.chunk;
    };

'''
s = s[:a] + new + s[b:]
def rep(old, new, cnt=1):
    global s
    assert s.count(old) == cnt, (old[:90], s.count(old))
    s = s.replace(old, new)
rep("""    UHdr cur;    // header of the current source (thread 0 writes)
    int ready_src;  // highest source (per-tile sequence number) whose flag thread 0 saw set
    T0 t0;""", """    UHdr cur[kWarps];       // header of the source each warp's lane 0 heads
    SrcCursor la[kWarps];   // lookahead cursor of each warp's lane 0
    int ready_src;  // highest source (per-tile sequence number) whose flag a lookahead saw set
    T0 t0;""")
rep("""struct T0 {
    SrcCursor la;
    int la_has, la_st, la_seq, la_pre;
    int E, F, nev, e_d0;""", """struct T0 {
    int E, F, nev, e_d0;""")
rep("""// Thread 0's per-tile header state (running bound, exponents, frame, lookahead cursor): kept in
// shared memory so that the other 511 threads do not carry it in registers.""", """// The per-tile running header state (bound, exponents, frame), handed from one source's duty
// thread to the next through shared memory.""")
rep("""    T0& z = sm.t0;  // thread 0's header and lookahead state""", """    T0& z = sm.t0;  // running header state (written by the duty threads)""")
open(p, 'w').write(s)
print("patched")
