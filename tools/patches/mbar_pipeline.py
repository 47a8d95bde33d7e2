"""Development patch (applied once, kept for the record): decoupled update pipeline with stage
mbarriers (cp.async + per-thread asynchronous arrivals), operand pre-scale on fragments, thread
0's state in shared memory, chunk refill after compute."""
import re, sys
p = sys.argv[1]
s = open(p).read()
def rep(old, new, cnt=1):
    global s
    assert s.count(old) == cnt, (old[:90], s.count(old))
    s = s.replace(old, new)

rep("""__device__ __forceinline__ int ld_acquire(const int* p) {""", """// mbarrier (CTA scope): arrive has release, try_wait acquire semantics
__device__ __forceinline__ void mbar_init(unsigned long long* b, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\\n" ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_inval(unsigned long long* b) {
    asm volatile("mbarrier.inval.shared::cta.b64 [%0];\\n" ::"r"((unsigned)__cvta_generic_to_shared(b)) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\\n" ::"r"((unsigned)__cvta_generic_to_shared(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, int parity) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(b);
    asm volatile(
        "{\\n .reg .pred p;\\n"
        "W_%=:\\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\\n"
        " @!p bra W_%=;\\n}\\n" ::"r"(a), "r"(parity) : "memory");
}
// cp.async completion of this thread's earlier copies counted as one arrival on b
__device__ __forceinline__ void cp_async_arrive(unsigned long long* b) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\\n" ::"r"(
                     (unsigned)__cvta_generic_to_shared(b)) : "memory");
}

__device__ __forceinline__ int ld_acquire(const int* p) {""")

# structs
a = s.index("struct SrcCursor {")
b = s.index("};", a) + 3
cursor = s[a:b]
s = s[:a] + s[b:]
rep("""struct USmem {""", cursor + """
// Thread 0's per-tile header state (running bound, exponents, frame, lookahead cursor): kept in
// shared memory so that the other 511 threads do not carry it in registers.
struct T0 {
    SrcCursor la;
    int la_has, la_st, la_seq, la_pre;
    int E, F, nev, e_d0;
    xq bound, q_omega, q_target;
};

struct USmem {""")
rep("""    int pre[2];  // lookahead published for the next issue call (parity slots, thread 0 writes)""",
    """    int ready_src;  // highest source (per-tile sequence number) whose flag thread 0 saw set
    T0 t0;""")

# fragment-level chunk GEMM
rep("""// Update phase of a tile task: one CTA accumulates""", """// One kKC-deep K chunk of the update GEMM on DMMA for a warp's 32 x 32 accumulator block; the
// fragments of k-step kk + 4 are loaded while the DMMAs of kk issue. kScale: the chunk header's
// exact power-of-two operand pre-scale (robust_update.cpp:46-57 in exponent form) applied to
// the fragments as they are loaded.
template <bool kScale>
__device__ __forceinline__ void mma_chunk(const double (*As)[kLDA], const double (*Bs)[kLDB],
                                          const UHdr& h, double (&acc)[4][4][2], int wm, int wn,
                                          int g, int q) {
    auto ldA = [&](int k, int mi) {
        double v = -As[k][wm * 32 + mi * 8 + g];
        if (kScale && h.sa) {
            v *= h.fa1;
            if (h.sa == 2) v *= h.fa2;
        }
        return v;
    };
    auto ldB = [&](int k, int ni) {
        double v = Bs[wn * 32 + ni * 8 + g][k];
        if (kScale && h.sb) {
            v *= h.fb1;
            if (h.sb == 2) v *= h.fb2;
        }
        return v;
    };
    double a[2][4], b[2][4];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi) a[0][mi] = ldA(q, mi);
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) b[0][ni] = ldB(q, ni);
#pragma unroll
    for (int kk = 0; kk < kKC; kk += 4) {
        const int cb = (kk >> 2) & 1;
        if (kk + 4 < kKC) {
#pragma unroll
            for (int mi = 0; mi < 4; ++mi) a[cb ^ 1][mi] = ldA(kk + 4 + q, mi);
#pragma unroll
            for (int ni = 0; ni < 4; ++ni) b[cb ^ 1][ni] = ldB(kk + 4 + q, ni);
        }
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
            for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni], a[cb][mi], b[cb][ni]);
    }
}

// Update phase of a tile task: one CTA accumulates""")

# thread-0 state -> z (update_phase body only)
a = s.index("__device__ void update_phase(")
b = s.index("// Solve phase: RobustSyl")
body = s[a:b]
names = ['la', 'la_has', 'la_st', 'E', 'F', 'nev', 'bound', 'q_omega', 'q_target', 'e_d0']
out = []
for line in body.split('\n'):
    code, sep, com = line.partition('//')
    for n in names:
        code = re.sub(r'(?<![\w.])' + n + r'\b', 'z.' + n, code)
    out.append(code + sep + com)
body = '\n'.join(out)
fixes = [
("""    const int z.e_d0 = P.yexp[i * N + j];
    int z.E = 0;
    // integer bounds in the per-source header (see struct xq)
    xq z.bound = xq_from(P.ynorm[i * N + j]);
    const xq z.q_omega = xq_from_down(P.omega), z.q_target = xq_from_down(P.omega * (1.0 - 0x1p-30));
    int z.nev = 0;""",
"""    T0& z = sm.t0;  // thread 0's header and lookahead state
    if (tid == 0) {
        z.e_d0 = P.yexp[i * N + j];
        z.E = 0;
        z.bound = xq_from(P.ynorm[i * N + j]);  // integer bounds in the header (struct xq)
        z.q_omega = xq_from_down(P.omega);
        z.q_target = xq_from_down(P.omega * (1.0 - 0x1p-30));
        z.nev = 0;
        z.F = 0;
    }"""),
("    int z.F = 0;\n", ""),
("""    SrcCursor z.la = cur;
    bool z.la_has = false;
    int z.la_st = 0;  // 0: poll flag, 1: poll in flight, 2: metadata in flight, 3: published
    int la_flag = 0, la_esrc = 0, la_s = 0;""",
"""    if (tid == 0) {
        z.la = cur;
        z.la_has = false;
        z.la_st = 0;  // 0: poll flag, 1: poll in flight, 2: metadata in flight, 3: published
        z.la_seq = 0;
        z.la_pre = false;
    }
    int la_flag = 0, la_esrc = 0, la_s = 0;  // (registers: loads in flight across calls)"""),
("""    int ncall = 0;""", """    int nsrc = -1;  // sequence number of the current source (every thread)"""),
("""        const int call = ncall++;
        bool fresh = false;""", """        bool fresh = false;"""),
("""            cur.chunk = 0;
            fresh = true;
            // CTA-uniform: published by thread 0 before the last barrier
            const bool pre = call >= kStages - 1 && sm.pre[call & 1] != 0;
            PROF_T0(t_w);
            if (kWaitFlags && !RSYLV_EXPERIMENT_NOWAIT && !pre) {
                if (tid == 0) {""",
"""            cur.chunk = 0;
            fresh = true;
            ++nsrc;
            // The source must be published before this warp's copies read it: thread 0 records
            // in sm.ready_src every flag its lookahead saw set; otherwise lane 0 spins on the flag
            // itself (no CTA barrier: the warps run decoupled through the stage mbarriers).
            const bool pre = tid == 0 && z.la_pre;
            PROF_T0(t_w);
            if (kWaitFlags && !RSYLV_EXPERIMENT_NOWAIT) {
                if (lane == 0 && !pre && *((volatile int*)&sm.ready_src) < nsrc) {"""),
("""                        __nanosleep(128);
                    }
                }
                __syncthreads();
            }
            PROF_ADD(9, t_w);   // source-ready wait (spin + barrier)""",
"""                        __nanosleep(128);
                    }
                }
                __syncwarp();
            }
            PROF_ADD(9, t_w);   // source-ready wait"""),
("""                z.la = cur;
                z.la_has = next_src(z.la, i, j, M);
                z.la_st = 0;
            }""", """                z.la = cur;
                z.la_has = next_src(z.la, i, j, M);
                z.la_seq = nsrc + 1;
                z.la_st = 0;
                z.la_pre = false;
            }"""),
("""                } else if (z.la_st == 1) {
                    if (la_flag != 0) {
                        la_meta();""", """                } else if (z.la_st == 1) {
                    if (la_flag != 0) {
                        *((volatile int*)&sm.ready_src) = z.la_seq;
                        la_meta();"""),
("""                } else if (z.la_st == 2) {
                    z.la_st = 3;  // metadata loads issued >= 1 call before they are consumed
                }
            }
            if (call >= kStages - 2) sm.pre[(call + 1) & 1] = (z.la_has && z.la_st == 3) ? 1 : 0;
        }
        if (tid == 0) {
            sm.hdr[stage] = sm.cur;
            if (!fresh) sm.hdr[stage].acc_shift = 0;
        }""", """                } else if (z.la_st == 2) {
                    z.la_st = 3;  // metadata loads issued >= 1 call before they are consumed
                    z.la_pre = true;
                }
            }
        }"""),
("""            cp_async16(&sm.B[stage][col][k2], cur.R + (k0 + k2) + (long long)col * TSP);
        }
        ++cur.chunk;""", """            cp_async16(&sm.B[stage][col][k2], cur.R + (k0 + k2) + (long long)col * TSP);
        }
        // the stage's full barrier completes when every thread's copies landed (asynchronous
        // arrivals) and thread 0 published the stage header (release)
        cp_async_arrive(&sfull[stage]);
        if (tid == 0) {
            sm.hdr[stage] = sm.cur;
            if (!fresh) sm.hdr[stage].acc_shift = 0;
            mbar_arrive(&sfull[stage]);
        }
        ++cur.chunk;"""),
("""    E_out = z.E;
    bound_out = xq_to_xf(z.bound);
    nev_out = z.nev;
    (void)z.e_d0;""", """    __syncthreads();  // every warp is done with the stage barriers
    if (tid == 0)
        for (int s = 0; s < kStages; ++s) {
            mbar_inval(&sfull[s]);
            mbar_inval(&sempty[s]);
        }
    E_out = z.E;
    bound_out = xq_to_xf(z.bound);
    nev_out = z.nev;"""),
("""    const int M = P.M, N = P.N, TSP = P.TSP;
    const double* Yd = y_slot(P, i, j);
""", """    const int M = P.M, N = P.N, TSP = P.TSP;
    const double* Yd = y_slot(P, i, j);
    // stage barriers (static shared memory: the solve phase reuses the dynamic buffers)
    __shared__ __align__(8) unsigned long long sfull[kStages], sempty[kStages];
    if (tid == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&sfull[s], kThreads + 1);  // one async arrival per thread + the header
            mbar_init(&sempty[s], kWarps);
        }
        sm.ready_src = -1;
    }
    __syncthreads();
"""),
]
for o, n in fixes:
    assert o in body, o[:70]
    body = body.replace(o, n)
# main loop
a2 = body.index("    int loaded = 0;")
b2 = body.index("    if (nchunks > 0) {  // back to the frame")
body = body[:a2] + """    int loaded = 0;
#pragma unroll 1
    for (int s = 0; s < kStages - 1; ++s) {
        if (loaded < nchunks) {
            issue(loaded % kStages);
            ++loaded;
        }
    }

    // Main loop. The warps run decoupled: a stage's full barrier completes when its copies
    // landed and its header is published, its empty barrier when all 16 warps finished reading
    // it. After computing chunk it, a warp refills the stage chunk it - 1 used (once everyone
    // released it) with chunk it + kStages - 1. There is no CTA-wide barrier per chunk: a late
    // warp (thread 0's header, a busy SM sub-partition) holds the others back only when it falls
    // a whole chunk behind. The L2 prefetch of the next source (la_prefetch) keeps the copies'
    // latency short even though they are issued only one chunk ahead.
#pragma unroll 1
    for (int it = 0; it < nchunks; ++it) {
        const int st = it % kStages;
        mbar_wait(&sfull[st], (it / kStages) & 1);
        const UHdr h = sm.hdr[st];
#ifdef RSYLV_PROFILE
        if (tid == 0) {
            atomicAdd(&g_prof[10], 1ull);
            if (h.live && (h.sa | h.sb)) atomicAdd(&g_prof[11], 1ull);
        }
#endif
        if (h.acc_shift != 0) {
#pragma unroll
            for (int mi = 0; mi < 4; ++mi)
#pragma unroll
                for (int ni = 0; ni < 4; ++ni) {
                    acc[mi][ni][0] = scale2(acc[mi][ni][0], h.acc_shift);
                    acc[mi][ni][1] = scale2(acc[mi][ni][1], h.acc_shift);
                }
        }
        if (h.live) {
            if (!RSYLV_EXPERIMENT_NOPRESCALE && (h.sa | h.sb))
                mma_chunk<true>(sm.A[st], sm.B[st], h, acc, wm, wn, g, q);
            else
                mma_chunk<false>(sm.A[st], sm.B[st], h, acc, wm, wn, g, q);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&sempty[st]);
        if (loaded < nchunks) {
            const int s2 = loaded % kStages;
            if (loaded >= kStages) mbar_wait(&sempty[s2], ((loaded - kStages) / kStages) & 1);
            issue(s2);
            ++loaded;
        }
    }
""" + body[b2:]
body = body.replace("""    cp_async_wait<0>();
    if (nchunks > 0) {  // back to the frame""", """    if (nchunks > 0) {  // back to the frame""")
s = s[:a] + body + s[b:]
open(p, 'w').write(s)
print("patched")
