"""Development patch: solved Y tiles stored normalized (norm in [2^-9, 2^-8)) with a per-tile
storage exponent yst, like the off-diagonal A/B source tiles."""
import sys
root = sys.argv[1]
def patch(path, pairs):
    s = open(path).read()
    for old, new in pairs:
        assert s.count(old) == 1, (path, old[:90], s.count(old))
        s = s.replace(old, new)
    open(path, 'w').write(s)

patch(root + '/common.cuh', [
("""    int* yexp;                  // M*N tile exponent (scale = 2^yexp, yexp <= 0)""",
 """    int* yexp;                  // M*N tile exponent (scale = 2^yexp, yexp <= 0)
    int* yst;                   // M*N (= yexp + M*N): a solved tile is stored as Y_ij * 2^-yst,
                                // normalized like the A/B sources (norm in [2^-9, 2^-8))"""),
])
K = root + '/kernels.cu'
patch(K, [
# header: the Y operand's storage exponent
("""    int la_flag = 0, la_esrc = 0, la_s = 0;  // (registers: loads in flight across calls)""",
 """    int la_flag = 0, la_esrc = 0, la_s = 0, la_t = 0;  // (registers: loads in flight)"""),
("""            la_esrc = ld_cg_pin(&P.yexp[la.idx * N + j]);
            la_s = ld_cg_pin(&P.aexp[i * M + la.idx]);""",
 """            la_esrc = ld_cg_pin(&P.yexp[la.idx * N + j]);
            la_s = ld_cg_pin(&P.aexp[i * M + la.idx]);
            la_t = ld_cg_pin(&P.yst[la.idx * N + j]);"""),
("""            la_esrc = ld_cg_pin(&P.yexp[i * N + la.idx]);
            la_s = ld_cg_pin(&P.bexp[la.idx * N + j]);""",
 """            la_esrc = ld_cg_pin(&P.yexp[i * N + la.idx]);
            la_s = ld_cg_pin(&P.bexp[la.idx * N + j]);
            la_t = ld_cg_pin(&P.yst[i * N + la.idx]);"""),
("""                const xq nl = la.kind == 0 ? xq_shift(xq_from(la_nl), -la_s) : xq_from(la_nl);
                const xq nr = la.kind == 0 ? xq_from(la_nr) : xq_shift(xq_from(la_nr), -la_s);
                const int esrc = la_esrc - la_s;""",
 """                // norms of the operands as stored: the static one carries 2^-aexp / 2^-bexp,
                // the solved Y tile 2^-yst
                const int sl = la.kind == 0 ? la_s : la_t, sr = la.kind == 0 ? la_t : la_s;
                const xq nl = xq_shift(xq_from(la_nl), -sl);
                const xq nr = xq_shift(xq_from(la_nr), -sr);
                const int esrc = la_esrc - la_s - la_t;"""),
# pack: storage exponent of C tiles is 0
("""    if (threadIdx.x == 0) {
        yexp[t] = 0;
        uexp[t] = 0;""", """    if (threadIdx.x == 0) {
        yexp[t] = 0;
        yexp[t + M * N] = 0;  // yst
        uexp[t] = 0;"""),
# finalize: normalized write-back + yst
("""    const int dfin = ss.dfin;
    // write back (full 128 x 128 slot, padding stays zero), scaled by 2^-dfin if needed
    for (int e = tid; e < kBM * kBM; e += kThreads) {
        const int r = e & (kBM - 1), c = e >> 7;
        double v = ss.T[r + c * kLDT];
        if (dfin) v = scale2(v, -dfin);
        __stcg(Yg + r + (long long)c * TSP, v);
    }""", """    const int dfin = ss.dfin;
    // write back (full 128 x 128 slot, padding stays zero), normalized: the tile at rest is
    // T * 2^-dfin (norm tn * 2^-dfin <= omega) and its slot holds that times 2^-yst with
    // yst = e(tn) - dfin + 8, i.e. T * 2^-(e(tn) + 8), norm in [2^-9, 2^-8). Sources then enter
    // the update GEMM at a common scale and the accumulator frame absorbs the relative exponent
    // (no operand pre-scale); only entries below 2^-1065 of the tile norm round.
    const int wsh = ss.redm[0] != 0.0 ? ss.rede[0] + 8 : dfin;
    for (int e = tid; e < kBM * kBM; e += kThreads) {
        const int r = e & (kBM - 1), c = e >> 7;
        double v = ss.T[r + c * kLDT];
        if (wsh) v = scale2(v, -wsh);
        __stcg(Yg + r + (long long)c * TSP, v);
    }"""),
("""            P.yexp[i * N + j] = e_out;
            P.ynorm[i * N + j] = xf_to_double(tnorm);""", """            P.yexp[i * N + j] = e_out;
            P.yst[i * N + j] = wsh - dfin;
            P.ynorm[i * N + j] = xf_to_double(tnorm);"""),
("""    if (P.nranks > 1 && !ss.failed) push_tile(P, i, j, ss.gmin, ss.redm[0]);""",
 """    if (P.nranks > 1 && !ss.failed) push_tile(P, i, j, ss.gmin, wsh - dfin, ss.redm[0]);"""),
("""__device__ void push_tile(const Problem& P, int i, int j, int e_out, double nrm) {""",
 """__device__ void push_tile(const Problem& P, int i, int j, int e_out, int yst, double nrm) {"""),
("""            P.peerYexp[r][i * N + j] = e_out;""", """            P.peerYexp[r][i * N + j] = e_out;
            P.peerYexp[r][i * N + j + P.M * N] = yst;  // the peer's yst (second half of yexp)"""),
# unpack
("""    const int f = alpha_exp - yexp[t];""", """    const int f = alpha_exp - yexp[t] + yexp[t + (long long)gridDim.x];  // + yst"""),
])
R = root + '/runtime.cpp'
patch(R, [
("""        B.yexp = buf<int>(ctx, ("yexp" + sfx).c_str(), ny);""",
 """        B.yexp = buf<int>(ctx, ("yexp" + sfx).c_str(), 2 * ny);  // yexp, then yst"""),
("""        Q.ynorm = B.ynorm;
        Q.yexp = B.yexp;
        Q.uexp = B.uexp;
        Q.state = B.state;""", """        Q.ynorm = B.ynorm;
        Q.yexp = B.yexp;
        Q.yst = B.yexp + ny;
        Q.uexp = B.uexp;
        Q.state = B.state;"""),
("""    Q.ynorm = B.ynorm;
    Q.yexp = B.yexp;
    Q.uexp = B.uexp;
    Q.ubnd = B.ubnd;""", """    Q.ynorm = B.ynorm;
    Q.yexp = B.yexp;
    Q.yst = B.yexp + (size_t)Q.M * Q.N;
    Q.uexp = B.uexp;
    Q.ubnd = B.ubnd;"""),
("""        int* ye = buf<int>(ctx, "ruye", 2);""", """        int* ye = buf<int>(ctx, "ruye", 4);  // yexp, then yst"""),
("""        P.yexp = ye;""", """        P.yexp = ye;
        P.yst = ye + 2;"""),
])
print("patched")
