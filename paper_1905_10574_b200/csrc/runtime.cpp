// rsylv-b200 host runtime: the C-ABI of include/rsylv_b200.h.
//
// Host-side orchestration of the tiled robust solve (reference: tiled_solve.cpp:183-194 and
// the TileGrid of tile_grid.cpp): argument validation in the reference's order, tile
// partitioning, device workspace management, kernel launches (persistent dataflow scheduler or
// host-driven wavefront), the alpha reduction (tile_grid.cpp:38-42) and the final verdict.
#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <functional>
#include <map>
#include <string>
#include <vector>

#include "../../include/rsylv_b200.h"
#include "launch.h"

using namespace rsb;

namespace {

struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
};

}  // namespace

struct rsylv_b200_ctx {
    int device = 0;
    int sms = 0;
    cudaStream_t own_stream = nullptr;
    std::map<std::string, DevBuf> bufs;
    std::string last_error;
    bool configured = false;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr, evp = nullptr, evd = nullptr;
    cudaStream_t side_stream = nullptr;                  // host pipeline: pack + validation
    cudaStream_t copy_stream = nullptr;                  // host pipeline: H2D copies (back to back)
    cudaEvent_t ev_side0 = nullptr, ev_side = nullptr;
    std::vector<cudaEvent_t> ev_shell;                   // host pipeline: shell t's copies landed
    struct rsylv_b200_plan_holder* holder = nullptr;
};

namespace {

struct Fail {
    int status;
};

void ck(rsylv_b200_ctx* ctx, cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        ctx->last_error = std::string(what) + ": " + cudaGetErrorString(e);
        throw Fail{RSYLV_CUDA_ERROR};
    }
}

template <class T>
T* buf(rsylv_b200_ctx* ctx, const char* name, size_t count) {
    DevBuf& b = ctx->bufs[name];
    const size_t bytes = count * sizeof(T) + 256;
    if (b.cap < bytes) {
        if (b.p) cudaFree(b.p);
        b.p = nullptr;
        b.cap = 0;
        ck(ctx, cudaMalloc(&b.p, bytes), name);
        b.cap = bytes;
    }
    return static_cast<T*>(b.p);
}

// TMA tensor maps of the update GEMM's operand ring (kernels.cu USmem). A slot array (column-
// major 128 x 128 slots, `nslots` of them) is viewed as a 3-D tensor: dim0 = 8 consecutive rows
// (8 B stride), dim1 = column over all slots (1 KB stride), dim2 = row group of 8 (64 B stride).
// An L operand chunk (128 rows x kKC k) is the box {8, kKC, 16} at (0, slot*128 + k0, 0), an R
// operand chunk (kKC k x 128 columns) the box {8, 128, kKC/8} at (0, slot*128, k0/8); both land
// in shared memory with SWIZZLE_64B, which makes every DMMA fragment load conflict-free.
// cuTensorMapEncodeTiled is resolved through the runtime (no link against libcuda).
typedef CUresult (*TmapEncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                 const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                 const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                 CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

void encode_slot_map(rsylv_b200_ctx* ctx, CUtensorMap* map, const double* base, size_t nslots,
                     bool as_left) {
    static TmapEncodeFn enc = nullptr;
    if (!enc) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        ck(ctx, cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q),
           "cuTensorMapEncodeTiled entry point");
        if (q != cudaDriverEntryPointSuccess || !fn) {
            ctx->last_error = "cuTensorMapEncodeTiled not available in this driver";
            throw Fail{RSYLV_CUDA_ERROR};
        }
        enc = reinterpret_cast<TmapEncodeFn>(fn);
    }
    const cuuint64_t dims[3] = {8, (cuuint64_t)std::max<size_t>(nslots, 1) * kBM, kBM / 8};
    const cuuint64_t strides[2] = {(cuuint64_t)kBM * 8, 64};
    const cuuint32_t box[3] = {8, (cuuint32_t)(as_left ? kKC : kBM),
                               (cuuint32_t)(as_left ? kBM / 8 : kKC / 8)};
    const cuuint32_t es[3] = {1, 1, 1};
    const CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims,
                           strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        ctx->last_error = "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")";
        throw Fail{RSYLV_CUDA_ERROR};
    }
}

// the four maps of one rank's Problem, copied to the device buffer `name`
const CUtensorMap* make_tmaps(rsylv_b200_ctx* ctx, const char* name, const double* Ap, size_t na,
                              const double* Bp, size_t nb, const double* Yp, size_t ny,
                              cudaStream_t st) {
    CUtensorMap h[4];
    encode_slot_map(ctx, &h[0], Ap, na, true);
    encode_slot_map(ctx, &h[1], Yp, ny, true);
    encode_slot_map(ctx, &h[2], Yp, ny, false);
    encode_slot_map(ctx, &h[3], Bp, nb, false);
    CUtensorMap* d = buf<CUtensorMap>(ctx, name, 4);
    ck(ctx, cudaMemcpyAsync(d, h, sizeof(h), cudaMemcpyHostToDevice, st), "tmaps h2d");
    ck(ctx, cudaStreamSynchronize(st), "sync");  // h goes out of scope
    return d;
}

// Tile partition: cut at running multiples of ts; a cut that would split a 2x2 block moves
// one index EARLIER (the reference moves it later, partition.cpp:74-91; Y/alpha does not depend
// on the partition and earlier cuts keep every tile within one padded slot).
std::vector<int> partition(const unsigned char* blk, size_t n, size_t ts) {
    std::vector<int> cuts{0};
    size_t pos = 0;
    while (pos < n) {
        size_t nx = pos + ts;
        if (nx >= n)
            nx = n;
        else if (blk && blk[nx - 1] == 2)
            --nx;
        cuts.push_back((int)nx);
        pos = nx;
    }
    return cuts;
}

xf host_xf(double v) { return xf_from(v); }

struct SolveArgs {
    size_t m, n;
    const double *a, *b, *c;
    size_t lda, ldb, ldc;
    const unsigned char *ablk, *bblk;
    double* y;
    size_t ldy;
    rsylv_b200_options opt;
    cudaStream_t st;
    rsylv_b200_result* res;
};

std::vector<unsigned char> codes_or_ones(const unsigned char* blk, size_t n) {
    std::vector<unsigned char> v(n, 1);
    if (blk) std::memcpy(v.data(), blk, n);
    return v;
}

// Per-rank device workspace (one per GPU; several per GPU in virtual-rank mode).
struct RankBufs {
    double* Yp = nullptr;
    double* ynorm = nullptr;
    int* yexp = nullptr;
    int* uexp = nullptr;
    double* ubnd = nullptr;
    int* state = nullptr;
    int* udone = nullptr;
    int* err = nullptr;
    double* piv = nullptr;
    double* tpiv = nullptr;  // per-tile pivots of singular failures
    unsigned long long* ev = nullptr;
    int* tnext = nullptr;
    int* tasks = nullptr;
    int ntasks = 0;
    const CUtensorMap* tmaps = nullptr;  // TMA views of Apack / Ypack / Bpack for this rank
};

// Everything one solve needs between its phases (kept in the context for the dist_* calls).
struct Plan {
    int M = 0, N = 0, TSP = 0, nranks = 1;
    size_t m = 0, n = 0, ny = 0;
    double omega = 0, small_num = 0;
    std::vector<int> rc, cc;
    std::vector<int> local;        // ranks served by this process
    std::vector<RankBufs> rb;      // one per local rank
    Problem base{};
    cudaStream_t st = nullptr;
    int scheduler = 0;
    rsylv_b200_probe_event* d_probe = nullptr;
    unsigned long long probe_cap = 0;
    int* d_reason = nullptr;  // host pipeline: first failing argument check (device)
};

}  // namespace

struct rsylv_b200_plan_holder {
    Plan plan;
    std::vector<std::vector<unsigned char>> peer_handles;  // opened handle bytes per peer
    std::vector<void*> peer_ptrs;                          // 5 per peer
    bool raw_peers = false;  // peer_ptrs are plain device pointers (single-process multi-GPU)
};

namespace {

rsylv_b200_plan_holder& ctx_holder(rsylv_b200_ctx* ctx) {
    if (!ctx->holder) ctx->holder = new rsylv_b200_plan_holder();
    return *ctx->holder;
}
Plan& ctx_plan(rsylv_b200_ctx* ctx) { return ctx_holder(ctx).plan; }

void close_peers(rsylv_b200_ctx* ctx) {
    rsylv_b200_plan_holder& H = ctx_holder(ctx);
    if (!H.raw_peers)
        for (void* p : H.peer_ptrs)
            if (p) cudaIpcCloseMemHandle(p);
    H.peer_ptrs.clear();
    H.peer_handles.clear();
    H.raw_peers = false;
}

// Steps shared by every mode: partition (tile cut moved earlier around 2x2 blocks), device
// workspaces, TileGrid + compute_bounds as one pack pass, validation in the reference order
// (tile_grid.cpp:59-74, tiled_solve.cpp:74-80), per-rank task lists in anti-diagonal order.
// deferred: the host pipeline packs (and validates) the inputs itself while the DAG runs
int plan_prepare(rsylv_b200_ctx* ctx, const SolveArgs& A, int nranks, const std::vector<int>& local,
                 bool deferred = false) {
    rsylv_b200_result* res = A.res;
    Plan& PL = ctx_plan(ctx);
    const size_t m = A.m, n = A.n;
    PL.m = m;
    PL.n = n;
    PL.omega = A.opt.omega > 0 ? A.opt.omega : DBL_MAX / 2;
    PL.small_num = A.opt.small_num > 0 ? A.opt.small_num : DBL_MIN / DBL_EPSILON;
    PL.nranks = nranks;
    PL.local = local;
    PL.st = A.st;
    PL.scheduler = A.opt.scheduler;
    if (!ctx->configured) {
        ck(ctx, configure_kernels(), "configure_kernels");
        ctx->configured = true;
    }
    cudaStream_t st = A.st;
    ck(ctx, cudaEventRecord(ctx->ev0, st), "event");
    const size_t ts = A.opt.tile_size > (size_t)kTileMax ? (size_t)kTileMax : A.opt.tile_size;
    std::vector<unsigned char> ac = codes_or_ones(A.ablk, m), bc = codes_or_ones(A.bblk, n);
    PL.rc = partition(ac.data(), m, ts);
    PL.cc = partition(bc.data(), n, ts);
    const std::vector<int>& rc = PL.rc;
    const std::vector<int>& cc = PL.cc;
    const int M = (int)rc.size() - 1, N = (int)cc.size() - 1;
    int tmax = 0;
    for (int t = 0; t < M; ++t) tmax = std::max(tmax, rc[t + 1] - rc[t]);
    for (int t = 0; t < N; ++t) tmax = std::max(tmax, cc[t + 1] - cc[t]);
    const int TSP = (tmax + kBM - 1) / kBM * kBM;
    const size_t slot = (size_t)TSP * TSP;
    const size_t slack = (size_t)64 * TSP + 1024;
    const size_t na = (size_t)M * (M + 1) / 2, nb = (size_t)N * (N + 1) / 2, ny = (size_t)M * N;
    PL.M = M;
    PL.N = N;
    PL.TSP = TSP;
    PL.ny = ny;
    res->row_tiles = M;
    res->col_tiles = N;

    Problem& P = PL.base;
    P = Problem{};
    P.M = M;
    P.N = N;
    P.TSP = TSP;
    P.m = (int)m;
    P.n = (int)n;
    int* d_rc = buf<int>(ctx, "rcut", M + 1);
    int* d_cc = buf<int>(ctx, "ccut", N + 1);
    unsigned char* d_ab = buf<unsigned char>(ctx, "ablk", m);
    unsigned char* d_bb = buf<unsigned char>(ctx, "bblk", n);
    double* Ap = buf<double>(ctx, "Apack", na * slot + slack);
    double* Bp = buf<double>(ctx, "Bpack", nb * slot + slack);
    double* anorm = buf<double>(ctx, "anorm", (size_t)M * M);
    double* bnorm = buf<double>(ctx, "bnorm", (size_t)N * N);
    int* aexp = buf<int>(ctx, "aexp", (size_t)M * M);
    int* bexp = buf<int>(ctx, "bexp", (size_t)N * N);
    ck(ctx, cudaMemcpyAsync(d_rc, rc.data(), sizeof(int) * (M + 1), cudaMemcpyHostToDevice, st), "h2d");
    ck(ctx, cudaMemcpyAsync(d_cc, cc.data(), sizeof(int) * (N + 1), cudaMemcpyHostToDevice, st), "h2d");
    ck(ctx, cudaMemcpyAsync(d_ab, ac.data(), m, cudaMemcpyHostToDevice, st), "h2d");
    ck(ctx, cudaMemcpyAsync(d_bb, bc.data(), n, cudaMemcpyHostToDevice, st), "h2d");
    ck(ctx, cudaMemsetAsync(Ap + na * slot, 0, slack * sizeof(double), st), "memset");
    ck(ctx, cudaMemsetAsync(Bp + nb * slot, 0, slack * sizeof(double), st), "memset");
    P.rcut = d_rc;
    P.ccut = d_cc;
    P.ablk = d_ab;
    P.bblk = d_bb;
    P.Apack = Ap;
    P.Bpack = Bp;
    P.anorm = anorm;
    P.bnorm = bnorm;
    P.aexp = aexp;
    P.bexp = bexp;
    P.nsub_r = P.nsub_c = TSP / kBM;
    P.omega = PL.omega;
    P.small_num = PL.small_num;
    P.x_omega = host_xf(PL.omega);
    P.x_target = host_xf(PL.omega * (1.0 - 0x1p-30));
    P.nranks = nranks;
    {   // update ring refill order: early on throughput-bound DAGs (>= one tile per SM on the long
        // anti-diagonals), late on latency-bound ones (RSYLV_B200_ISSUE_EARLY=0/1 overrides)
        const char* ev = std::getenv("RSYLV_B200_ISSUE_EARLY");
        P.issue_early = ev ? (ev[0] == '1') : (std::min(M, N) >= ctx->sms ? 1 : 0);
    }
    {   // diagonal-tile solve path (RSYLV_B200_FAST_DIAG=1 opts in, for experiments)
        const char* ev = std::getenv("RSYLV_B200_FAST_DIAG");
        P.fast_solve = (A.opt.fast_diag || (ev && ev[0] == '1')) ? 1 : 0;
    }

    PL.d_reason = nullptr;
    if (deferred) {
        int* rdy = buf<int>(ctx, "inready", 4);
        PL.d_reason = buf<int>(ctx, "reason", 1);
        const int four = 4;
        ck(ctx, cudaMemsetAsync(rdy, 0, 4 * sizeof(int), st), "memset");
        ck(ctx, cudaMemcpyAsync(PL.d_reason, &four, sizeof(int), cudaMemcpyHostToDevice, st), "h2d");
        P.in_ready = rdy;
    } else {
        launch_pack_upper(A.a, (long long)A.lda, d_rc, M, TSP, Ap, anorm, aexp, st,
                          !std::isinf(PL.omega));
        launch_pack_upper(A.b, (long long)A.ldb, d_cc, N, TSP, Bp, bnorm, bexp, st,
                          !std::isinf(PL.omega));
    }

    PL.rb.assign(local.size(), RankBufs{});
    PL.d_probe = nullptr;
    for (size_t li = 0; li < local.size(); ++li) {
        const int r = local[li];
        const std::string sfx = local.size() > 1 ? "#" + std::to_string(r) : std::string();
        RankBufs& B = PL.rb[li];
        B.Yp = buf<double>(ctx, ("Ypack" + sfx).c_str(), ny * slot + slack);
        B.ynorm = buf<double>(ctx, ("ynorm" + sfx).c_str(), ny);
        B.yexp = buf<int>(ctx, ("yexp" + sfx).c_str(), 2 * ny);  // yexp, then yst
        B.uexp = buf<int>(ctx, ("uexp" + sfx).c_str(), ny);
        B.ubnd = buf<double>(ctx, ("ubnd" + sfx).c_str(), ny);
        B.state = buf<int>(ctx, ("state" + sfx).c_str(), ny);
        B.udone = buf<int>(ctx, ("udone" + sfx).c_str(), ny);
        B.err = buf<int>(ctx, ("err" + sfx).c_str(), 4);
        B.piv = buf<double>(ctx, ("pivot" + sfx).c_str(), 1);
        B.tpiv = buf<double>(ctx, ("tpivot" + sfx).c_str(), ny);
        B.ev = buf<unsigned long long>(ctx, ("events" + sfx).c_str(), 2);
        B.tnext = buf<int>(ctx, ("tnext" + sfx).c_str(), 1);
        ck(ctx, cudaMemsetAsync(B.Yp + ny * slot, 0, slack * sizeof(double), st), "memset");
        ck(ctx, cudaMemsetAsync(B.err, 0, 4 * sizeof(int), st), "memset");
        ck(ctx, cudaMemsetAsync(B.ev, 0, 2 * sizeof(unsigned long long), st), "memset");
        ck(ctx, cudaMemsetAsync(B.tnext, 0, sizeof(int), st), "memset");
        B.tmaps = make_tmaps(ctx, ("tmaps" + sfx).c_str(), Ap, na, Bp, nb, B.Yp, ny, st);
        Problem Q = P;
        Q.rank = r;  // (multi-rank: C packed for the owned tile columns only)
        Q.Ypack = B.Yp;
        Q.ynorm = B.ynorm;
        Q.yexp = B.yexp;
        Q.yst = B.yexp + ny;
        Q.uexp = B.uexp;
        Q.state = B.state;
        Q.udone = B.udone;
        if (!deferred) launch_pack_full(A.c, (long long)A.ldc, Q, B.ynorm, st);
        // task list: owned tile columns, anti-diagonal order
        std::vector<int> T;
        for (int d = 0; d <= M + N - 2; ++d) {
            const int jlo = std::max(0, d - (M - 1)), jhi = std::min(N - 1, d);
            for (int j = jlo; j <= jhi; ++j) {
                if (j % nranks != r) continue;
                T.push_back(M - 1 - d + j);
                T.push_back(j);
            }
        }
        B.ntasks = (int)T.size() / 2;
        B.tasks = buf<int>(ctx, ("tasks" + sfx).c_str(), T.size() + 2);
        if (!T.empty())
            ck(ctx, cudaMemcpyAsync(B.tasks, T.data(), sizeof(int) * T.size(), cudaMemcpyHostToDevice, st), "h2d");
        ck(ctx, cudaStreamSynchronize(st), "sync");  // T goes out of scope
    }
    PL.probe_cap = 0;
    if (res->probe_log && res->probe_cap && nranks == 1) {
        PL.d_probe = buf<rsylv_b200_probe_event>(ctx, "probe", res->probe_cap);
        PL.probe_cap = res->probe_cap;
    }
    ck(ctx, cudaGetLastError(), "pack");

    if (deferred) return RSYLV_OK;  // validated on the device after the last pack
    std::vector<double> h_an((size_t)M * M), h_bn((size_t)N * N), h_yn(ny);
    ck(ctx, cudaMemcpyAsync(h_an.data(), anorm, sizeof(double) * M * M, cudaMemcpyDeviceToHost, st), "d2h");
    ck(ctx, cudaMemcpyAsync(h_bn.data(), bnorm, sizeof(double) * N * N, cudaMemcpyDeviceToHost, st), "d2h");
    // C tile norms: every local rank packed its owned tile columns (multi-rank)
    for (size_t li = 0; li < local.size(); ++li) {
        std::vector<double> part(ny);
        ck(ctx, cudaMemcpyAsync(part.data(), PL.rb[li].ynorm, sizeof(double) * ny, cudaMemcpyDeviceToHost, st), "d2h");
        ck(ctx, cudaStreamSynchronize(st), "sync");
        for (size_t t = 0; t < ny; ++t)
            if (nranks == 1 || (int)(t % N) % nranks == local[li]) h_yn[t] = part[t];
    }
    ck(ctx, cudaStreamSynchronize(st), "sync");
    for (int i = 0; i < M; ++i)
        for (int k = i; k < M; ++k)
            if (!(h_an[(size_t)i * M + k] <= PL.omega)) {
                res->invalid_reason = RSYLV_REASON_A_BOUND;
                return RSYLV_INVALID_ARGUMENT;
            }
    for (int l = 0; l < N; ++l)
        for (int j = l; j < N; ++j)
            if (!(h_bn[(size_t)l * N + j] <= PL.omega)) {
                res->invalid_reason = RSYLV_REASON_B_BOUND;
                return RSYLV_INVALID_ARGUMENT;
            }
    for (size_t t = 0; t < ny; ++t)  // (one rank per process: its owned columns; together all)
        if (!(h_yn[t] <= PL.omega)) {
            res->invalid_reason = RSYLV_REASON_C_BOUND;
            return RSYLV_INVALID_ARGUMENT;
        }
    return RSYLV_OK;
}

// Problem of local rank index li with its peers' pointers (virtual ranks: the other local
// workspaces; distributed: IPC-mapped peer workspaces).
Problem rank_problem(rsylv_b200_ctx* ctx, size_t li) {
    Plan& PL = ctx_plan(ctx);
    const RankBufs& B = PL.rb[li];
    Problem Q = PL.base;
    Q.Ypack = B.Yp;
    Q.tmaps = B.tmaps;
    Q.ynorm = B.ynorm;
    Q.yexp = B.yexp;
    Q.yst = B.yexp + (size_t)Q.M * Q.N;
    Q.uexp = B.uexp;
    Q.ubnd = B.ubnd;
    Q.state = B.state;
    Q.udone = B.udone;
    Q.err = B.err;
    Q.err_pivot = B.piv;
    Q.tile_pivot = B.tpiv;
    Q.events = B.ev;
    Q.task_next = B.tnext;
    Q.tasks = B.tasks;
    Q.ntasks = B.ntasks;
    Q.rank = PL.local[li];
    Q.nranks = PL.nranks;
    Q.sys_scope = 0;
    if (PL.d_probe) {
        Q.probe = reinterpret_cast<ProbeEv*>(PL.d_probe);
        Q.probe_count = B.ev + 1;
        Q.probe_cap = PL.probe_cap;  // every launch of the solve (main and side streams) logs
    }
    if (PL.nranks > 1) {
        // RSYLV_B200_SYS_SCOPE=1 (tests): system-scope flags and fences also for virtual ranks,
        // so the multi-GPU acquire / release code runs on one device
        const char* ss = std::getenv("RSYLV_B200_SYS_SCOPE");
        if (ss && ss[0] == '1') Q.sys_scope = 1;
        if (PL.local.size() > 1) {  // virtual ranks on this device
            for (size_t lj = 0; lj < PL.local.size(); ++lj) {
                const RankBufs& O = PL.rb[lj];
                const int r = PL.local[lj];
                Q.peerY[r] = O.Yp;
                Q.peerYexp[r] = O.yexp;
                Q.peerYnorm[r] = O.ynorm;
                Q.peerState[r] = O.state;
                Q.peerErr[r] = O.err;
            }
        } else {  // one rank per GPU
            rsylv_b200_plan_holder& H = ctx_holder(ctx);
            Q.sys_scope = 1;
            for (int r = 0; r < PL.nranks && (size_t)(5 * r + 4) < H.peer_ptrs.size(); ++r) {
                if (r == Q.rank) continue;
                Q.peerY[r] = static_cast<double*>(H.peer_ptrs[5 * r + 0]);
                Q.peerYexp[r] = static_cast<int*>(H.peer_ptrs[5 * r + 1]);
                Q.peerYnorm[r] = static_cast<double*>(H.peer_ptrs[5 * r + 2]);
                Q.peerState[r] = static_cast<int*>(H.peer_ptrs[5 * r + 3]);
                Q.peerErr[r] = static_cast<int*>(H.peer_ptrs[5 * r + 4]);
            }
        }
    }
    return Q;
}

// The tile DAG on every local rank, then the per-rank results: local alpha exponent minimum
// and max tile norm relative to it (owned tiles only).
// side: host pipeline -- the DAG starts on all but kPipeReserve SMs, side() enqueues the H2D +
// pack + validation work (and the remaining DAG CTAs) on the side stream, which the main
// stream joins before the alpha reduction
// RSYLV_B200_DEBUG_TIMING: events around the main DAG launch of the pipelined path
static cudaEvent_t g_dbg_a = nullptr, g_dbg_b = nullptr;
static int pipe_reserve() {  // SMs kept free of the main DAG launch for the pack kernels
    const char* e = std::getenv("RSYLV_B200_PIPE_RESERVE");
    const int r = e ? std::atoi(e) : 4;
    return r < 1 ? 1 : r;
}
#define kPipeReserve pipe_reserve()
// plan_launch enqueues the tile DAG (asynchronous); plan_collect waits for it and reduces.
// plan_run = both. A single-process multi-GPU solve launches every device first, then collects
// (a device's kernel waits on tiles its peers produce).
int plan_launch(rsylv_b200_ctx* ctx, rsylv_b200_result* res,
                const std::function<void(int)>* side = nullptr) {
    Plan& PL = ctx_plan(ctx);
    cudaStream_t st = PL.st;
    const int M = PL.M, N = PL.N;
    ck(ctx, cudaEventRecord(ctx->evp, st), "event");
    if (PL.nranks == 1) {
        Problem P = rank_problem(ctx, 0);
        if (PL.scheduler == 2) {  // development: update-phase throughput (garbage results)
            launch_update_bench(P, ctx->sms, st);
            res->dag_launches = 1;
        } else if (PL.scheduler == 1) {
            res->dag_launches = 0;
            for (int d = 0; d <= M + N - 2; ++d) {
                const int jlo = std::max(0, d - (M - 1)), jhi = std::min(N - 1, d);
                launch_tile_diag(P, d, jhi - jlo + 1, st);
                res->dag_launches += 1;
            }
        } else if (side) {
            // the side streams start after the setup on st, NOT after the DAG launched below.
            // Serialized execution (CUDA_LAUNCH_BLOCKING=1, RSYLV_B200_SAFE_ORDER=1): every
            // producer (H2D, pack, validation, ready counters) is enqueued BEFORE the spinning
            // DAG kernel, whose progress then never depends on the streams running concurrently
            // (the side stream's own DAG CTAs then solve everything). Otherwise only the first
            // shells are enqueued before it and the rest right after the launch (side(1))
            ck(ctx, cudaEventRecord(ctx->ev_side0, st), "event");
            (*side)(0);
            const bool dbgt = std::getenv("RSYLV_B200_DEBUG_TIMING") != nullptr;
            if (dbgt && !g_dbg_a) {
                cudaEventCreate(&g_dbg_a);
                cudaEventCreate(&g_dbg_b);
            }
            if (dbgt) cudaEventRecord(g_dbg_a, st);
            launch_persistent(P, std::max(1, ctx->sms - kPipeReserve), st);
            if (dbgt) cudaEventRecord(g_dbg_b, st);
            (*side)(1);
            ck(ctx, cudaStreamWaitEvent(st, ctx->ev_side, 0), "join");
            res->dag_launches = 2;
        } else {
            launch_persistent(P, ctx->sms, st);
            res->dag_launches = 1;
        }
        ck(ctx, cudaGetLastError(), "dag");
    } else if (PL.local.size() > 1) {
        std::vector<Problem> probs;
        for (size_t li = 0; li < PL.local.size(); ++li) probs.push_back(rank_problem(ctx, li));
        Problem* d_probs = buf<Problem>(ctx, "probs", probs.size());
        ck(ctx, cudaMemcpyAsync(d_probs, probs.data(), sizeof(Problem) * probs.size(),
                                cudaMemcpyHostToDevice, st), "h2d");
        const int R = (int)probs.size();
        const int grid = std::max(R, ctx->sms / R * R);
        ck(ctx, launch_persistent_mr(d_probs, R, grid, st), "persistent_mr");
        res->dag_launches = 1;
    } else {
        Problem P = rank_problem(ctx, 0);
        launch_persistent(P, ctx->sms, st);
        ck(ctx, cudaGetLastError(), "dag");
        res->dag_launches = 1;
    }
    ck(ctx, cudaEventRecord(ctx->evd, st), "event");
    return RSYLV_OK;
}

// pivot_owned (optional): set when a singular failure's pivot was read from a tile this
// context owns (multi-GPU: the owner's pivot is the one to report)
int plan_collect(rsylv_b200_ctx* ctx, rsylv_b200_result* res, int* emin_out, double* numax_out,
                 bool* pivot_owned = nullptr) {
    Plan& PL = ctx_plan(ctx);
    cudaStream_t st = PL.st;
    const int M = PL.M, N = PL.N;
    const size_t ny = PL.ny;
    if (pivot_owned) *pivot_owned = false;

    // ---- alpha reduction (tile_grid.cpp:38-42) over the owned tiles, exponent form
    std::vector<int> ye_all(ny, 0);
    std::vector<double> yn_all(ny, 0.0);
    int emin = 0;
    double numax_rel = 0.0;  // max ynorm * 2^(emin - yexp) over owned tiles
    int first_err = 0;
    double piv = 0.0;
    int best_enc = -1;  // singular failures: the earliest tile in the reference order wins
    res->scaling_events = 0;
    for (size_t li = 0; li < PL.local.size(); ++li) {
        const RankBufs& B = PL.rb[li];
        std::vector<int> ye(ny);
        std::vector<double> yn(ny);
        int h_err[4];
        double h_piv = 0;
        unsigned long long h_ev[2];
        ck(ctx, cudaMemcpyAsync(ye.data(), B.yexp, sizeof(int) * ny, cudaMemcpyDeviceToHost, st), "d2h");
        ck(ctx, cudaMemcpyAsync(yn.data(), B.ynorm, sizeof(double) * ny, cudaMemcpyDeviceToHost, st), "d2h");
        ck(ctx, cudaMemcpyAsync(h_err, B.err, sizeof h_err, cudaMemcpyDeviceToHost, st), "d2h");
        ck(ctx, cudaMemcpyAsync(&h_piv, B.piv, sizeof h_piv, cudaMemcpyDeviceToHost, st), "d2h");
        ck(ctx, cudaMemcpyAsync(h_ev, B.ev, sizeof h_ev, cudaMemcpyDeviceToHost, st), "d2h");
        ck(ctx, cudaStreamSynchronize(st), "solve");
        res->scaling_events += h_ev[0];
        if (PL.d_probe && li == 0) {
            res->probe_count = (size_t)h_ev[1];
            const size_t nc = std::min(res->probe_count, res->probe_cap);
            ck(ctx, cudaMemcpy(res->probe_log, PL.d_probe, nc * sizeof(rsylv_b200_probe_event),
                               cudaMemcpyDeviceToHost), "d2h");
        }
        if (h_err[0] == kErrSingular) {
            if (h_err[1] > best_enc) {  // enc = INT_MAX - priority: larger is earlier
                best_enc = h_err[1];
                const int pri = 0x7fffffff - h_err[1];
                const int k = M - 1 - pri / N, l = pri % N;
                if ((l % PL.nranks) == PL.local[li]) {
                    ck(ctx, cudaMemcpy(&piv, B.tpiv + (size_t)k * N + l, sizeof(double),
                                       cudaMemcpyDeviceToHost), "d2h");
                    if (pivot_owned) *pivot_owned = true;
                }
            }
            if (!first_err) first_err = h_err[0];
        } else if (h_err[0] != 0 && (!first_err || first_err == kErrSingular)) {
            first_err = h_err[0];  // non-singular errors (watchdog, invalid) dominate
            piv = h_piv;
        }
        for (size_t t = 0; t < ny; ++t)
            if ((int)(t % N) % PL.nranks == PL.local[li]) {
                ye_all[t] = ye[t];
                yn_all[t] = yn[t];
                emin = std::min(emin, ye[t]);
            }
    }
    if (first_err) {
        res->pivot = piv;
        if (first_err == kErrInvalid && PL.d_reason) {  // host pipeline: device-side checks
            int code = 4;
            ck(ctx, cudaMemcpy(&code, PL.d_reason, sizeof(int), cudaMemcpyDeviceToHost), "d2h");
            res->invalid_reason = code == 1 ? RSYLV_REASON_A_BOUND
                                : code == 2 ? RSYLV_REASON_B_BOUND : RSYLV_REASON_C_BOUND;
            return RSYLV_INVALID_ARGUMENT;
        }
        return first_err == kErrSingular ? RSYLV_SINGULAR : RSYLV_CUDA_ERROR;
    }
    for (size_t li = 0; li < PL.local.size(); ++li)
        for (size_t t = 0; t < ny; ++t)
            if ((int)(t % N) % PL.nranks == PL.local[li])
                numax_rel = std::max(numax_rel, std::ldexp(yn_all[t], emin - ye_all[t]));
    *emin_out = emin;
    *numax_out = numax_rel;
    return RSYLV_OK;
}

int plan_run(rsylv_b200_ctx* ctx, rsylv_b200_result* res, int* emin_out, double* numax_out,
             const std::function<void(int)>* side = nullptr) {
    const int st = plan_launch(ctx, res, side);
    if (st != RSYLV_OK) return st;
    return plan_collect(ctx, res, emin_out, numax_out);
}

// Largest s >= 0 with numax * 2^s <= omega and emin + s <= 0 (joint renormalisation).
int alpha_exponent(int emin, double numax, double omega) {
    int s = -emin;
    if (numax > 0.0) {
        int en = 0, eo = 0;
        const double mn = std::frexp(numax, &en), mo = std::frexp(omega, &eo);
        const int smax = eo - en - (mn <= mo ? 0 : 1);
        s = std::max(0, std::min(s, smax));
    }
    return emin + s;
}

// Consistency scaling fused with the copy-out of the owned columns (tile_grid.cpp:44-52).
int plan_finish(rsylv_b200_ctx* ctx, int alpha_exp, double numax, int emin, double* y, size_t ldy,
                rsylv_b200_result* res) {
    Plan& PL = ctx_plan(ctx);
    cudaStream_t st = PL.st;
    res->alpha_exp = alpha_exp;
    res->alpha = alpha_exp >= -1022 ? std::ldexp(1.0, alpha_exp) : 0.0;
    res->max_tile_norm = std::ldexp(numax, alpha_exp - emin);
    for (size_t li = 0; li < PL.local.size(); ++li) {
        Problem Q = rank_problem(ctx, li);
        launch_unpack(Q, alpha_exp, y, (long long)ldy, st);
    }
    ck(ctx, cudaGetLastError(), "unpack");
    ck(ctx, cudaEventRecord(ctx->ev1, st), "event");
    ck(ctx, cudaEventSynchronize(ctx->ev1), "sync");
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
    res->device_ms = ms;
    cudaEventElapsedTime(&ms, ctx->ev0, ctx->evp);
    res->pack_ms = ms;
    cudaEventElapsedTime(&ms, ctx->evp, ctx->evd);
    res->dag_ms = ms;
    cudaEventElapsedTime(&ms, ctx->evd, ctx->ev1);
    res->unpack_ms = ms;
    return alpha_exp >= -1022 ? RSYLV_OK : RSYLV_SCALE_UNDERFLOW;
}

int solve_device_impl(rsylv_b200_ctx* ctx, const SolveArgs& A) {
    rsylv_b200_result* res = A.res;
    if (A.opt.tile_size < 2) {  // partition.cpp:75-76
        res->invalid_reason = RSYLV_REASON_TILE_SIZE;
        return RSYLV_INVALID_ARGUMENT;
    }
    if (A.m == 0 || A.n == 0) {
        res->alpha = 1.0;
        res->alpha_exp = 0;
        return RSYLV_OK;
    }
    const int R = std::max(1, std::min(A.opt.virtual_ranks, kMaxRanks));
    std::vector<int> local;
    for (int r = 0; r < R; ++r) local.push_back(r);
    int st = plan_prepare(ctx, A, R, local);
    if (st != RSYLV_OK) return st;
    int emin = 0;
    double numax = 0.0;
    st = plan_run(ctx, res, &emin, &numax);
    if (st != RSYLV_OK) return st;
    const int ae = alpha_exponent(emin, numax, ctx_plan(ctx).omega);
    return plan_finish(ctx, ae, numax, emin, A.y, A.ldy, res);
}

int guarded_call(rsylv_b200_ctx* ctx, int (*fn)(rsylv_b200_ctx*, const SolveArgs&),
                 const SolveArgs& a) {
    try {
        return fn(ctx, a);
    } catch (const Fail& f) {
        return f.status;
    }
}

}  // namespace

namespace {
// host <-> device staging for the debug entries (plain cudaMalloc / cudaMemcpy, synchronous)
struct Staging {
    std::vector<void*> ptrs;
    bool ok = true;
    template <class T>
    T* up(const T* h, size_t n) {
        void* d = nullptr;
        if (cudaMalloc(&d, sizeof(T) * (n ? n : 1)) != cudaSuccess) {
            ok = false;
            return nullptr;
        }
        ptrs.push_back(d);
        if (h && n && cudaMemcpy(d, h, sizeof(T) * n, cudaMemcpyHostToDevice) != cudaSuccess) ok = false;
        return static_cast<T*>(d);
    }
    template <class T>
    void down(T* h, const T* d, size_t n) {
        if (ok && n && cudaMemcpy(h, d, sizeof(T) * n, cudaMemcpyDeviceToHost) != cudaSuccess) ok = false;
    }
    ~Staging() {
        for (void* p : ptrs) cudaFree(p);
    }
};
}  // namespace

namespace {
// ||x||_F of an m x n column-major device matrix without overflow: max |x| first, then the sum
// of squares of x * 2^-e(max). Returns the norm as (mantissa part, binary exponent).
void frob_norm(rsylv_b200_ctx* ctx, const double* x, size_t m, size_t n, size_t ld,
               cudaStream_t st, double* nm, int* ne) {
    const int blocks = 2 * ctx->sms;
    double* part = buf<double>(ctx, "res_part", 2 * (size_t)blocks);
    std::vector<double> hm(blocks), hs(blocks);
    ck(ctx, launch_absmax_sumsq((int)m, (int)n, x, (long long)ld, 0, blocks, part, part + blocks, st),
       "absmax");
    ck(ctx, cudaMemcpyAsync(hm.data(), part, sizeof(double) * blocks, cudaMemcpyDeviceToHost, st), "d2h");
    ck(ctx, cudaStreamSynchronize(st), "sync");
    double mx = 0.0;
    for (double v : hm) mx = (v != v || mx != mx) ? NAN : std::max(mx, v);
    if (!(mx > 0.0) || std::isinf(mx)) {
        *nm = mx;
        *ne = 0;
        return;
    }
    int e = 0;
    std::frexp(mx, &e);
    ck(ctx, launch_absmax_sumsq((int)m, (int)n, x, (long long)ld, -e, blocks, part, part + blocks, st),
       "sumsq");
    ck(ctx, cudaMemcpyAsync(hs.data(), part + blocks, sizeof(double) * blocks, cudaMemcpyDeviceToHost, st), "d2h");
    ck(ctx, cudaStreamSynchronize(st), "sync");
    double s = 0.0;
    for (double v : hs) s += v;
    *nm = std::sqrt(s);
    *ne = e;
}
}  // namespace

extern "C" {

const char* rsylv_b200_status_string(int s) {
    switch (s) {
        case RSYLV_OK: return "ok";
        case RSYLV_INVALID_ARGUMENT: return "invalid_argument";
        case RSYLV_SINGULAR: return "SingularEquationError";
        case RSYLV_SCALE_UNDERFLOW: return "ScaleUnderflowError";
        case RSYLV_CUDA_ERROR: return "cuda_error";
        case RSYLV_NO_DEVICE: return "no_device";
        default: return "unknown";
    }
}

const char* rsylv_b200_last_error(const rsylv_b200_ctx* ctx) {
    return ctx ? ctx->last_error.c_str() : "";
}

int rsylv_b200_create(int device, rsylv_b200_ctx** out) {
    *out = nullptr;
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) return RSYLV_NO_DEVICE;
    if (device < 0) cudaGetDevice(&device);
    if (device >= count) return RSYLV_NO_DEVICE;
    if (cudaSetDevice(device) != cudaSuccess) return RSYLV_NO_DEVICE;
    auto* ctx = new rsylv_b200_ctx();
    ctx->device = device;
    cudaDeviceGetAttribute(&ctx->sms, cudaDevAttrMultiProcessorCount, device);
    if (cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&ctx->side_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->ev_side0, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->ev_side, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreate(&ctx->ev0) != cudaSuccess || cudaEventCreate(&ctx->ev1) != cudaSuccess ||
        cudaEventCreate(&ctx->evp) != cudaSuccess || cudaEventCreate(&ctx->evd) != cudaSuccess) {
        delete ctx;
        return RSYLV_CUDA_ERROR;
    }
    *out = ctx;
    return RSYLV_OK;
}

void rsylv_b200_destroy(rsylv_b200_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    for (auto& kv : ctx->bufs)
        if (kv.second.p) cudaFree(kv.second.p);
    if (ctx->ev0) cudaEventDestroy(ctx->ev0);
    if (ctx->ev1) cudaEventDestroy(ctx->ev1);
    if (ctx->holder) {
        close_peers(ctx);
        delete ctx->holder;
    }
    if (ctx->evp) cudaEventDestroy(ctx->evp);
    if (ctx->evd) cudaEventDestroy(ctx->evd);
    if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
    if (ctx->side_stream) cudaStreamDestroy(ctx->side_stream);
    if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
    for (cudaEvent_t e : ctx->ev_shell) cudaEventDestroy(e);
    if (ctx->ev_side0) cudaEventDestroy(ctx->ev_side0);
    if (ctx->ev_side) cudaEventDestroy(ctx->ev_side);
    delete ctx;
}

// The stream argument of the device-resident entry points: NULL is the legacy default stream
// (include/rsylv_b200.h), so the solve is ordered after the caller's work on it (torch's
// default stream handle is 0).
static cudaStream_t as_stream(void* stream) {
    return stream ? (cudaStream_t)stream : cudaStreamLegacy;
}

static void init_result(rsylv_b200_result* r) {
    rsylv_b200_probe_event* log = r->probe_log;
    size_t cap = r->probe_cap;
    std::memset(r, 0, sizeof *r);
    r->probe_log = log;
    r->probe_cap = cap;
}

int rsylv_b200_solve_device(rsylv_b200_ctx* ctx, size_t m, size_t n, const double* a,
                            size_t lda, const unsigned char* ablk, const double* b, size_t ldb,
                            const unsigned char* bblk, const double* c, size_t ldc, double* y,
                            size_t ldy, const rsylv_b200_options* opt, void* stream,
                            rsylv_b200_result* res) {
    if (!ctx || !opt || !res) return RSYLV_INVALID_ARGUMENT;
    init_result(res);
    if (cudaSetDevice(ctx->device) != cudaSuccess) return RSYLV_CUDA_ERROR;
    SolveArgs A{m, n, a, b, c, lda, ldb, ldc, ablk, bblk, y, ldy, *opt, as_stream(stream), res};
    return guarded_call(ctx, solve_device_impl, A);
}

// Host pipeline (rsylv_b200_options.host_pipeline): the DAG starts on all but kPipeReserve SMs
// while a copy stream uploads the inputs in shells (shell t: tile row M-1-t of A from its
// diagonal tile on, tile column t of B, the matching L-shaped piece of C -- what the tiles with
// max(M-1-i, j) == t need beyond the earlier shells) and a side stream packs each shell on the
// reserved SMs, checks its tile norms on the device (the reference's argument checks and reason
// order; a failure aborts the DAG and returns RSYLV_INVALID_ARGUMENT) and publishes the shell
// count (tile tasks wait on these counters at their start); finally it launches the remaining
// DAG CTAs, which join the task queue. Overlaps the H2D traffic with the solve.
static int solve_host_pipelined(rsylv_b200_ctx* ctx, const SolveArgs& H, double* da, double* db,
                                double* dc, double* dy) {
    cudaStream_t st = H.st;
    const size_t m = H.m, n = H.n;
    SolveArgs D = H;
    D.a = da;
    D.b = db;
    D.c = dc;
    D.y = dy;
    D.lda = m;
    D.ldb = n;
    D.ldc = m;
    D.ldy = m;
    int status = plan_prepare(ctx, D, 1, std::vector<int>{0}, true);
    if (status != RSYLV_OK) return status;
    Plan& PL = ctx_plan(ctx);
    const int M = PL.M, N = PL.N, TSP = PL.TSP;
    const Problem Q = rank_problem(ctx, 0);
    unsigned long long h2d = 0;
    static const bool dbg = std::getenv("RSYLV_B200_DEBUG_TIMING") != nullptr;
    static cudaEvent_t dbg0 = nullptr, dbg1 = nullptr, dbg2 = nullptr;
    static int* h_next = nullptr;
    // phase 0: before the main DAG launch; phase 1: right after it. Enqueuing the later shells'
    // 2-D copies costs the host ~0.1 s at c5 (one DMA descriptor per 8 KB strip row, up to 40000
    // per copy), which used to delay the launch of the DAG kernel itself; now only the first
    // shells (short strips) go before it. With CUDA_LAUNCH_BLOCKING=1 (or
    // RSYLV_B200_SAFE_ORDER=1) every producer is still enqueued before the spinning kernel.
    int next_tlo = 0;
    bool side_done = false;
    std::function<void(int)> side = [&](int phase) {
        if (side_done) return;
        // copies on their own stream, back to back; the packs of shell t (on the 4 spare SMs)
        // follow its copies through an event, so the copy engine never waits for a pack kernel
        // (one stream for both serialized them: ~0.1 s of the c5 call)
        cudaStream_t ss = ctx->side_stream, cs = ctx->copy_stream;
        if (phase == 0) {
            ck(ctx, cudaStreamWaitEvent(ss, ctx->ev_side0, 0), "wait");
            ck(ctx, cudaStreamWaitEvent(cs, ctx->ev_side0, 0), "wait");
        }
        if (dbg && !dbg0) {
            cudaEventCreate(&dbg0);
            cudaEventCreate(&dbg1);
        }
        if (dbg && phase == 0) cudaEventRecord(dbg0, cs);
        while ((int)ctx->ev_shell.size() < std::max(M, N)) {
            cudaEvent_t e = nullptr;
            ck(ctx, cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
            ctx->ev_shell.push_back(e);
        }
        // Shell order: shell t brings what the tiles (i, j) with max(M-1-i, j) == t need beyond
        // the earlier shells -- tile row r = M-1-t of A from its diagonal tile on (the trailing
        // square A[r:, r:] grows by one tile row), tile column t of B (the leading square), and
        // of C the tiles (i >= r, t) and (r, j < t). The work the DAG can start on then grows
        // like (copied fraction)^1.5 instead of ^3 (whole tile columns of A from the right and
        // of C from the left), so the DAG is input-starved for ~100 ms instead of ~220 ms of the
        // 0.47 s c5 upload.
        // (copies are issued for kG shells at a time: the row strips are then kG tiles = kG KB
        //  wide per column instead of 1 KB, which the copy engine moves at full PCIe rate; a
        //  group's strip of A also carries the few below-diagonal tiles inside it, zeros)
        const int kG = [] {  // (read per call: tests vary it)
            const char* e = std::getenv("RSYLV_B200_SHELL_GROUP");
            const int g = e ? std::atoi(e) : 8;
            return g < 1 ? 1 : g;
        }();
        const int T = std::max(M, N);
        static const bool safe_order = [] {
            const char* a = std::getenv("CUDA_LAUNCH_BLOCKING");
            const char* b = std::getenv("RSYLV_B200_SAFE_ORDER");
            return (a && a[0] == '1') || (b && b[0] == '1');
        }();
        // phase 0 stops after the shells whose strips are short (a quarter of them: ~6 % of the
        // strip rows); they feed the DAG for the first ~30 ms of the upload
        const int tend = (phase == 0 && !safe_order) ? std::min(T, (T / 4 + kG - 1) / kG * kG) : T;
        for (int tlo = next_tlo; tlo < tend; tlo += kG) {
            const int thi = std::min(tlo + kG, T);
            const int rlo = std::max(0, M - thi);  // tile rows [rlo, M-1-tlo] (A, C), if tlo < M
            const size_t R0 = PL.rc[rlo];
            if (tlo < M) {
                const size_t R1 = PL.rc[M - tlo];
                ck(ctx, cudaMemcpy2DAsync(da + R0 + R0 * m, m * 8, H.a + R0 + R0 * H.lda, H.lda * 8,
                                          (R1 - R0) * 8, m - R0, cudaMemcpyHostToDevice, cs), "h2d A");
                h2d += 8ull * (R1 - R0) * (m - R0);
                const size_t cend = PL.cc[std::min(tlo, N)];
                if (cend > 0) {  // C: the group's tile rows, the tile columns of earlier groups
                    ck(ctx, cudaMemcpy2DAsync(dc + R0, m * 8, H.c + R0, H.ldc * 8, (R1 - R0) * 8, cend,
                                              cudaMemcpyHostToDevice, cs), "h2d C rows");
                    h2d += 8ull * (R1 - R0) * cend;
                }
            }
            if (tlo < N) {  // B tile columns [tlo, chi) (upper part) and the C column pieces
                const int chi = std::min(thi, N);
                const size_t c0 = PL.cc[tlo], c1 = PL.cc[chi];
                ck(ctx, cudaMemcpy2DAsync(db + c0 * n, n * 8, H.b + c0 * H.ldb, H.ldb * 8, c1 * 8,
                                          c1 - c0, cudaMemcpyHostToDevice, cs), "h2d B");
                ck(ctx, cudaMemcpy2DAsync(dc + R0 + c0 * m, m * 8, H.c + R0 + c0 * H.ldc, H.ldc * 8,
                                          (m - R0) * 8, c1 - c0, cudaMemcpyHostToDevice, cs), "h2d C cols");
                h2d += 8ull * c1 * (c1 - c0) + 8ull * (m - R0) * (c1 - c0);
            }
            ck(ctx, cudaEventRecord(ctx->ev_shell[tlo], cs), "event");
            ck(ctx, cudaStreamWaitEvent(ss, ctx->ev_shell[tlo], 0), "wait");
            for (int t = tlo; t < thi; ++t) {
                const int r = M - 1 - t;              // tile row of this shell (A, C), if any
                const int jend = std::min(t, N);      // C row strip: tile columns [0, jend)
                const int i0 = std::max(0, r);        // C column piece: tile rows [i0, M)
                if (t < M) {
                    launch_pack_upper_row(da, (long long)m, Q.rcut, M, TSP, const_cast<double*>(Q.Apack),
                                          Q.anorm, Q.aexp, r, ss, !std::isinf(PL.omega));
                    if (jend > 0) launch_pack_full_row(dc, (long long)m, Q, Q.ynorm, r, jend, ss);
                }
                if (t < N) {
                    launch_pack_upper_col(db, (long long)n, Q.ccut, N, TSP, const_cast<double*>(Q.Bpack),
                                          Q.bnorm, Q.bexp, t, ss, !std::isinf(PL.omega));
                    launch_pack_full_col(dc, (long long)m, Q, Q.ynorm, t, i0, ss);
                }
                launch_validate_shell(Q, PL.d_reason, t < M ? r : -1, t < N ? t : -1, t < N ? t : -1, i0,
                                      (t < M && jend > 0) ? r : -1, jend, ss);
                launch_set_ready(Q.in_ready, t < M ? t + 1 : -1, t < N ? t + 1 : -1, t + 1, ss);
            }
        }
        next_tlo = std::max(next_tlo, tend);
        if (next_tlo < T) return;   // (phase 0 of the split order: the rest follows the DAG launch)
        if (phase == 0 && !safe_order) return;  // everything fitted into phase 0: finish in phase 1
        side_done = true;
        if (dbg) {  // (read after the solve: nothing here may block the host before the DAG launch)
            if (!dbg2) cudaEventCreate(&dbg2);
            if (!h_next) cudaMallocHost(&h_next, sizeof(int));
            cudaEventRecord(dbg1, cs);
            cudaMemcpyAsync(h_next, Q.task_next, sizeof(int), cudaMemcpyDeviceToHost, ss);
            cudaEventRecord(dbg2, ss);
        }
        launch_persistent(Q, std::min(kPipeReserve, ctx->sms - 1), ss);
        ck(ctx, cudaGetLastError(), "pipeline");
        ck(ctx, cudaEventRecord(ctx->ev_side, ss), "event");
    };
    int emin = 0;
    double numax = 0.0;
    status = plan_run(ctx, H.res, &emin, &numax, &side);
    H.res->h2d_bytes = h2d;
    if (dbg && dbg2) {
        cudaEventSynchronize(dbg1);
        cudaEventSynchronize(dbg2);
        float ms = 0, ms2 = 0;
        cudaEventElapsedTime(&ms, dbg0, dbg1);
        cudaEventElapsedTime(&ms2, dbg0, dbg2);
        std::fprintf(stderr, "[rsylv_b200] host pipeline: H2D copies %.1f ms for %.2f GB (%.1f GB/s); last shell "
                     "packed at %.1f ms, %d of %d tile tasks taken by then\n", ms, h2d / 1e9, h2d / 1e6 / ms, ms2,
                     *h_next, Q.ntasks);
        if (g_dbg_a) {
            float t0 = 0, t1 = 0, t2 = 0;
            cudaEventSynchronize(ctx->evd);
            cudaEventElapsedTime(&t0, ctx->evp, g_dbg_a);
            cudaEventElapsedTime(&t1, g_dbg_a, g_dbg_b);
            cudaEventElapsedTime(&t2, g_dbg_b, ctx->evd);
            std::fprintf(stderr, "[rsylv_b200] host pipeline: main DAG kernel starts %.1f ms after the solve's setup, "
                         "runs %.1f ms, the side stream's DAG CTAs end %.1f ms later\n", t0, t1, t2);
        }
    }
    if (status != RSYLV_OK) return status;
    const int ae = alpha_exponent(emin, numax, PL.omega);
    status = plan_finish(ctx, ae, numax, emin, dy, m, H.res);
    ck(ctx, cudaMemcpy2DAsync(H.y, H.ldy * 8, dy, m * 8, m * 8, n, cudaMemcpyDeviceToHost, st), "d2h Y");
    ck(ctx, cudaStreamSynchronize(st), "sync");
    H.res->d2h_bytes = 8ull * m * n;
    return status;
}

// Optionally page-locks the caller's host buffers for one rsylv_b200_solve (the reference's
// DenseMatrix storage is ordinary pageable memory, whose cudaMemcpy*Async is staged and blocks
// the host thread, so the host pipeline's per-column copies no longer overlap the DAG). Measured
// at c4 (tools/e2e_pageable.py, profiles/r02/e2e_pageable_c4.jsonl): pinned 272 ms, pageable
// 793 ms, pageable + cudaHostRegister for the call 1147 ms -- pinning 10 GB costs more than the
// overlap it buys, so it is off unless RSYLV_B200_HOST_REGISTER=1 (worth it only for callers
// that keep registering the same buffers themselves: pass pinned memory). Buffers that are
// already pinned / registered, or smaller than 64 MB, are left alone.
struct HostRegistration {
    std::vector<void*> regs;
    bool enabled = false;
    HostRegistration() {
        const char* e = std::getenv("RSYLV_B200_HOST_REGISTER");
        enabled = e && e[0] == '1';
    }
    void add(const void* p, size_t bytes, bool read_only) {
        if (!enabled || !p || bytes < ((size_t)64 << 20)) return;
        cudaPointerAttributes at;
        if (cudaPointerGetAttributes(&at, p) == cudaSuccess && at.type != cudaMemoryTypeUnregistered)
            return;
        (void)cudaGetLastError();
        const unsigned fl = cudaHostRegisterDefault | (read_only ? cudaHostRegisterReadOnly : 0);
        if (cudaHostRegister(const_cast<void*>(p), bytes, fl) == cudaSuccess)
            regs.push_back(const_cast<void*>(p));
        else
            (void)cudaGetLastError();  // (overlapping ranges, limits: the plain path still works)
    }
    ~HostRegistration() {
        for (void* p : regs) cudaHostUnregister(p);
    }
};

static int solve_host_impl(rsylv_b200_ctx* ctx, const SolveArgs& H) {
    HostRegistration reg;
    const auto span = [](size_t rows, size_t cols, size_t ld) {
        return cols ? ((cols - 1) * ld + rows) * sizeof(double) : 0;
    };
    reg.add(H.a, span(H.m, H.m, H.lda), true);
    reg.add(H.b, span(H.n, H.n, H.ldb), true);
    reg.add(H.c, span(H.m, H.n, H.ldc), true);
    reg.add(H.y, span(H.m, H.n, H.ldy), false);
    cudaStream_t st = H.st;
    const size_t m = H.m, n = H.n;
    double* da = buf<double>(ctx, "hA", m * m);
    double* db = buf<double>(ctx, "hB", n * n);
    double* dc = buf<double>(ctx, "hC", m * n);
    double* dy = buf<double>(ctx, "hY", m * n);
    {   // host pipeline: on request, or automatically from 64 tiles up (single GPU, persistent)
        const size_t ts = std::min<size_t>(std::max<size_t>(2, H.opt.tile_size), (size_t)kTileMax);
        const size_t tiles = ((m + ts - 1) / ts) * ((n + ts - 1) / ts);
        const bool pipe = H.opt.host_pipeline > 0 ||
                          (H.opt.host_pipeline == 0 && tiles >= 64);
        if (pipe && H.opt.scheduler == 0 && H.opt.virtual_ranks <= 1 && H.opt.tile_size >= 2)
            return solve_host_pipelined(ctx, H, da, db, dc, dy);
    }
    unsigned long long h2d = 8ull * m * n;
    // A and B are quasi-upper-triangular: only the upper tiles travel (tile column k needs rows
    // 0 .. end of tile k), halving their PCIe traffic; pack_upper never reads below them.
    auto copy_upper = [&](double* dst, const double* src, size_t ld, size_t dim,
                          const unsigned char* blk) {
        std::vector<unsigned char> codes = codes_or_ones(blk, dim);
        const size_t ts = H.opt.tile_size > (size_t)kTileMax ? (size_t)kTileMax
                                                              : std::max<size_t>(2, H.opt.tile_size);
        const std::vector<int> cuts = partition(codes.data(), dim, ts);
        for (size_t k = 0; k + 1 < cuts.size(); ++k) {
            const size_t c0 = cuts[k], c1 = cuts[k + 1];
            ck(ctx, cudaMemcpy2DAsync(dst + c0 * dim, dim * 8, src + c0 * ld, ld * 8, c1 * 8,
                                      c1 - c0, cudaMemcpyHostToDevice, st), "h2d upper");
            h2d += 8ull * c1 * (c1 - c0);
        }
    };
    copy_upper(da, H.a, H.lda, m, H.ablk);
    copy_upper(db, H.b, H.ldb, n, H.bblk);
    ck(ctx, cudaMemcpy2DAsync(dc, m * 8, H.c, H.ldc * 8, m * 8, n, cudaMemcpyHostToDevice, st), "h2d C");
    SolveArgs D = H;
    D.a = da;
    D.b = db;
    D.c = dc;
    D.y = dy;
    D.lda = m;
    D.ldb = n;
    D.ldc = m;
    D.ldy = m;
    const int status = solve_device_impl(ctx, D);
    H.res->h2d_bytes = h2d;
    if (status == RSYLV_OK || status == RSYLV_SCALE_UNDERFLOW) {
        ck(ctx, cudaMemcpy2DAsync(H.y, H.ldy * 8, dy, m * 8, m * 8, n, cudaMemcpyDeviceToHost, st), "d2h Y");
        ck(ctx, cudaStreamSynchronize(st), "sync");
        H.res->d2h_bytes = 8ull * m * n;
    }
    return status;
}

int rsylv_b200_solve(rsylv_b200_ctx* ctx, size_t m, size_t n, const double* a, size_t lda,
                     const unsigned char* ablk, const double* b, size_t ldb,
                     const unsigned char* bblk, const double* c, size_t ldc, double* y,
                     size_t ldy, const rsylv_b200_options* opt, rsylv_b200_result* res) {
    if (!ctx || !opt || !res) return RSYLV_INVALID_ARGUMENT;
    init_result(res);
    if (cudaSetDevice(ctx->device) != cudaSuccess) return RSYLV_CUDA_ERROR;
    if (opt->tile_size < 2) {
        res->invalid_reason = RSYLV_REASON_TILE_SIZE;
        return RSYLV_INVALID_ARGUMENT;
    }
    if (m == 0 || n == 0) {
        res->alpha = 1.0;
        return RSYLV_OK;
    }
    SolveArgs A{m, n, a, b, c, lda, ldb, ldc, ablk, bblk, y, ldy, *opt, ctx->own_stream, res};
    return guarded_call(ctx, solve_host_impl, A);
}

// Single-process multi-GPU solve on HOST buffers: one context per GPU (distinct devices), tile
// columns block-cyclic over them (column j on ctxs[j % R]). Every GPU gets the upper tiles of A
// and B (replicated: any tile row may need any A_ik) and only its owned tile columns of C; Y is
// copied back per owned column. Solved tiles are pushed to the peers over NVLink through plain
// peer pointers (cudaDeviceEnablePeerAccess; the multi-process form uses CUDA IPC), the alpha
// reduction is the host-side MIN over the contexts, then each GPU rescales and copies out its
// columns. The reference's parallel API maps here (ExecutionMode::workers -> GPUs, the shim).
int rsylv_b200_solve_group(rsylv_b200_ctx* const* ctxs, int R, size_t m, size_t n,
                           const double* a, size_t lda, const unsigned char* ablk, const double* b,
                           size_t ldb, const unsigned char* bblk, const double* c, size_t ldc,
                           double* y, size_t ldy, const rsylv_b200_options* opt,
                           rsylv_b200_result* res) {
    if (!ctxs || R < 1 || R > kMaxRanks || !opt || !res) return RSYLV_INVALID_ARGUMENT;
    for (int r = 0; r < R; ++r)
        if (!ctxs[r]) return RSYLV_INVALID_ARGUMENT;
    if (R == 1) return rsylv_b200_solve(ctxs[0], m, n, a, lda, ablk, b, ldb, bblk, c, ldc, y, ldy, opt, res);
    for (int r = 0; r < R; ++r)
        for (int q = r + 1; q < R; ++q)
            if (ctxs[r]->device == ctxs[q]->device) return RSYLV_INVALID_ARGUMENT;  // distinct GPUs
    init_result(res);
    if (opt->tile_size < 2) {
        res->invalid_reason = RSYLV_REASON_TILE_SIZE;
        return RSYLV_INVALID_ARGUMENT;
    }
    if (m == 0 || n == 0) {
        res->alpha = 1.0;
        return RSYLV_OK;
    }
    rsylv_b200_ctx* failed = ctxs[0];
    try {
        const size_t ts = std::min<size_t>(opt->tile_size, (size_t)kTileMax);
        std::vector<unsigned char> acodes = codes_or_ones(ablk, m), bcodes = codes_or_ones(bblk, n);
        const std::vector<int> rcut = partition(acodes.data(), m, ts);
        const std::vector<int> ccut = partition(bcodes.data(), n, ts);
        const int N = (int)ccut.size() - 1;
        std::vector<rsylv_b200_result> rr(R);
        std::vector<double*> dy(R);
        unsigned long long h2d = 0, d2h = 0;
        // 1. per GPU: upper tiles of A and B, owned tile columns of C; plan + pack + validate
        for (int r = 0; r < R; ++r) {
            rsylv_b200_ctx* ctx = ctxs[r];
            failed = ctx;
            ck(ctx, cudaSetDevice(ctx->device), "device");
            cudaStream_t st = ctx->own_stream;
            double* da = buf<double>(ctx, "hA", m * m);
            double* db = buf<double>(ctx, "hB", n * n);
            double* dc = buf<double>(ctx, "hC", m * n);
            dy[r] = buf<double>(ctx, "hY", m * n);
            for (size_t k = 0; k + 1 < rcut.size(); ++k) {
                const size_t c0 = rcut[k], c1 = rcut[k + 1];
                ck(ctx, cudaMemcpy2DAsync(da + c0 * m, m * 8, a + c0 * lda, lda * 8, c1 * 8, c1 - c0,
                                          cudaMemcpyHostToDevice, st), "h2d A");
                h2d += 8ull * c1 * (c1 - c0);
            }
            for (int j = 0; j < N; ++j) {
                const size_t c0 = ccut[j], c1 = ccut[j + 1];
                ck(ctx, cudaMemcpy2DAsync(db + c0 * n, n * 8, b + c0 * ldb, ldb * 8, c1 * 8, c1 - c0,
                                          cudaMemcpyHostToDevice, st), "h2d B");
                h2d += 8ull * c1 * (c1 - c0);
                if (j % R != r) continue;
                ck(ctx, cudaMemcpy2DAsync(dc + c0 * m, m * 8, c + c0 * ldc, ldc * 8, m * 8, c1 - c0,
                                          cudaMemcpyHostToDevice, st), "h2d C");
                h2d += 8ull * m * (c1 - c0);
            }
            SolveArgs D{m, n, da, db, dc, m, n, m, ablk, bblk, dy[r], m, *opt, st, &rr[r]};
            D.opt.scheduler = 0;
            init_result(&rr[r]);
            const int sp = plan_prepare(ctx, D, R, std::vector<int>{r});
            if (sp != RSYLV_OK) {
                res->invalid_reason = rr[r].invalid_reason;
                return sp;
            }
        }
        // 2. peer access + the peers' workspace pointers
        for (int r = 0; r < R; ++r) {
            failed = ctxs[r];
            ck(ctxs[r], cudaSetDevice(ctxs[r]->device), "device");
            for (int q = 0; q < R; ++q) {
                if (q == r) continue;
                int can = 0;
                ck(ctxs[r], cudaDeviceCanAccessPeer(&can, ctxs[r]->device, ctxs[q]->device), "peer query");
                if (!can) {
                    ctxs[r]->last_error = "no peer access between the GPUs of the group";
                    return RSYLV_CUDA_ERROR;
                }
                const cudaError_t e = cudaDeviceEnablePeerAccess(ctxs[q]->device, 0);
                if (e == cudaErrorPeerAccessAlreadyEnabled)
                    (void)cudaGetLastError();
                else
                    ck(ctxs[r], e, "enable peer access");
            }
            close_peers(ctxs[r]);
            rsylv_b200_plan_holder& H = ctx_holder(ctxs[r]);
            H.peer_ptrs.assign(5 * R, nullptr);
            H.peer_handles.assign(R, {});
            H.raw_peers = true;
            for (int q = 0; q < R; ++q) {
                if (q == r) continue;
                const RankBufs& Bq = ctx_plan(ctxs[q]).rb[0];
                void* ptrs[5] = {Bq.Yp, Bq.yexp, Bq.ynorm, Bq.state, Bq.err};
                for (int k = 0; k < 5; ++k) H.peer_ptrs[5 * q + k] = ptrs[k];
            }
        }
        // 3. launch every GPU's tile DAG, then 4. collect (a GPU waits on its peers' tiles)
        for (int r = 0; r < R; ++r) {
            failed = ctxs[r];
            ck(ctxs[r], cudaSetDevice(ctxs[r]->device), "device");
            const int sl = plan_launch(ctxs[r], &rr[r]);
            if (sl != RSYLV_OK) return sl;
        }
        int emin = 0, status = RSYLV_OK;
        double numax = 0.0, pivot = 0.0;
        std::vector<int> em(R);
        std::vector<double> nu(R);
        unsigned long long events = 0;
        for (int r = 0; r < R; ++r) {
            failed = ctxs[r];
            ck(ctxs[r], cudaSetDevice(ctxs[r]->device), "device");
            bool owned = false;
            const int sc = plan_collect(ctxs[r], &rr[r], &em[r], &nu[r], &owned);
            events += rr[r].scaling_events;
            if (sc != RSYLV_OK) {
                if (status == RSYLV_OK || status == RSYLV_SINGULAR) {
                    if (sc == RSYLV_SINGULAR) {
                        if (owned || status == RSYLV_OK) pivot = rr[r].pivot;
                    }
                    status = (status == RSYLV_OK || sc != RSYLV_SINGULAR) ? sc : status;
                }
                continue;
            }
            emin = std::min(emin, em[r]);
        }
        res->scaling_events = events;
        res->row_tiles = rr[0].row_tiles;
        res->col_tiles = rr[0].col_tiles;
        if (status != RSYLV_OK) {
            res->pivot = pivot;
            return status;
        }
        for (int r = 0; r < R; ++r) numax = std::max(numax, std::ldexp(nu[r], emin - em[r]));
        const int ae = alpha_exponent(emin, numax, ctx_plan(ctxs[0]).omega);
        // 5. consistency scaling + copy-out of the owned columns
        int fin = RSYLV_OK;
        double dev_ms = 0.0;
        for (int r = 0; r < R; ++r) {
            rsylv_b200_ctx* ctx = ctxs[r];
            failed = ctx;
            ck(ctx, cudaSetDevice(ctx->device), "device");
            fin = plan_finish(ctx, ae, numax, emin, dy[r], m, &rr[r]);
            dev_ms = std::max(dev_ms, rr[r].device_ms);
            for (int j = r; j < N; j += R) {
                const size_t c0 = ccut[j], c1 = ccut[j + 1];
                ck(ctx, cudaMemcpy2DAsync(y + c0 * ldy, ldy * 8, dy[r] + c0 * m, m * 8, m * 8, c1 - c0,
                                          cudaMemcpyDeviceToHost, ctx->own_stream), "d2h Y");
                d2h += 8ull * m * (c1 - c0);
            }
        }
        for (int r = 0; r < R; ++r) ck(ctxs[r], cudaStreamSynchronize(ctxs[r]->own_stream), "sync");
        res->alpha_exp = ae;
        res->alpha = rr[0].alpha;
        res->max_tile_norm = rr[0].max_tile_norm;
        res->device_ms = dev_ms;
        res->dag_launches = R;
        res->h2d_bytes = h2d;
        res->d2h_bytes = d2h;
        return fin;
    } catch (const Fail& f) {
        (void)failed;
        return f.status;
    }
}

int rsylv_b200_has_fast_diag(void) { return has_fast_diag(); }

int rsylv_b200_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        (void)cudaGetLastError();
        return 0;
    }
    return n;
}

int rsylv_b200_dist_prepare(rsylv_b200_ctx* ctx, int nranks, int rank, size_t m, size_t n,
                            const double* a, size_t lda, const unsigned char* ablk,
                            const double* b, size_t ldb, const unsigned char* bblk,
                            const double* c, size_t ldc, const rsylv_b200_options* opt,
                            void* stream, void* handle_out, rsylv_b200_result* res) {
    if (!ctx || !opt || !res || nranks < 1 || nranks > kMaxRanks || rank < 0 || rank >= nranks)
        return RSYLV_INVALID_ARGUMENT;
    init_result(res);
    if (opt->tile_size < 2) {
        res->invalid_reason = RSYLV_REASON_TILE_SIZE;
        return RSYLV_INVALID_ARGUMENT;
    }
    if (m == 0 || n == 0) return RSYLV_INVALID_ARGUMENT;
    if (cudaSetDevice(ctx->device) != cudaSuccess) return RSYLV_CUDA_ERROR;
    try {
        SolveArgs A{m, n, a, b, c, lda, ldb, ldc, ablk, bblk, nullptr, 0, *opt, as_stream(stream),
                    res};
        A.opt.scheduler = 0;
        const int st = plan_prepare(ctx, A, nranks, std::vector<int>{rank});
        if (st != RSYLV_OK) return st;
        const RankBufs& B = ctx_plan(ctx).rb[0];
        void* ptrs[5] = {B.Yp, B.yexp, B.ynorm, B.state, B.err};
        unsigned char* out = static_cast<unsigned char*>(handle_out);
        for (int k = 0; k < 5; ++k) {
            cudaIpcMemHandle_t h;
            ck(ctx, cudaIpcGetMemHandle(&h, ptrs[k]), "ipc handle");
            std::memcpy(out + 64 * k, &h, 64);
        }
        return RSYLV_OK;
    } catch (const Fail& f) {
        return f.status;
    }
}

int rsylv_b200_dist_run(rsylv_b200_ctx* ctx, const void* all_handles, void* stream,
                        rsylv_b200_result* res) {
    if (!ctx || !res) return RSYLV_INVALID_ARGUMENT;
    if (cudaSetDevice(ctx->device) != cudaSuccess) return RSYLV_CUDA_ERROR;
    try {
        Plan& PL = ctx_plan(ctx);
        PL.st = as_stream(stream);
        rsylv_b200_plan_holder& H = ctx_holder(ctx);
        const unsigned char* in = static_cast<const unsigned char*>(all_handles);
        const int R = PL.nranks, me = PL.local[0];
        if ((int)H.peer_handles.size() != R) {
            close_peers(ctx);
            H.peer_handles.assign(R, {});
            H.peer_ptrs.assign(5 * R, nullptr);
        }
        for (int r = 0; r < R; ++r) {
            if (r == me) continue;
            std::vector<unsigned char> hb(in + RSYLV_DIST_HANDLE_BYTES * r,
                                          in + RSYLV_DIST_HANDLE_BYTES * (r + 1));
            if (H.peer_handles[r] == hb) continue;
            for (int k = 0; k < 5; ++k)
                if (H.peer_ptrs[5 * r + k]) cudaIpcCloseMemHandle(H.peer_ptrs[5 * r + k]);
            for (int k = 0; k < 5; ++k) {
                cudaIpcMemHandle_t h;
                std::memcpy(&h, hb.data() + 64 * k, 64);
                void* p = nullptr;
                ck(ctx, cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess), "ipc open");
                H.peer_ptrs[5 * r + k] = p;
            }
            H.peer_handles[r] = hb;
        }
        int emin = 0;
        double numax = 0.0;
        const int st = plan_run(ctx, res, &emin, &numax);
        res->alpha_exp = emin;
        res->max_tile_norm = numax;
        return st;
    } catch (const Fail& f) {
        return f.status;
    }
}

int rsylv_b200_dist_finish(rsylv_b200_ctx* ctx, int alpha_exp, double* y, size_t ldy,
                           void* stream, rsylv_b200_result* res) {
    if (!ctx || !res) return RSYLV_INVALID_ARGUMENT;
    if (cudaSetDevice(ctx->device) != cudaSuccess) return RSYLV_CUDA_ERROR;
    try {
        Plan& PL = ctx_plan(ctx);
        PL.st = as_stream(stream);
        // res->alpha_exp / max_tile_norm on entry: the global emin and numax (relative to emin)
        const int emin = res->alpha_exp;
        const double numax = res->max_tile_norm;
        return plan_finish(ctx, alpha_exp, numax, emin, y, ldy, res);
    } catch (const Fail& f) {
        return f.status;
    }
}

int rsylv_b200_robust_update(rsylv_b200_ctx* ctx, size_t m, size_t k, size_t n, double* c,
                             int32_t* c_exp, double* c_norm, const double* a, const double* b,
                             int32_t ab_exp, double omega, uint64_t* events) {
    if (!ctx || m == 0 || k == 0 || n == 0 || m > kTileMax || k > kTileMax || n > kTileMax)
        return RSYLV_INVALID_ARGUMENT;
    if (cudaSetDevice(ctx->device) != cudaSuccess) return RSYLV_CUDA_ERROR;
    try {
        if (!ctx->configured) {
            ck(ctx, configure_kernels(), "configure_kernels");
            ctx->configured = true;
        }
        cudaStream_t st = ctx->own_stream;
        // embed the update as column update Y_00 -= A_01 * Y_10 of a 2 x 1 tile grid
        const size_t mk = m + k;
        std::vector<double> abig(mk * mk, 0.0), ybig(mk * n, 0.0);
        for (size_t j = 0; j < k; ++j)
            for (size_t i = 0; i < m; ++i) abig[i + (m + j) * mk] = a[i + j * m];
        for (size_t j = 0; j < mk; ++j) abig[j + j * mk] = 1.0;
        for (size_t j = 0; j < n; ++j) {
            for (size_t i = 0; i < m; ++i) ybig[i + j * mk] = c[i + j * m];
            for (size_t i = 0; i < k; ++i) ybig[m + i + j * mk] = b[i + j * k];
        }
        const int M = 2, N = 1;
        std::vector<int> rc{0, (int)m, (int)mk}, cc{0, (int)n};
        const int tmax = (int)std::max(std::max(m, k), n);
        const int TSP = (tmax + kBM - 1) / kBM * kBM;
        const size_t slot = (size_t)TSP * TSP, slack = (size_t)64 * TSP + 1024;
        double* dA = buf<double>(ctx, "ruA", mk * mk);
        double* dY = buf<double>(ctx, "ruY", mk * n);
        double* Ap = buf<double>(ctx, "ruApack", 3 * slot + slack);
        double* Bp = buf<double>(ctx, "ruBpack", 1 * slot + slack);
        double* Yp = buf<double>(ctx, "ruYpack", 2 * slot + slack);
        double* an = buf<double>(ctx, "ruan", 4);
        double* bn = buf<double>(ctx, "rubn", 1);
        int* ax = buf<int>(ctx, "ruax", 4);
        int* bx = buf<int>(ctx, "rubx", 1);
        double* yn = buf<double>(ctx, "ruyn", 2);
        int* ye = buf<int>(ctx, "ruye", 4);  // yexp, then yst
        int* ue = buf<int>(ctx, "ruue", 2);
        double* ub = buf<double>(ctx, "ruub", 2);
        int* sta = buf<int>(ctx, "rust", 2);
        int* ud = buf<int>(ctx, "ruud", 2);
        int* errw = buf<int>(ctx, "ruerr", 4);
        double* pivw = buf<double>(ctx, "rupiv", 1);
        unsigned long long* evw = buf<unsigned long long>(ctx, "ruev", 2);
        int* d_rc = buf<int>(ctx, "rurc", 3);
        int* d_cc = buf<int>(ctx, "rucc", 2);
        ck(ctx, cudaMemcpyAsync(dA, abig.data(), abig.size() * 8, cudaMemcpyHostToDevice, st), "h2d");
        ck(ctx, cudaMemcpyAsync(dY, ybig.data(), ybig.size() * 8, cudaMemcpyHostToDevice, st), "h2d");
        ck(ctx, cudaMemcpyAsync(d_rc, rc.data(), 12, cudaMemcpyHostToDevice, st), "h2d");
        ck(ctx, cudaMemcpyAsync(d_cc, cc.data(), 8, cudaMemcpyHostToDevice, st), "h2d");
        ck(ctx, cudaMemsetAsync(Ap, 0, (3 * slot + slack) * 8, st), "memset");
        ck(ctx, cudaMemsetAsync(Bp, 0, (slot + slack) * 8, st), "memset");
        ck(ctx, cudaMemsetAsync(Yp + 2 * slot, 0, slack * 8, st), "memset");
        ck(ctx, cudaMemsetAsync(errw, 0, 16, st), "memset");
        ck(ctx, cudaMemsetAsync(evw, 0, 16, st), "memset");
        Problem P{};
        P.M = M;
        P.N = N;
        P.TSP = TSP;
        P.m = (int)mk;
        P.n = (int)n;
        P.rcut = d_rc;
        P.ccut = d_cc;
        P.Apack = Ap;
        P.Bpack = Bp;
        P.Ypack = Yp;
        P.anorm = an;
        P.bnorm = bn;
        P.aexp = ax;
        P.bexp = bx;
        P.ynorm = yn;
        P.yexp = ye;
        P.yst = ye + 2;
        P.uexp = ue;
        P.ubnd = ub;
        P.state = sta;
        P.udone = ud;
        P.err = errw;
        P.err_pivot = pivw;
        P.events = evw;
        P.tmaps = make_tmaps(ctx, "rutmaps", Ap, 3, Bp, 1, Yp, 2, st);
        P.nsub_r = P.nsub_c = TSP / kBM;
        P.omega = omega > 0 ? omega : DBL_MAX / 2;
        P.small_num = DBL_MIN / DBL_EPSILON;
        P.x_omega = host_xf(P.omega);
        P.x_target = host_xf(P.omega * (1.0 - 0x1p-30));
        launch_pack_upper(dA, (long long)mk, d_rc, M, TSP, Ap, an, ax, st, !std::isinf(P.omega));
        ck(ctx, cudaMemsetAsync(bx, 0, sizeof(int), st), "memset");
        launch_pack_full(dY, (long long)mk, P, yn, st);
        const int exps[2] = {c_exp ? *c_exp : 0, ab_exp};
        ck(ctx, cudaMemcpyAsync(ye, exps, 8, cudaMemcpyHostToDevice, st), "h2d");
        launch_update_only(P, 0, 0, st);
        ck(ctx, cudaGetLastError(), "update");
        int ue_h = 0;
        unsigned long long ev_h[2];
        std::vector<double> out(slot);
        ck(ctx, cudaMemcpyAsync(&ue_h, ue, 4, cudaMemcpyDeviceToHost, st), "d2h");
        ck(ctx, cudaMemcpyAsync(ev_h, evw, 16, cudaMemcpyDeviceToHost, st), "d2h");
        ck(ctx, cudaMemcpyAsync(out.data(), Yp, slot * 8, cudaMemcpyDeviceToHost, st), "d2h");
        ck(ctx, cudaStreamSynchronize(st), "sync");
        double nrm = 0.0;
        for (size_t i = 0; i < m; ++i) {
            double s = 0.0;
            for (size_t j = 0; j < n; ++j) {
                c[i + j * m] = out[i + j * TSP];
                s += std::fabs(c[i + j * m]);
            }
            nrm = std::max(nrm, s);
        }
        if (c_exp) *c_exp = ue_h;
        if (c_norm) *c_norm = nrm;
        if (events) *events = ev_h[0];
        return RSYLV_OK;
    } catch (const Fail& f) {
        return f.status;
    }
}

// development: per-phase cycle counters of the tile tasks (reset=1 clears them)
int rsylv_b200_dgemm(rsylv_b200_ctx* ctx, int ta, int tb, size_t m, size_t n, size_t k,
                     double alpha, const double* a, size_t lda, const double* b, size_t ldb,
                     double beta, double* c, size_t ldc, int a_upper, int b_upper, void* stream) {
    if (!ctx || (m && n && k && (!a || !b)) || (m && n && !c)) return RSYLV_INVALID_ARGUMENT;
    if (cudaSetDevice(ctx->device) != cudaSuccess) return RSYLV_CUDA_ERROR;
    try {
        ck(ctx, launch_dgemm(ta, tb, (int)m, (int)n, (int)k, alpha, a, (long long)lda, b,
                             (long long)ldb, beta, c, (long long)ldc, a_upper, b_upper,
                             as_stream(stream)), "dgemm");
    } catch (const Fail& f) {
        return f.status;
    }
    return RSYLV_OK;
}

int rsylv_b200_relative_residual(rsylv_b200_ctx* ctx, size_t m, size_t n, const double* a,
                                 size_t lda, const double* b, size_t ldb, const double* c,
                                 size_t ldc, const double* y, size_t ldy, int32_t alpha_exp,
                                 void* stream, double* out7) {
    if (!ctx || !out7 || m == 0 || n == 0) return RSYLV_INVALID_ARGUMENT;
    if (cudaSetDevice(ctx->device) != cudaSuccess) return RSYLV_CUDA_ERROR;
    try {
        cudaStream_t st = as_stream(stream);
        double ym;
        int ye;
        frob_norm(ctx, y, m, n, ldy, st, &ym, &ye);  // (only its max is needed: ye)
        // the frame: Y * 2^s with max |Y 2^s| <= 2^400
        const int s = ye > 400 ? 400 - ye : 0;
        double* Ys = buf<double>(ctx, "res_ys", m * n);
        double* R = buf<double>(ctx, "res_r", m * n);
        ck(ctx, launch_scale_copy((int)m, (int)n, y, (long long)ldy, Ys, (long long)m, s, st), "scale");
        ck(ctx, launch_scale_copy((int)m, (int)n, c, (long long)ldc, R, (long long)m, alpha_exp + s, st),
           "scale");
        double rn, an, bn, yn, cn;
        int re, ae, be, yse, ce;
        frob_norm(ctx, R, m, n, m, st, &cn, &ce);
        // R = A Ys - R, then R += Ys B (triangular K ranges skipped)
        ck(ctx, launch_dgemm(0, 0, (int)m, (int)n, (int)m, 1.0, a, (long long)lda, Ys, (long long)m,
                             -1.0, R, (long long)m, 1, 0, st), "dgemm");
        ck(ctx, launch_dgemm(0, 0, (int)m, (int)n, (int)n, 1.0, Ys, (long long)m, b, (long long)ldb,
                             1.0, R, (long long)m, 0, 1, st), "dgemm");
        frob_norm(ctx, R, m, n, m, st, &rn, &re);
        frob_norm(ctx, a, m, m, lda, st, &an, &ae);
        frob_norm(ctx, b, n, n, ldb, st, &bn, &be);
        frob_norm(ctx, Ys, m, n, m, st, &yn, &yse);
        auto val = [](double v, int e) { return std::ldexp(v, e); };
        // denominator in the common frame 2^yse (||A||, ||B|| are moderate: tile norms <= omega)
        const double ab = val(an, ae) + val(bn, be);
        const int top = std::max({yse + 0, ce, re});
        const double den = ab * val(yn, yse - top) + val(cn, ce - top);
        out7[0] = val(rn, re - top) / den;
        out7[1] = val(rn, re);
        out7[2] = val(an, ae);
        out7[3] = val(bn, be);
        out7[4] = val(yn, yse);
        out7[5] = val(cn, ce);
        out7[6] = s;
    } catch (const Fail& f) {
        return f.status;
    }
    return RSYLV_OK;
}

int rsylv_b200_debug_small_solve(size_t n, const int32_t* rs, const int32_t* cs, const double* a,
                                 const double* b, const double* c, double omega,
                                 double small_num, double* z, int32_t* dz, int32_t* status,
                                 double* pivot) {
    if (n == 0) return RSYLV_OK;
    if (!rs || !cs || !a || !b || !c || !z || !dz || !status || !pivot) return RSYLV_INVALID_ARGUMENT;
    for (size_t t = 0; t < n; ++t)
        if (rs[t] < 1 || rs[t] > 2 || cs[t] < 1 || cs[t] > 2) return RSYLV_INVALID_ARGUMENT;
    Staging S;
    const int* drs = S.up(rs, n);
    const int* dcs = S.up(cs, n);
    const double* da = S.up(a, 4 * n);
    const double* db = S.up(b, 4 * n);
    const double* dc = S.up(c, 4 * n);
    double* dzv = S.up<double>(nullptr, 4 * n);
    int* ddz = S.up<int>(nullptr, n);
    int* dst = S.up<int>(nullptr, n);
    double* dpv = S.up<double>(nullptr, n);
    if (!S.ok) return RSYLV_CUDA_ERROR;
    launch_debug_small((int)n, drs, dcs, da, db, dc, omega > 0 ? omega : DBL_MAX / 2,
                       small_num > 0 ? small_num : DBL_MIN / DBL_EPSILON, dzv, ddz, dst, dpv);
    if (cudaGetLastError() != cudaSuccess) return RSYLV_CUDA_ERROR;
    S.down(z, dzv, 4 * n);
    S.down(dz, ddz, n);
    S.down(status, dst, n);
    S.down(pivot, dpv, n);
    return S.ok ? RSYLV_OK : RSYLV_CUDA_ERROR;
}

int rsylv_b200_debug_guards(size_t n, const double* c, const double* a, const double* b,
                            const double* bnd, const double* t, double omega, int32_t* d_upd_xq,
                            int32_t* d_upd_xf, int32_t* d_div) {
    if (n == 0) return RSYLV_OK;
    if (!c || !a || !b || !bnd || !t || !d_upd_xq || !d_upd_xf || !d_div) return RSYLV_INVALID_ARGUMENT;
    Staging S;
    const double *dc = S.up(c, n), *da = S.up(a, n), *db = S.up(b, n), *dbn = S.up(bnd, n),
                 *dt = S.up(t, n);
    int *o1 = S.up<int>(nullptr, n), *o2 = S.up<int>(nullptr, n), *o3 = S.up<int>(nullptr, n);
    if (!S.ok) return RSYLV_CUDA_ERROR;
    launch_debug_guards((int)n, dc, da, db, dbn, dt, omega, o1, o2, o3);
    if (cudaGetLastError() != cudaSuccess) return RSYLV_CUDA_ERROR;
    S.down(d_upd_xq, o1, n);
    S.down(d_upd_xf, o2, n);
    S.down(d_div, o3, n);
    return S.ok ? RSYLV_OK : RSYLV_CUDA_ERROR;
}

int rsylv_b200_debug_counters(unsigned long long* out32, int reset) {
    if (reset) return reset_prof() == cudaSuccess ? RSYLV_OK : RSYLV_CUDA_ERROR;
    return read_prof(out32) == cudaSuccess ? RSYLV_OK : RSYLV_CUDA_ERROR;
}

// development: average cycles of one warp-level 16x16 sub-block solve (mixed: 2x2 blocks)
int rsylv_b200_debug_subsolve(int reps, int mode, long long* cycles, double* out256) {
    return bench_subsolve(reps, mode, cycles, out256) == 0 ? RSYLV_OK : RSYLV_CUDA_ERROR;
}

int rsylv_b200_generate_quasi_triangular(size_t n, double* dev, size_t ld,
                                         const unsigned char* blk_host, uint64_t seed,
                                         double up_lo, double up_hi, double d_lo, double d_hi,
                                         double off_lo, double off_hi, void* stream) {
    unsigned char* d_blk = nullptr;
    if (blk_host) {
        if (cudaMalloc(&d_blk, n) != cudaSuccess) return RSYLV_CUDA_ERROR;
        cudaMemcpy(d_blk, blk_host, n, cudaMemcpyHostToDevice);
    }
    launch_gen_qt((int)n, dev, (long long)ld, d_blk, seed, up_lo, up_hi, d_lo, d_hi, off_lo,
                  off_hi, (cudaStream_t)stream);
    cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
    if (d_blk) cudaFree(d_blk);
    return e == cudaSuccess ? RSYLV_OK : RSYLV_CUDA_ERROR;
}

int rsylv_b200_generate_rhs(size_t m, size_t n, double* dev, size_t ld, uint64_t seed, int dist,
                            double lo, double hi, const int32_t* hot_tiles, size_t n_hot,
                            size_t hot_tile, double hot_factor, void* stream) {
    int* d_hot = nullptr;
    if (n_hot) {
        if (cudaMalloc(&d_hot, n_hot * 2 * sizeof(int)) != cudaSuccess) return RSYLV_CUDA_ERROR;
        cudaMemcpy(d_hot, hot_tiles, n_hot * 2 * sizeof(int), cudaMemcpyHostToDevice);
    }
    launch_gen_rhs((int)m, (int)n, dev, (long long)ld, seed, dist, lo, hi, d_hot, (int)n_hot,
                   (int)(hot_tile ? hot_tile : 1), hot_factor, (cudaStream_t)stream);
    cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
    if (d_hot) cudaFree(d_hot);
    return e == cudaSuccess ? RSYLV_OK : RSYLV_CUDA_ERROR;
}

}  // extern "C"
