// rsylv-b200 device-side common definitions (sm_100a).
//
// Scale factors are powers of two kept as int32 exponents, so every rescale is exact and no
// local scale can underflow mid-solve (the reference keeps doubles in (0,1] and throws
// ScaleUnderflowError from accumulate_scale, overflow.cpp:42-46). Growth bounds that the
// reference evaluates in x87 long double (overflow.cpp:29-57, robust_update.cpp:36-39) are
// evaluated here in mantissa/exponent form ("xf"), which cannot overflow.
#pragma once

#include <cstdint>
#include <cuda.h>  // CUtensorMap (type only: the encoder is resolved at run time, no libcuda link)
#include <cuda_runtime.h>

namespace rsb {

#ifndef RSYLV_KSUB
#define RSYLV_KSUB 16
#endif
constexpr int kSub = RSYLV_KSUB; // sub-block edge inside a diagonal-tile solve (8 or 16)
constexpr int kBM = 128;         // internal tile edge: one CTA task owns one <= 128 x 128 tile
constexpr int kTileMax = kBM;    // largest internal tile edge
// max sub-blocks per tile edge (tile <= 128, sub-blocks >= kSub - 1)
constexpr int kSubMax = (kBM + kSub - 2) / (kSub - 1);
constexpr int kFS = 8;                                 // fast-path sub-block edge
constexpr int kFSMax = (kBM + kFS - 2) / (kFS - 1);    // fast-path sub-blocks per tile edge
constexpr int kFLA = 8, kFLB = 9;                      // fast-path staged A / B leading dims
constexpr int kLDT = kBM + 1;    // shared-memory tile leading dim (odd: conflict-free columns)
constexpr int kLDD = kSub + 1;   // staged diagonal sub-block of B leading dim (column reads across lanes)
constexpr int kLDDA = kSub;      // staged diagonal sub-block of A: row reads across lanes (r0 + 16 c: distinct banks)
constexpr int kMaxRanks = 8;     // GPUs (or virtual ranks) sharing one solve
#ifndef RSYLV_KC
#define RSYLV_KC 32
#endif
#ifndef RSYLV_STAGES
#define RSYLV_STAGES 3
#endif
constexpr int kKC = RSYLV_KC;          // K depth of one pipeline stage (a multiple of 8)
constexpr int kStages = RSYLV_STAGES;  // depth of the TMA operand ring
constexpr int kThreads = 512;    // 16 warps, for both task kinds
constexpr int kWarps = kThreads / 32;
constexpr int kYNormExp = 500;   // solved Y tiles are stored with norm in [2^499, 2^500)
constexpr int kSolvers = kSubMax < kWarps ? kSubMax : kWarps;  // warps solving sub-blocks at once
constexpr int kLDA = kBM + 4;    // smem A stage: [kKC][kLDA] (rows contiguous), conflict-free
constexpr int kLDB = kKC + 4;    // smem B stage: [kBM][kLDB] (k contiguous), conflict-free

// error codes written to the device error word (first writer wins)
enum : int { kErrNone = 0, kErrSingular = 2, kErrWatchdog = 8, kErrInternal = 9, kErrInvalid = 10 };
constexpr unsigned long long kWatchdogNs = 60ull * 1000000000ull;  // a source tile never arriving

// 2^e as a double for e in [-1022, 1023] (exact, no libm call).
__host__ __device__ __forceinline__ double pow2(int e) {
#ifdef __CUDA_ARCH__
    return __longlong_as_double((long long)(e + 1023) << 52);
#else
    return ldexp(1.0, e);
#endif
}

// ---------------------------------------------------------------------------------------
// xf: nonnegative value m * 2^e with m in [0.5, 1), or zero (m == 0).
struct xf {
    double m;
    int e;
};

__host__ __device__ __forceinline__ xf xf_zero() { return {0.0, 0}; }

// v >= 0 (finite, or +inf which maps to a value above every double)
__host__ __device__ __forceinline__ xf xf_from(double v) {
#ifdef __CUDA_ARCH__
    const long long b = __double_as_longlong(v);
    const int ex = (int)((b >> 52) & 0x7ff);
    if (ex != 0 && ex != 0x7ff)
        return {__longlong_as_double((b & 0x800fffffffffffffLL) | (1022LL << 52)), ex - 1022};
    if (ex == 0x7ff) return {0.5, 1 << 20};
#endif
    if (v == 0.0) return {0.0, 0};
    if (!(v <= 1.7976931348623157e308)) return {0.5, 1 << 20};  // +inf (omega = inf: no guard)
    int e = 0;
    const double m = frexp(v, &e);
    return {m, e};
}

__host__ __device__ __forceinline__ xf xf_renorm(double m, int e) {
    const xf t = xf_from(m);
    if (t.m == 0.0) return t;
    return {t.m, t.e + e};
}

__host__ __device__ __forceinline__ xf xf_mul(xf a, xf b) {
    if (a.m == 0.0 || b.m == 0.0) return {0.0, 0};
    return xf_renorm(a.m * b.m, a.e + b.e);
}

__host__ __device__ __forceinline__ xf xf_shift(xf a, int k) {
    if (a.m == 0.0) return a;
    return {a.m, a.e + k};
}

// Upper-bound-preserving sum: a difference of more than ~1074 binades drops the smaller term,
// an error far inside the 2^-30 shave headroom (overflow.cpp:17).
__host__ __device__ __forceinline__ xf xf_add(xf a, xf b) {
    if (a.m == 0.0) return b;
    if (b.m == 0.0) return a;
    if (a.e < b.e) {
        xf t = a;
        a = b;
        b = t;
    }
    const int d = a.e - b.e;
    const double s = d > 1000 ? a.m : a.m + b.m * pow2(-d);
    return xf_renorm(s, a.e);
}

__host__ __device__ __forceinline__ bool xf_le(xf a, xf b) {
    if (a.m == 0.0) return true;
    if (b.m == 0.0) return false;
    if (a.e != b.e) return a.e < b.e;
    return a.m <= b.m;
}

__host__ __device__ __forceinline__ xf xf_max(xf a, xf b) { return xf_le(a, b) ? b : a; }

// Integer upper bounds for the update-phase source headers: value <= m * 2^(e - 32) with
// m in [2^31, 2^32) (or m = 0 for zero), the same exponent convention as xf. Everything here
// is integer arithmetic: the scalar FP64 pipe shares its datapath with DMMA, so FP64 bound
// arithmetic in the middle of the update GEMM stalls behind the tensor work. Bounds round UP
// (xq_from, xq_mul, xq_add); the comparison limits omega / target round DOWN (xq_from_down),
// so a guard never fires later than the exact rule (at most one binade earlier, and only
// within 2^-31 of the limit, far inside the 2^-30 shave headroom of overflow.cpp:17).
#ifdef __CUDACC__
struct xq {
    unsigned int m;
    int e;
};

__device__ __forceinline__ xq xq_norm64(unsigned long long p, int e) {
    // p in [2^63, 2^64): m = ceil(p / 2^32)
    unsigned long long m = (p >> 32) + ((p & 0xffffffffull) != 0 ? 1 : 0);
    if (m >> 32) {
        m >>= 1;
        ++e;
    }
    return {(unsigned int)m, e};
}

__device__ __forceinline__ xq xq_from_bits(double v, bool up) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(v) & 0x7fffffffffffffffull;
    const int ex = (int)(b >> 52);
    if (ex == 0x7ff) return {0x80000000u, 1 << 20};  // +inf: above every double (no guard)
    if (b == 0) return {0u, 0};
    unsigned long long f = b & 0x000fffffffffffffull;
    int e;
    if (ex != 0) {
        f |= 1ull << 52;  // value = f * 2^(ex - 1075)
        e = ex - 1022;
    } else {              // subnormal: value = f * 2^-1074
        const int lz = __clzll(f) - 11;  // shift the leading one to bit 52
        f <<= lz;
        e = 1 - 1022 - lz;
    }
    // f in [2^52, 2^53): value = (f / 2^53) * 2^e
    const unsigned long long p = f << 11;  // [2^63, 2^64)
    if (up) return xq_norm64(p, e);
    return {(unsigned int)(p >> 32), e};
}
__device__ __forceinline__ xq xq_from(double v) { return xq_from_bits(v, true); }
__device__ __forceinline__ xq xq_from_down(double v) { return xq_from_bits(v, false); }

__device__ __forceinline__ xq xq_shift(xq a, int k) { return a.m ? xq{a.m, a.e + k} : a; }

__device__ __forceinline__ xq xq_mul(xq a, xq b) {
    if (a.m == 0 || b.m == 0) return {0u, 0};
    unsigned long long p = (unsigned long long)a.m * b.m;  // [2^62, 2^64)
    int e = a.e + b.e;
    if (!(p >> 63)) {
        p <<= 1;
        --e;
    }
    return xq_norm64(p, e);
}

__device__ __forceinline__ xq xq_add(xq a, xq b) {
    if (a.m == 0) return b;
    if (b.m == 0) return a;
    if (a.e < b.e) {
        const xq t = a;
        a = b;
        b = t;
    }
    const int d = a.e - b.e;
    // b < 2^(b.e) <= 2^(a.e - d): below one unit of a's last place when d >= 32
    const unsigned long long bs = d >= 32 ? 1ull : ((unsigned long long)b.m >> d) + ((b.m & ((1u << d) - 1u)) != 0 ? 1 : 0);
    unsigned long long s = (unsigned long long)a.m + bs;
    int e = a.e;
    if (s >> 32) {
        s = (s >> 1) + (s & 1);
        ++e;
        if (s >> 32) {
            s >>= 1;
            ++e;
        }
    }
    return {(unsigned int)s, e};
}

__device__ __forceinline__ bool xq_le(xq a, xq b) {
    if (a.m == 0) return true;
    if (b.m == 0) return false;
    if (a.e != b.e) return a.e < b.e;
    return a.m <= b.m;
}

// xf_guard on integer bounds (omega / target from xq_from_down)
__device__ __forceinline__ int xq_guard(xq g, xq omega, xq target) {
    if (omega.e >= (1 << 19) || xq_le(g, omega)) return 0;
    const int d = g.e - target.e + (g.m > target.m ? 1 : 0);
    return d < 1 ? 1 : d;
}

__device__ __forceinline__ xf xq_to_xf(xq a) {
    if (a.m == 0) return xf_zero();
    return {(double)a.m * 0x1p-32, a.e};  // exact; (m / 2^32) in [0.5, 1)
}
#endif  // __CUDACC__

// Power-of-two guard (the exponent form of update_scale, overflow.cpp:29-40): 0 when
// g <= omega; otherwise the least d >= 1 with g * 2^-d <= target (= omega * (1 - 2^-30)).
__host__ __device__ __forceinline__ int xf_guard(xf g, xf omega, xf target) {
    // omega = +inf (xf_from gives e = 1 << 20): the non-robust solve, no guard ever fires and
    // Inf / NaN propagate as in the reference's plain substitution
    if (omega.e >= (1 << 19) || xf_le(g, omega)) return 0;
    int d = g.e - target.e + (g.m > target.m ? 1 : 0);
    return d < 1 ? 1 : d;
}

__host__ __device__ __forceinline__ double xf_to_double(xf a) { return ldexp(a.m, a.e); }

// x * 2^e for any e. Inside the normal exponent range one multiply (exact, or a single
// rounding when the result is subnormal); outside it ldexp (single rounding). pow2(e) must only
// ever see e in [-1022, 1023].
__host__ __device__ __forceinline__ double scale2(double x, int e) {
    if (e >= -1022 && e <= 1023) return x * pow2(e);
    return ldexp(x, e);
}

// ---------------------------------------------------------------------------------------
// Problem descriptor shared by all kernels (device pointers unless noted).
struct ProbeEv {
    unsigned int k, l;
    int scale_exp;
    int pad;
    double norm;
};

struct Problem {
    int M, N;       // row / column tile counts
    int TSP;        // packed tile slot leading dimension (multiple of kBM)
    int m, n;
    const int* rcut;            // M+1 row-tile cuts
    const int* ccut;            // N+1 col-tile cuts
    const unsigned char* ablk;  // m block codes
    const unsigned char* bblk;  // n block codes
    const CUtensorMap* tmaps;   // device array of 4 TMA tensor maps over the packed slots:
                                // [0] Apack as L operand, [1] Ypack as L, [2] Ypack as R,
                                // [3] Bpack as R (runtime.cpp make_tmaps; kernels.cu USmem)
    const double* Apack;        // upper tiles of A, slot tri(i,k) = k*(k+1)/2 + i
    const double* Bpack;        // upper tiles of B
    double* Ypack;              // all tiles of Y, slot i*N + j
    double* anorm;              // M*M, (i,k) at i*M+k (upper)
    double* bnorm;              // N*N, (l,j) at l*N+j (upper)
    int* in_ready;              // host pipeline: shells packed so far for A (tile rows from the bottom), B,
                                // C (from the left); nullptr when every input is packed upfront
    int* aexp;                  // M*M: off-diagonal A tiles are stored as A_ik * 2^-aexp (pack)
    int* bexp;                  // N*N: the same for B
    double* ynorm;              // M*N current cached tile norm
    int* yexp;                  // M*N tile exponent (scale = 2^yexp, yexp <= 0)
    int* yst;                   // M*N (= yexp + M*N): a solved tile is stored as Y_ij * 2^-yst,
                                // normalized (norm in [2^(kYNormExp-1), 2^kYNormExp))
    int* uexp;                  // M*N exponent after the update phase
    double* ubnd;               // M*N update-phase growth bound (cached norm at rest)
    int* state;                 // M*N: 1 once solved (persistent scheduler flags)
    int* udone;                 // M*N: finished update subtasks
    int* err;                   // first error code
    double* err_pivot;
    double* tile_pivot;         // M*N: pivot of a tile's singular block (err[1] picks the tile)
    unsigned long long* events; // scaling events
    ProbeEv* probe;             // optional probe log
    unsigned long long* probe_count;
    unsigned long long probe_cap;
    int* task_next;             // persistent scheduler: next task index
    const int* tasks;           // persistent scheduler: packed (i, j, sr, sc) task list
    int ntasks;
    int nsub_r, nsub_c;         // subtiles per tile edge (TSP / kBM)
    double omega, small_num;
    xf x_omega, x_target;       // omega and omega * (1 - 2^-30) in xf form
    // multi-rank: tile columns block-cyclic over nranks (column j owned by rank j % nranks).
    // Solved tiles are pushed into the peers' slots; peers are other GPUs (sys_scope = 1,
    // CUDA-IPC-mapped pointers) or virtual ranks sharing one GPU (sys_scope = 0).
    int fast_solve;             // diagonal-tile solve: 0 = exact sub-block path (default),
                                // 1 = fast plain-FP64 attempt first + exact fallback
    int issue_early;            // update ring: refill a stage before (1) / after (0) computing the
                                // current chunk (kernels.cu update_phase; host: plan_prepare)
    int nranks, rank, sys_scope;
    double* peerY[kMaxRanks];
    int* peerYexp[kMaxRanks];
    double* peerYnorm[kMaxRanks];
    int* peerState[kMaxRanks];
    int* peerErr[kMaxRanks];
};

__host__ __device__ __forceinline__ long long tri_slot(int i, int k) {
    return (long long)k * (k + 1) / 2 + i;
}

}  // namespace rsb
