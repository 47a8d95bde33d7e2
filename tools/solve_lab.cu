// Development lab (not product code): throughput/latency probes for the building blocks of the
// diagonal-tile solve and candidate 16x16 sub-block solvers, timed on one SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo tools/solve_lab.cu -o tools/solve_lab
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define FULL 0xffffffffu

// ---------------------------------------------------------------------------- probes
// nw warps, each issues n independent (4 chains) 64-bit shuffles / LDS.64 / DFMA.
__global__ void k_tput(int n, int kind, double* out, long long* cyc) {
    __shared__ double sm[4096];
    for (int t = threadIdx.x; t < 4096; t += blockDim.x) sm[t] = 1.0 + t;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    double a0 = lane, a1 = lane + 1, a2 = lane + 2, a3 = lane + 3;
    int i0 = lane, i1 = lane + 32, i2 = lane + 64, i3 = lane + 96;
    __syncthreads();
    long long t0 = clock64();
    if (kind == 0) {
        for (int i = 0; i < n; ++i) {
            a0 = __shfl_sync(FULL, a0, (lane + 1) & 31);
            a1 = __shfl_sync(FULL, a1, (lane + 3) & 31);
            a2 = __shfl_sync(FULL, a2, (lane + 5) & 31);
            a3 = __shfl_sync(FULL, a3, (lane + 7) & 31);
        }
    } else if (kind == 1) {
        for (int i = 0; i < n; ++i) {
            a0 += sm[i0];
            a1 += sm[i1];
            a2 += sm[i2];
            a3 += sm[i3];
            i0 = (i0 + 32) & 4095;
            i1 = (i1 + 32) & 4095;
            i2 = (i2 + 32) & 4095;
            i3 = (i3 + 32) & 4095;
        }
    } else if (kind == 2) {
        double b0 = 1.0000001;
        for (int i = 0; i < n; ++i) {
            a0 = fma(a0, b0, 1e-9);
            a1 = fma(a1, b0, 1e-9);
            a2 = fma(a2, b0, 1e-9);
            a3 = fma(a3, b0, 1e-9);
        }
    } else if (kind == 3) {  // dependent 64-bit shuffle chain (latency)
        for (int i = 0; i < n; ++i) a0 = __shfl_sync(FULL, a0, (lane + 1) & 31);
    } else if (kind == 4) {  // dependent dfma chain
        for (int i = 0; i < n; ++i) a0 = fma(a0, 1.0000001, 1e-9);
    } else if (kind == 5) {  // dependent LDS chain (address from value)
        int p = lane;
        for (int i = 0; i < n; ++i) p = (int)sm[p] & 4095;
        a0 = p;
    } else if (kind == 6) {  // shuffle -> dfma dependent chain
        for (int i = 0; i < n; ++i) a0 = fma(__shfl_sync(FULL, a0, (lane + 1) & 31), 0.5, 1.0);
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + i0 + i1 + i2 + i3;
    if (lane == 0) cyc[threadIdx.x >> 5] = t1 - t0;
}

// ---------------------------------------------------------------------------- solvers
// Problem for one 16x16 sub-block: A (16x16 upper, ld 16), B (16x16 upper, ld 17), C (16x16,
// ld 129), all 1x1 blocks. X overwrites C.
constexpr int LDW = 129, LDA = 16, LDB = 17;

// Register-skew wavefront, two sub-blocks per warp (one per 16-lane half). Lane r holds row r
// skewed: R[k] = element (r, k - 15 + r), solved at step k. Column direction: the value x just
// solved by lane r + d lands in R[s + d] (shfl_down by d). Row direction: in-lane, coefficient
// B(c, c + e) with the lane's current column c (kBLds: from shared memory; else shuffled from
// lane c, which holds row c of B).
template <bool kBLds, bool kWin = false>
__device__ __forceinline__ bool skew16(double* W, const double* Ad, const double* Bd, int pr,
                                       int qc, double small_num, double limit) {
    const int r = threadIdx.x & 15;
    double Ask[16];
#pragma unroll
    for (int d = 0; d < 16; ++d) Ask[d] = (r + d < pr) ? Ad[r + (r + d) * LDA] : 0.0;
    double Brow[16];
    if (!kBLds) {
#pragma unroll
        for (int e = 0; e < 16; ++e) Brow[e] = (r + e < qc) ? Bd[r + (r + e) * LDB] : 0.0;
    } else {
        Brow[0] = r < qc ? Bd[r + r * LDB] : 0.0;
    }
    constexpr int NR = kWin ? 16 : 31;
    double R[NR];
    auto init = [&](int k) {
        const int c = k - 15 + r;
        return (r < pr && c >= 0 && c < qc) ? W[r + c * LDW] : 0.0;
    };
#pragma unroll
    for (int k = 0; k < NR; ++k) R[k] = init(k);
    bool ok = true;
#pragma unroll
    for (int s = 0; s < 31; ++s) {
        const int c = s - 15 + r;
        const bool act = r < pr && c >= 0 && c < qc;
        const int cs = min(max(c, 0), 15);
        const double bcc = __shfl_sync(FULL, Brow[0], cs, 16);
        const double den = Ask[0] + bcc;
        const double rc = 1.0 / den;
        ok &= !act || fabs(den) >= small_num;
        const double x = act ? R[s % NR] * rc : 0.0;
        ok &= !act || fabs(x) <= limit;
        if (act) W[r + c * LDW] = x;
#pragma unroll
        for (int d = 1; d < 16; ++d)
            if (s + d < 31) {
                const double v = __shfl_down_sync(FULL, x, d, 16);
                R[(s + d) % NR] = fma(-Ask[d], v, R[(s + d) % NR]);
            }
#pragma unroll
        for (int e = 1; e < 16; ++e)
            if (s + e < 31) {
                double b;
                if (kBLds)
                    b = (cs + e < 16) ? Bd[cs + (cs + e) * LDB] : 0.0;
                else
                    b = __shfl_sync(FULL, Brow[e], cs, 16);
                R[(s + e) % NR] = fma(-x, b, R[(s + e) % NR]);
            }
        if (kWin && s + 16 <= 30) R[s % NR] = init(s + 16);
    }
    return ok;
}

// One warp per pair of sub-blocks; nblk sub-block problems laid out consecutively.
template <int kVariant>
__global__ void k_solve(int nblk, int reps, double* Cg, const double* Ag, const double* Bg,
                        long long* cyc, int* okout, const unsigned char* codes1) {
    extern __shared__ double sh[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, half = lane >> 4;
    const int nw = blockDim.x >> 5;
    double* Wb = sh;                        // nw*2 blocks of 16 x LDW
    double* Ab = Wb + nw * 2 * 16 * LDW;    // nw*2 blocks of 16*LDA
    double* Bb = Ab + nw * 2 * 16 * LDA;    // nw*2 blocks of 16*LDB
    const int blk = (blockIdx.x * nw + warp) * 2 + half;
    double* W = Wb + (warp * 2 + half) * 16 * LDW;
    double* A = Ab + (warp * 2 + half) * 16 * LDA;
    double* B = Bb + (warp * 2 + half) * 16 * LDB;
    const int r = lane & 15;
    long long tot = 0;
    bool ok = true;
    for (int rep = 0; rep < reps; ++rep) {
        for (int c = 0; c < 16; ++c) {
            W[r + c * LDW] = Cg[(long long)blk * 256 + r + c * 16];
            A[r + c * LDA] = Ag[(long long)blk * 256 + r + c * 16];
            B[r + c * LDB] = Bg[(long long)blk * 256 + r + c * 16];
        }
        __syncwarp();
        const long long t0 = clock64();
        if (kVariant == 0) ok &= skew16<false>(W, A, B, 16, 16, 1e-290, 1e300);
        if (kVariant == 1) ok &= skew16<true>(W, A, B, 16, 16, 1e-290, 1e300);
        if (kVariant == 2) ok &= skew16<false, true>(W, A, B, 16, 16, 1e-290, 1e300);
        if (kVariant == 3) ok &= skew16<true, true>(W, A, B, 16, 16, 1e-290, 1e300);

        __syncwarp();
        tot += clock64() - t0;
        if (rep == 0 && lane == 0) cyc[64 + blockIdx.x * nw + warp] = clock64() - t0;
    }
    for (int c = 0; c < 16; ++c) Cg[(long long)blk * 256 + r + c * 16] = W[r + c * LDW];
    if (lane == 0) cyc[blockIdx.x * nw + warp] = tot / reps;
    if (!ok) atomicAdd(okout, 1);
}

#ifndef KSDL_BOUNDS
#define KSDL_BOUNDS __launch_bounds__(512, 1)
#endif
// The DAG's layout for a 16-wide register-wavefront solve: the sub-block inside a 128 x 129 tile
// at (r0, c0), A / B diagonal sub-blocks in 9 x 16 x 16 / 9 x 16 x 17 arrays, 16 warps of which
// `nact` solve (the others wait at the barrier, like the DAG's non-solver warps). Round 2 ran the
// package's 16-wide fast_subsolve_1x1 here: 13.9 k cycles per call when the compiler may use 165
// registers (-DKSDL_BOUNDS=), 37.5 k under __launch_bounds__(512, 1) (125 registers).
// skew16<true, true> is the same algorithm in this file.
template <int kSepW>
__global__ void KSDL_BOUNDS k_solve_daglayout(int nact, int reps, const double* Cg,
                                              const double* Ag, const double* Bg,
                                              long long* cyc) {
    extern __shared__ double sh[];
    double* T = sh;                            // 128 x 129
    double* Ad = T + 128 * 129;                // 9 x 16 x 16
    double* Bd = Ad + 9 * 16 * 16;             // 9 x 16 x 17
    const int warp = threadIdx.x >> 5;
    long long tot = 0;
    for (int rep = 0; rep < reps; ++rep) {
        for (int e = threadIdx.x; e < 128 * 128; e += blockDim.x) T[(e & 127) + (e >> 7) * 129] = Cg[e & 255];
        for (int e = threadIdx.x; e < 9 * 256; e += blockDim.x) {
            const int p = e / 256, r = e % 16, c = (e / 16) % 16;
            Ad[p * 256 + r + c * 16] = Ag[r + c * 16];
            Bd[p * 272 + r + c * 17] = Bg[r + c * 16];
        }
        __syncthreads();
        const long long t0 = clock64();
        if (warp < nact) {
            const int qb = warp, pb = qb;
            double* W = kSepW ? T + warp * 16 * 129 : T + pb * 16 + qb * 16 * 129;
            skew16<true, true>(W, Ad + pb * 256, Bd + qb * 272, 16, 16, 1e-290, 1e300);
        }
        __syncthreads();
        tot += clock64() - t0;
    }
    if (threadIdx.x == 0) cyc[0] = tot / reps;
}

// ---------------------------------------------------------------------------- host
static void cpu_solve(const double* A, const double* B, double* C) {
    // 1x1 blocks: X(r,c) = (C(r,c) - sum_{p>r} A(r,p) X(p,c) - sum_{q<c} X(r,q) B(q,c)) / (A(r,r)+B(c,c))
    for (int c = 0; c < 16; ++c)
        for (int r = 15; r >= 0; --r) {
            double v = C[r + c * 16];
            for (int p = r + 1; p < 16; ++p) v -= A[r + p * 16] * C[p + c * 16];
            for (int q = 0; q < c; ++q) v -= C[r + q * 16] * B[q + c * 16];
            C[r + c * 16] = v / (A[r + r * 16] + B[c + c * 16]);
        }
}

int main(int argc, char** argv) {
    double* dout;
    long long* dcyc;
    cudaMalloc(&dout, 1 << 20);
    cudaMalloc(&dcyc, 1 << 16);
    const char* names[] = {"shfl64 tput", "lds64 tput", "dfma tput", "shfl64 lat", "dfma lat",
                           "lds lat(chase)", "shfl64->dfma lat"};
    for (int kind = 0; kind < 7; ++kind) {
        for (int nw : {1, 4, 8, 16}) {
            if (kind >= 3 && nw > 1) continue;
            const int n = 4096;
            k_tput<<<1, 32 * nw>>>(n, kind, dout, dcyc);
            k_tput<<<1, 32 * nw>>>(n, kind, dout, dcyc);
            cudaDeviceSynchronize();
            std::vector<long long> h(nw);
            cudaMemcpy(h.data(), dcyc, 8 * nw, cudaMemcpyDeviceToHost);
            long long mx = 0;
            for (long long v : h) mx = v > mx ? v : mx;
            const double ops = kind < 3 ? 4.0 * n : n;
            printf("%-18s nw=%2d: %.2f cyc per warp-op (per-warp view), %.3f warp-ops/cyc/SM\n",
                   names[kind], nw, mx / ops, nw * ops / mx);
        }
    }
    // solver benches
    const int nblkmax = 16 * 2;
    std::vector<double> A(nblkmax * 256), B(nblkmax * 256), C(nblkmax * 256), X;
    srand(7);
    auto u = [] { return rand() / (double)RAND_MAX * 2 - 1; };
    for (int b = 0; b < nblkmax; ++b)
        for (int c = 0; c < 16; ++c)
            for (int r = 0; r < 16; ++r) {
                A[b * 256 + r + c * 16] = r < c ? u() : (r == c ? 1.5 + 0.5 * u() : 0.0);
                B[b * 256 + r + c * 16] = r < c ? u() : (r == c ? 1.5 + 0.5 * u() : 0.0);
                C[b * 256 + r + c * 16] = u();
            }
    X = C;
    for (int b = 0; b < nblkmax; ++b) cpu_solve(&A[b * 256], &B[b * 256], &X[b * 256]);
    double *dA, *dB, *dC;
    int* dok;
    cudaMalloc(&dA, A.size() * 8);
    cudaMalloc(&dB, B.size() * 8);
    cudaMalloc(&dC, C.size() * 8);
    cudaMalloc(&dok, 4);
    unsigned char* dcodes;
    cudaMalloc(&dcodes, 64);
    cudaMemset(dcodes, 1, 64);
    cudaMemcpy(dA, A.data(), A.size() * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 8, cudaMemcpyHostToDevice);
    for (int variant = 0; variant < 4; ++variant)
        for (int nw : {1, 4}) {
            const size_t shb = (size_t)nw * 2 * 16 * (LDW + LDA + LDB) * 8;
            cudaMemcpy(dC, C.data(), C.size() * 8, cudaMemcpyHostToDevice);
            cudaMemset(dok, 0, 4);
            auto kf = variant == 0 ? k_solve<0> : variant == 1 ? k_solve<1> : variant == 2 ? k_solve<2> : k_solve<3>;
            cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shb);
            kf<<<1, 32 * nw, shb>>>(nw * 2, 1, dC, dA, dB, dcyc, dok, dcodes);
            cudaDeviceSynchronize();
            std::vector<double> G(C.size());
            cudaMemcpy(G.data(), dC, G.size() * 8, cudaMemcpyDeviceToHost);
            double err = 0;
            for (int i = 0; i < nw * 2 * 256; ++i)
                err = fmax(err, fabs(G[i] - X[i]) / (fabs(X[i]) + 1e-300));
            cudaMemcpy(dC, C.data(), C.size() * 8, cudaMemcpyHostToDevice);
            kf<<<1, 32 * nw, shb>>>(nw * 2, 20, dC, dA, dB, dcyc, dok, dcodes);
            cudaError_t e = cudaDeviceSynchronize();
            std::vector<long long> h(nw);
            cudaMemcpy(h.data(), dcyc, 8 * nw, cudaMemcpyDeviceToHost);
            long long mx = 0;
            for (long long v : h) mx = v > mx ? v : mx;
            int okc = 0;
            cudaMemcpy(&okc, dok, 4, cudaMemcpyDeviceToHost);
            long long first = 0;
            cudaMemcpy(&first, dcyc + 64, 8, cudaMemcpyDeviceToHost);
            printf("first call %lld cycles; ", first);
            printf("skew16 variant %d (B %s%s) nw=%d: %lld cycles per warp (2 sub-blocks), max rel err %.2e, fails %d %s\n",
                   variant, (variant & 1) ? "lds" : "shfl", variant >= 2 ? ", window" : "", nw, mx, err, okc, cudaGetErrorString(e));
        }
    {   // the DAG's layout and warp population
        const size_t shb = (128 * 129 + 9 * 256 + 9 * 272) * 8;
        for (int sep = 0; sep < 2; ++sep) {
            auto kf = sep ? k_solve_daglayout<1> : k_solve_daglayout<0>;
            cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shb);
            for (int nact : {1, 4}) {
                kf<<<1, 512, shb>>>(nact, 1, dC, dA, dB, dcyc);
                kf<<<1, 512, shb>>>(nact, 20, dC, dA, dB, dcyc);
                cudaError_t e = cudaDeviceSynchronize();
                long long h = 0;
                cudaMemcpy(&h, dcyc, 8, cudaMemcpyDeviceToHost);
                printf("daglayout%s 1x1 nact=%d (16 warps): %lld cycles per call %s\n", sep ? "(W separate)" : "", nact, h, cudaGetErrorString(e));
            }
        }
    }
    return 0;
}
