// rsylv-b200 utility kernels (sm_100a): a general FP64 GEMM on the DMMA tensor path and the
// reductions of the overflow-safe relative residual.
//
// * k_dgemm: C = alpha * op(A) * op(B) + beta * C, column-major, op = N or T. One 512-thread
//   CTA per 128 x 128 tile of C, 16 warps of 32 x 32 DMMA (mma.sync.m8n8k4.f64) accumulators,
//   a 3-stage cp.async ring of 32-deep K chunks (zero-filled at the edges, 8-byte copies so any
//   leading dimension / alignment works). Structural zeros are skipped: `a_upper` (A upper
//   quasi-triangular: A(i, k) = 0 for k < i - 1) and `b_upper` (B(k, j) = 0 for k > j + 1)
//   restrict the K range of each tile, which halves the triangular products of the residual
//   A Y + Y B. Used by rsylv_b200_relative_residual (the residual of src/testgen.cpp:64-79,
//   evaluated in a power-of-two prescaled frame) and the Bartels-Stewart transforms.
// * k_scale_copy / k_absmax / k_sumsq: elementwise exact power-of-two scaling and the
//   max / scaled sum-of-squares reductions of the Frobenius norms.
#include <cstdio>

#include "common.cuh"

namespace rsb {

namespace {

constexpr int GBM = 128, GKC = 32, GST = 3, GTH = 512;
constexpr int GLDA = GBM + 4;  // A stage [GKC][GLDA]: rows contiguous (fragment reads conflict-free)
constexpr int GLDB = GKC + 4;  // B stage [GBM][GLDB]: k contiguous

struct GSmem {
    double A[GST][GKC][GLDA];
    double B[GST][GBM][GLDB];
};

__device__ __forceinline__ void dmma_g(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

// 8-byte async copy, zero-filled when `valid` is false (src-size 0)
__device__ __forceinline__ void cp_async8(void* smem, const double* gmem, bool valid) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    const int n = valid ? 8 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(n)
                 : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

}  // namespace

__global__ void __launch_bounds__(GTH, 1)
    k_dgemm(int ta, int tb, int m, int n, int k, double alpha, const double* __restrict__ A,
            long long lda, const double* __restrict__ B, long long ldb, double beta,
            double* __restrict__ C, long long ldc, int a_upper, int b_upper) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    GSmem& sm = *reinterpret_cast<GSmem*>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, q = lane & 3, wm = warp >> 2, wn = warp & 3;
    const int i0 = blockIdx.x * GBM, j0 = blockIdx.y * GBM;
    // K range holding nonzeros of this tile's row / column block
    int klo = 0, khi = k;
    if (a_upper) klo = max(klo, i0 - 1);
    if (b_upper) khi = min(khi, j0 + GBM + 1);
    klo = klo / GKC * GKC;
    const int nch = khi > klo ? (khi - klo + GKC - 1) / GKC : 0;

    auto load = [&](int stage, int ch) {
        const int k0 = klo + ch * GKC;
        // A stage: As[kk][r] = op(A)(i0 + r, k0 + kk)
#pragma unroll
        for (int t = 0; t < GKC * GBM / GTH; ++t) {
            const int e = tid + t * GTH;
            int r, kk;
            if (!ta) {  // consecutive threads along rows (column-major A: contiguous)
                r = e % GBM;
                kk = e / GBM;
            } else {    // along k (A^T: A(k, i) contiguous in k)
                kk = e % GKC;
                r = e / GKC;
            }
            const int gi = i0 + r, gk = k0 + kk;
            const bool v = gi < m && gk < khi;
            const double* src = ta ? A + gk + (long long)gi * lda : A + gi + (long long)gk * lda;
            cp_async8(&sm.A[stage][kk][r], v ? src : A, v);
        }
        // B stage: Bs[c][kk] = op(B)(k0 + kk, j0 + c)
#pragma unroll
        for (int t = 0; t < GKC * GBM / GTH; ++t) {
            const int e = tid + t * GTH;
            int c, kk;
            if (!tb) {  // along k (column-major B: contiguous)
                kk = e % GKC;
                c = e / GKC;
            } else {    // along columns (B^T: B(j, k) contiguous in j)
                c = e % GBM;
                kk = e / GBM;
            }
            const int gj = j0 + c, gk = k0 + kk;
            const bool v = gj < n && gk < khi;
            const double* src = tb ? B + gj + (long long)gk * ldb : B + gk + (long long)gj * ldb;
            cp_async8(&sm.B[stage][c][kk], v ? src : B, v);
        }
    };

    double acc[4][4][2];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;

#pragma unroll
    for (int s = 0; s < GST - 1; ++s) {
        if (s < nch) load(s, s);
        cp_commit();
    }
#pragma unroll 1
    for (int it = 0; it < nch; ++it) {
        cp_wait<GST - 2>();
        __syncthreads();
        const int st = it % GST;
        if (it + GST - 1 < nch) load((it + GST - 1) % GST, it + GST - 1);
        cp_commit();
        const double(*As)[GLDA] = sm.A[st];
        const double(*Bs)[GLDB] = sm.B[st];
#pragma unroll
        for (int kk = 0; kk < GKC; kk += 4) {
            double a[4], b[4];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi) a[mi] = As[kk + q][wm * 32 + mi * 8 + g];
#pragma unroll
            for (int ni = 0; ni < 4; ++ni) b[ni] = Bs[wn * 32 + ni * 8 + g][kk + q];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi)
#pragma unroll
                for (int ni = 0; ni < 4; ++ni) dmma_g(acc[mi][ni], a[mi], b[ni]);
        }
    }
    cp_wait<0>();
    // epilogue: C = alpha * acc + beta * C (beta == 0: C is not read)
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int r = i0 + wm * 32 + mi * 8 + g, c = j0 + wn * 32 + ni * 8 + 2 * q + h;
                if (r < m && c < n) {
                    double* p = C + r + (long long)c * ldc;
                    const double v = alpha * acc[mi][ni][h];
                    *p = beta == 0.0 ? v : fma(beta, *p, v);
                }
            }
}

// dst = src * 2^e (exact for normal results), column-major m x n
__global__ void k_scale_copy(int m, int n, const double* __restrict__ src, long long lds,
                             double* __restrict__ dst, long long ldd, int e) {
    const int j = blockIdx.y;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x)
        dst[i + (long long)j * ldd] = scale2(src[i + (long long)j * lds], e);
}

// per-block partials of max |x| and of sum (x * 2^e)^2 (column-major m x n); NaN propagates
__global__ void k_absmax_sumsq(int m, int n, const double* __restrict__ x, long long ld, int e,
                               double* __restrict__ pmax, double* __restrict__ psum) {
    double mx = 0.0, s = 0.0;
    const long long total = (long long)m * n;
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const long long j = t / m, i = t - j * m;
        const double v = x[i + j * ld];
        mx = (v != v || mx != mx) ? v : fmax(mx, fabs(v));
        const double w = scale2(v, e);
        s = fma(w, w, s);
    }
    __shared__ double smx[32], ss[32];
    for (int o = 16; o; o >>= 1) {
        const double om = __shfl_xor_sync(0xffffffffu, mx, o);
        mx = (om != om || mx != mx) ? (mx != mx ? mx : om) : fmax(mx, om);
        s += __shfl_xor_sync(0xffffffffu, s, o);
    }
    if ((threadIdx.x & 31) == 0) {
        smx[threadIdx.x >> 5] = mx;
        ss[threadIdx.x >> 5] = s;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double m2 = 0.0, s2 = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            m2 = (smx[w] != smx[w] || m2 != m2) ? (m2 != m2 ? m2 : smx[w]) : fmax(m2, smx[w]);
            s2 += ss[w];
        }
        pmax[blockIdx.x] = m2;
        psum[blockIdx.x] = s2;
    }
}

size_t smem_gemm() { return sizeof(GSmem); }

cudaError_t launch_dgemm(int ta, int tb, int m, int n, int k, double alpha, const double* A,
                         long long lda, const double* B, long long ldb, double beta, double* C,
                         long long ldc, int a_upper, int b_upper, cudaStream_t st) {
    static bool configured = false;
    if (!configured) {
        const cudaError_t e = cudaFuncSetAttribute(k_dgemm, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   (int)sizeof(GSmem));
        if (e != cudaSuccess) return e;
        configured = true;
    }
    if (m <= 0 || n <= 0) return cudaSuccess;
    dim3 grid((m + GBM - 1) / GBM, (n + GBM - 1) / GBM);
    k_dgemm<<<grid, GTH, sizeof(GSmem), st>>>(ta, tb, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc,
                                              a_upper, b_upper);
    return cudaGetLastError();
}

cudaError_t launch_scale_copy(int m, int n, const double* src, long long lds, double* dst,
                              long long ldd, int e, cudaStream_t st) {
    if (m <= 0 || n <= 0) return cudaSuccess;
    dim3 grid((m + 255) / 256 < 64 ? (m + 255) / 256 : 64, n);
    k_scale_copy<<<grid, 256, 0, st>>>(m, n, src, lds, dst, ldd, e);
    return cudaGetLastError();
}

cudaError_t launch_absmax_sumsq(int m, int n, const double* x, long long ld, int e, int blocks,
                                double* pmax, double* psum, cudaStream_t st) {
    k_absmax_sumsq<<<blocks, 512, 0, st>>>(m, n, x, ld, e, pmax, psum);
    return cudaGetLastError();
}

}  // namespace rsb
