#include <cstdio>
__global__ void k(double* out, long long* cyc, int n, double a, double inv) {
    double c = threadIdx.x * 0.001 + 1.0;
    const int lane = threadIdx.x & 31;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        const int s = i & 15;
        double z = __shfl_sync(0xffffffffu, c * inv, s);
        c = fma(-a, z, c);
    }
    long long t1 = clock64();
    // dmul + dfma only
    double d = c;
    long long t2 = clock64();
    for (int i = 0; i < n; ++i) { double z = d * inv; d = fma(-a, z, d); }
    long long t3 = clock64();
    // shfl only (double)
    double e = d;
    long long t4 = clock64();
    for (int i = 0; i < n; ++i) { e = __shfl_sync(0xffffffffu, e, (lane + 1) & 31); }
    long long t5 = clock64();
    // int shfl
    int f = lane;
    long long t6 = clock64();
    for (int i = 0; i < n; ++i) { f = __shfl_sync(0xffffffffu, f, (lane + 1) & 31); }
    long long t7 = clock64();
    out[threadIdx.x] = c + d + e + f;
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t3 - t2; cyc[2] = t5 - t4; cyc[3] = t7 - t6; }
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 256); cudaMalloc(&c, 64);
    int n = 4096;
    k<<<1, 32>>>(o, c, n, 0.5, 0.25);
    k<<<1, 32>>>(o, c, n, 0.5, 0.25);
    long long h[4]; cudaMemcpy(h, c, 32, cudaMemcpyDeviceToHost);
    printf("per step: dmul+shfl(double)+dfma %.1f  dmul+dfma %.1f  shfl(double) %.1f  shfl(int) %.1f cycles\n",
           h[0] / (double)n, h[1] / (double)n, h[2] / (double)n, h[3] / (double)n);
}
