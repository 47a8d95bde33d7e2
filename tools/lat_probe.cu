// Latency microbenchmark (single warp): dependent DFMA, DADD, DDIV, LDS chains on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, double x0) {
    __shared__ double sm[1024];
    __shared__ int idx[1024];
    for (int t = threadIdx.x; t < 1024; t += 32) { sm[t] = 1.0 + t * 1e-9; idx[t] = (t * 37 + 11) & 1023; }
    __syncwarp();
    double a = x0, b = 1.0000001, c = 1e-9;
    long long t0 = clock64();
    for (int i = 0; i < 1024; ++i) a = fma(a, b, c);
    long long t1 = clock64();
    for (int i = 0; i < 1024; ++i) a = a + c;
    long long t2 = clock64();
    for (int i = 0; i < 256; ++i) a = b / a;
    long long t3 = clock64();
    int p = threadIdx.x;
    for (int i = 0; i < 1024; ++i) p = idx[p];
    long long t4 = clock64();
    double s = 0;
    for (int i = 0; i < 1024; ++i) s = fma(sm[(p + i) & 1023], s, c);  // LDS feeding a DFMA chain
    long long t5 = clock64();
    out[threadIdx.x] = a + p + s;
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; }
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 256); cudaMalloc(&c, 64);
    k<<<1, 32>>>(o, c, 1.0); k<<<1, 32>>>(o, c, 1.0); cudaDeviceSynchronize();
    long long h[5]; cudaMemcpy(h, c, 40, cudaMemcpyDeviceToHost);
    printf("DFMA dep: %.1f cyc, DADD dep: %.1f cyc, DDIV dep: %.1f cyc, LDS chase: %.1f cyc, LDS->DFMA chain: %.1f cyc\n",
           h[0] / 1024.0, h[1] / 1024.0, h[2] / 256.0, h[3] / 1024.0, h[4] / 1024.0);
    return 0;
}
