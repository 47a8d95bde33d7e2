// FP64 peak microbenchmark for B200 (sm_100a): DMMA (mma.sync f64 -> SASS DMMA.8x8x4)
// versus plain DFMA. Used to ground the FP64 roofline denominator (MEASURED_PEAKS.json
// carries only HBM and bf16 figures). Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); return 1; } } while (0)

template <int NACC>
__global__ void dmma_peak(double* out, int iters, double seed) {
  double acc[NACC][2];
  double a = seed + threadIdx.x * 1e-9, b = seed - threadIdx.x * 1e-9;
#pragma unroll
  for (int i = 0; i < NACC; ++i) { acc[i][0] = 0.0; acc[i][1] = 0.0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += acc[i][0] + acc[i][1];
  if (s == 1234.5) out[0] = s;
}

template <int NACC>
__global__ void dfma_peak(double* out, int iters, double seed) {
  double acc[NACC];
  double a = seed + threadIdx.x * 1e-9, b = 1.0 - 1e-12;
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) acc[i] = fma(acc[i], b, a);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += acc[i];
  if (s == 1234.5) out[0] = s;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  double* out; CK(cudaMalloc(&out, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 20000;
  for (int wpb : {4, 8, 16}) {
    for (int bps : {1, 2}) {
      int blocks = sms * bps, threads = 32 * wpb;
      dmma_peak<8><<<blocks, threads>>>(out, 100, 1.0);
      CK(cudaDeviceSynchronize());
      cudaEventRecord(e0);
      dmma_peak<8><<<blocks, threads>>>(out, iters, 1.0);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 256.0 * 8 * iters * (double)blocks * wpb;
      std::printf("DMMA  warps/blk=%2d blk/SM=%d : %.2f TFLOP/s (%.3f ms)\n", wpb, bps, flops / ms / 1e9, ms);
    }
  }
  for (int wpb : {8, 16, 32}) {
    int blocks = sms * 2, threads = 32 * wpb;
    dfma_peak<8><<<blocks, threads>>>(out, 100, 1.0);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    dfma_peak<8><<<blocks, threads>>>(out, iters, 1.0);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * iters * (double)blocks * threads;
    std::printf("DFMA  warps/blk=%2d blk/SM=2 : %.2f TFLOP/s (%.3f ms)\n", wpb, flops / ms / 1e9, ms);
  }
  std::printf("SMs=%d clock(kHz)=%d\n", sms, clk);
  return 0;
}
