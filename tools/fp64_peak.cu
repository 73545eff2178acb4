// Microbenchmark: sustained fp64 throughput on B200 (DFMA pipe vs DMMA m8n8k4).
// Used to set the "alu"/fp64 roofline peak in DESIGN.md. Not part of the product.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

template<int NACC>
__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double acc[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += acc[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

// half of the warps on DMMA, half on DFMA: are the tensor and CUDA-core fp64 paths separate?
__global__ void mixed_loop(double* out, int iters_mma, int iters_fma, double a0, double b0) {
  const int warp = threadIdx.x >> 5;
  if (warp & 1) {
    double acc[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = threadIdx.x * 1e-9 + i;
    for (int it = 0; it < iters_fma; ++it) {
#pragma unroll
      for (int i = 0; i < 16; ++i) acc[i] = fma(acc[i], a0, b0);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += acc[i];
    if (s == 12345.678) out[0] = s;
  } else {
    double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
    double c[4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i) { c[i][0] = 0; c[i][1] = 0; }
    for (int it = 0; it < iters_mma; ++it) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1];
    if (s == 12345.678) out[0] = s;
  }
}

int main() {
  double* d; CK(cudaMalloc(&d, 8));
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs %d clock(kHz) %d\n", sms, clk);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 20000;
  for (int threads : {256, 512, 1024}) for (int bps : {1, 2, 4}) {
    int grid = sms * bps;
    dfma_loop<16><<<grid, threads>>>(d, 100, 1.0000001, 1e-7);
    cudaEventRecord(e0);
    dfma_loop<16><<<grid, threads>>>(d, iters, 1.0000001, 1e-7);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 16 * iters * (double)grid * threads;
    printf("DFMA threads=%d blocks/SM=%d : %.2f TFLOP/s\n", threads, bps, flops / ms / 1e9);
  }
  for (int threads : {128, 256, 512}) for (int bps : {1, 2, 4}) {
    int grid = sms * bps;
    dmma_loop<<<grid, threads>>>(d, 100);
    cudaEventRecord(e0);
    dmma_loop<<<grid, threads>>>(d, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 8 * 4 * 4 * (double)iters * grid * (threads / 32);
    printf("DMMA threads=%d blocks/SM=%d : %.2f TFLOP/s\n", threads, bps, flops / ms / 1e9);
  }
  // mixed: DMMA warps do iters_mma, DFMA warps iters_fma; report the combined rate
  for (int ratio : {1, 2, 4, 8}) {
    int threads = 512, grid = sms * 2;
    int im = iters, ifm = iters * ratio / 4;
    mixed_loop<<<grid, threads>>>(d, 100, 100, 1.0000001, 1e-7);
    cudaEventRecord(e0);
    mixed_loop<<<grid, threads>>>(d, im, ifm, 1.0000001, 1e-7);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double wpb = threads / 64.0;  // warps of each kind per block
    double fm = 2.0 * 8 * 8 * 4 * 4 * (double)im * grid * wpb;
    double ff = 2.0 * 16 * 32 * (double)ifm * grid * wpb;
    printf("MIXED dfma/dmma iters=%d/4 : dmma %.2f + dfma %.2f = %.2f TFLOP/s\n", ratio, fm / ms / 1e9, ff / ms / 1e9,
           (fm + ff) / ms / 1e9);
  }
  CK(cudaGetLastError());
  return 0;
}
