// PCIe probe: 2D (column-chunk) host<->device copies, DMA vs copy kernel, alone and concurrent.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void mv(const double2* s, long lds, double2* d, long ldd, long n, int h) {
  long tot = n * h;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < tot; i += (long)gridDim.x * blockDim.x) {
    long r = i / h; int c = (int)(i - r * h);
    d[r * ldd + c] = s[r * lds + c];
  }
}
int main() {
  const long N = 65536, B = 4096, bc = 512;
  double *xh, *yh, *xd, *yd;
  cudaHostAlloc(&xh, N * B * 8, 0); cudaHostAlloc(&yh, N * B * 8, 0);
  cudaMalloc(&xd, N * bc * 8 * 2); cudaMalloc(&yd, N * bc * 8 * 2);
  cudaStream_t s1, s2; cudaStreamCreate(&s1); cudaStreamCreate(&s2);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  double gb = N * B * 8 / 1e9;
  for (int mode = 0; mode < 6; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaDeviceSynchronize(); cudaEventRecord(a, 0); cudaStreamWaitEvent(s1, a, 0); cudaStreamWaitEvent(s2, a, 0);
      for (long c0 = 0; c0 < B; c0 += bc) {
        int i = (c0 / bc) & 1;
        bool in = mode == 0 || mode == 2 || mode == 3 || mode == 5, out = mode == 1 || mode == 2 || mode == 4 || mode == 5;
        bool ker = mode >= 3;
        if (in) { if (ker) mv<<<64, 256, 0, s1>>>((const double2*)(xh + c0), B / 2, (double2*)(xd + i * N * bc), bc / 2, N, bc / 2);
                  else cudaMemcpy2DAsync(xd + i * N * bc, bc * 8, xh + c0, B * 8, bc * 8, N, cudaMemcpyHostToDevice, s1); }
        if (out) { if (ker) mv<<<64, 256, 0, s2>>>((const double2*)(yd + i * N * bc), bc / 2, (double2*)(yh + c0), B / 2, N, bc / 2);
                   else cudaMemcpy2DAsync(yh + c0, B * 8, yd + i * N * bc, bc * 8, bc * 8, N, cudaMemcpyDeviceToHost, s2); }
      }
      cudaEventRecord(b, s1); cudaStreamWaitEvent(0, b, 0); cudaEventRecord(b, s2); cudaStreamWaitEvent(0, b, 0);
      cudaEventRecord(b, 0); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (rep) printf("%s %s: %.1f ms  (%.1f GB/s per direction)\n", mode >= 3 ? "kernel" : "dma2d",
                      (mode % 3) == 0 ? "H2D" : (mode % 3) == 1 ? "D2H" : "both", ms, gb / (ms / 1e3));
    }
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
