// stride_probe.cu -- DRAM bandwidth of the C2R passes' access pattern: a CTA copies tiles of R rows x
// cb complex columns (16 B each), rows `stride` bytes apart, from one 2.8 GB array to another (the
// same pattern on both sides), persistent grid, cp.async-free plain 16-B loads/stores.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o stride_probe tools/stride_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void probe(const double2* __restrict__ in, double2* __restrict__ out, long rows, long cols, int R,
                      int cb, long ntiles, int blocked) {
  // tile t: column block (t % (cols / cb)), rows [ (t / (cols/cb)) * R, + R )
  const long ncb = cols / cb;
  for (long t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const long c0 = (t % ncb) * cb, r0 = (t / ncb) * R;
    for (int i = threadIdx.x; i < R * cb; i += blockDim.x) {
      const int r = i / cb, c = i - r * cb;
      long a;
      if (blocked) a = (c0 / cb) * rows * cb + (r0 + r) * cb + c;  // [colblock][row][cb]
      else a = (r0 + r) * cols + c0 + c;                              // [row][col]
      out[a] = in[a];
    }
  }
}

int main() {
  const long cols = 4096, rows = 43200;
  double2 *a, *b;
  cudaMalloc(&a, rows * cols * 16);
  cudaMalloc(&b, rows * cols * 16);
  cudaMemset(a, 0, rows * cols * 16);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int nsm = 148;
  for (int blocked = 0; blocked < 2; ++blocked)
    for (int cb : {4, 8, 16, 32})
      for (int R : {200, 216}) {
        const long ntiles = (rows / R) * (cols / cb);
        probe<<<nsm * 4, 256>>>(a, b, rows, cols, R, cb, ntiles, blocked);
        cudaEventRecord(e0);
        for (int it = 0; it < 5; ++it) probe<<<nsm * 4, 256>>>(a, b, rows, cols, R, cb, ntiles, blocked);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double bytes = 2.0 * (rows / R) * R * cols * 16 * 5;
        printf("layout %s cb %2d (%4d B rows) R %d: %.0f GB/s\n", blocked ? "blocked" : "row-major", cb, cb * 16, R,
               bytes / (ms * 1e-3) / 1e9);
      }
  return 0;
}
