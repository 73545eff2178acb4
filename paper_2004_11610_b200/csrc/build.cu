// build.cu -- fill the tensor-core tiles of the compressed operator (precompute).
//
// Output axis (XC_DIR_A, Alg. 2 / block form): an item covers one group of 4 bins
// [4g, 4g+4) and a node range; its A fragment for step s is
//     A[row][kk] = comp(row&1) of S[k0 + 4s + kk][4g + row/2]     (0 outside the band)
// Tail (direct method for degrees [0, t)): groups of 8 degrees,
//     A[row][kk] = phi_{8g+row}(x_{k0+4s+kk}).
// Input axis (XC_DIR_WAT, Alg. 1 / block form): an item covers 8 nodes [8g, 8g+8)
// and a bin range; the half spectrum is folded with c_q = 1 (q = 0, L/2) or 2:
//     A[row][kk] = c_q Re S[node][q]   (kk even)  |  -c_q Im S[node][q]   (kk odd),
//     node = 8g + row, q = k0 + 2s + kk/2
// and its tail A[row][kk] = phi_{k0+4s+kk}(x_{8g+row}).
// In every case lane l of a warp holds A[l/4][l%4] (spmm.cu).
#include "build.h"
#include "xc_internal.cuh"

namespace {

__device__ __forceinline__ double band_val(int k, int q, int comp, const int* start, const int* len,
                                           const int64_t* off, const double2* vals) {
  int s = start[k];
  if (q < s || q >= s + len[k]) return 0.0;
  double2 v = vals[off[k] + (q - s)];
  return comp ? v.y : v.x;
}

__global__ void fill_out_cplx(const FillItem* fi, const int* start, const int* len, const int64_t* off,
                              const double2* vals, int N, int H, double* tiles) {
  const FillItem it = fi[blockIdx.x];
  for (int idx = threadIdx.x; idx < it.nsteps * 32; idx += blockDim.x) {
    int s = idx >> 5, lane = idx & 31;
    int k = it.k0 + 4 * s + (lane & 3);
    int row = lane >> 2;
    int q = 4 * it.g + (row >> 1);
    double v = 0.0;
    if (k < N && q < H) v = band_val(k, q, row & 1, start, len, off, vals);
    tiles[it.a_off + idx] = v;
  }
}

__global__ void fill_out_real(const FillItem* fi, const double* P, int t, int N, double* tiles) {
  const FillItem it = fi[blockIdx.x];
  for (int idx = threadIdx.x; idx < it.nsteps * 32; idx += blockDim.x) {
    int s = idx >> 5, lane = idx & 31;
    int k = it.k0 + 4 * s + (lane & 3);
    int j = 8 * it.g + (lane >> 2);
    tiles[it.a_off + idx] = (k < N && j < t) ? P[(int64_t)j * N + k] : 0.0;
  }
}

__global__ void fill_in_cplx(const FillItem* fi, const int* start, const int* len, const int64_t* off,
                             const double2* vals, int N, int H, double* tiles) {
  const FillItem it = fi[blockIdx.x];
  for (int idx = threadIdx.x; idx < it.nsteps * 32; idx += blockDim.x) {
    int s = idx >> 5, lane = idx & 31;
    int node = 8 * it.g + (lane >> 2);
    int kk = lane & 3;
    int q = it.k0 + 2 * s + (kk >> 1);
    double v = 0.0;
    if (node < N && q < H) {
      double c = (q == 0 || q == H - 1) ? 1.0 : 2.0;
      double a = band_val(node, q, kk & 1, start, len, off, vals);
      v = (kk & 1) ? -c * a : c * a;
    }
    tiles[it.a_off + idx] = v;
  }
}

__global__ void fill_in_real(const FillItem* fi, const double* P, int t, int N, double* tiles) {
  const FillItem it = fi[blockIdx.x];
  for (int idx = threadIdx.x; idx < it.nsteps * 32; idx += blockDim.x) {
    int s = idx >> 5, lane = idx & 31;
    int node = 8 * it.g + (lane >> 2);
    int j = it.k0 + 4 * s + (lane & 3);
    tiles[it.a_off + idx] = (node < N && j < t) ? P[(int64_t)j * N + node] : 0.0;
  }
}

}  // namespace

xc_status fill_tiles(int mode, const FillItem* fi, int n, const int* start, const int* len, const int64_t* off,
                     const double2* vals, const double* P, int t, int N, int H, double* tiles, cudaStream_t st) {
  if (n <= 0) return XC_OK;
  switch (mode) {
    case FILL_OUT_CPLX: fill_out_cplx<<<n, 128, 0, st>>>(fi, start, len, off, vals, N, H, tiles); break;
    case FILL_OUT_REAL: fill_out_real<<<n, 128, 0, st>>>(fi, P, t, N, tiles); break;
    case FILL_IN_CPLX: fill_in_cplx<<<n, 128, 0, st>>>(fi, start, len, off, vals, N, H, tiles); break;
    default: fill_in_real<<<n, 128, 0, st>>>(fi, P, t, N, tiles); break;
  }
  XC_CUDA(cudaGetLastError());
  return XC_OK;
}
