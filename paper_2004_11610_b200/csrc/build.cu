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
// In every case lane l of a warp holds A[l/4][l%4] (spmm.cu); an item carries two M-tiles
// (or one), interleaved per lane; each M-tile is filled from its own family's bands.  Steps come
// in pairs: steps 2k, 2k+1 of lane l are the 4 doubles at a_off + 128 k + 4 l (slot 0, slot 1 of
// step 2k, then of step 2k+1), one 32-byte load per lane for two steps (an odd step count is
// padded with a zero step).
#include "build.h"
#include "xc_internal.cuh"

namespace {

// entry of bin q of node k's run [s, s + len) -- taken mod H: runs of complex rows may wrap
__device__ __forceinline__ double2 band_cval(int k, int q, int H, const int* start, const int* len,
                                            const int64_t* off, const double2* vals) {
  int d = q - start[k];
  if (d < 0) d += H;
  if (d >= len[k]) return make_double2(0.0, 0.0);
  return vals[off[k] + d];
}
__device__ __forceinline__ double band_val(int k, int q, int comp, int H, const int* start, const int* len,
                                           const int64_t* off, const double2* vals) {
  const double2 v = band_cval(k, q, H, start, len, off, vals);
  return comp ? v.y : v.x;
}

__device__ __forceinline__ int64_t tile_at(int64_t a_off, int s, int lane, int mt) {
  return a_off + 64 * (s & ~1) + 4 * lane + 2 * (s & 1) + mt;
}

// lane l of a warp holds A[l/4][l%4] of each M-tile: row r = l/4, B row R = k0 + 4s + l%4
template <int MODE>
__global__ void fill_k(const FillItem* fi, const int* start, const int* len, const int64_t* off,
                       const double2* vals, const double* P, int t, int N, int H, double* tiles) {
  const FillItem it = fi[blockIdx.x];
  for (int idx = threadIdx.x; idx < it.nsteps * 32; idx += blockDim.x) {
    const int s = idx >> 5, lane = idx & 31, gm = it.g;
    double v = 0.0;
    const int R = it.k0 + 4 * s + (lane & 3);
    const int r = lane >> 2;
    if (R < it.lo || R >= it.hi) {
      tiles[tile_at(it.a_off, s, lane, it.mt)] = 0.0;
      continue;
    }
    if (MODE == FILL_OUT_CPLX) {        // node R, bin 4 gm + r/2, component r&1
      int q = 4 * gm + (r >> 1);
      if (R < N && q < H) v = band_val(R, q, r & 1, H, start, len, off, vals);
    } else if (MODE == FILL_OUT_CC) {   // XC_EXP: B row R = (node R/2, re/im of X); row r = (bin, re/im of u)
      const int node = R >> 1, xc = R & 1, q = 4 * gm + (r >> 1), uc = r & 1;
      if (node < N && q < H) {
        const double2 sv = band_cval(node, q, H, start, len, off, vals);
        // u_re = S_re X_re - S_im X_im,  u_im = S_im X_re + S_re X_im
        v = uc == 0 ? (xc == 0 ? sv.x : -sv.y) : (xc == 0 ? sv.y : sv.x);
      }
    } else if (MODE == FILL_OUT_REAL) { // node R, degree 8 gm + r
      int j = 8 * gm + r;
      if (R < N && j < t) v = P[(int64_t)j * N + R];
    } else if (MODE == FILL_IN_CC) {    // XC_EXP input axis: gm = 2 G + part, node 8 G + r, bin R/2
      // Y = sum_q S z'_q: part 0 rows Re Y = S_re z'_re - S_im z'_im, part 1 rows Im Y = S_im z'_re + S_re z'_im
      const int node = 8 * (gm >> 1) + r, part = gm & 1, q = R >> 1, pl = R & 1;
      if (node < N && q < H) {
        const double2 sv = band_cval(node, q, H, start, len, off, vals);
        v = part == 0 ? (pl == 0 ? sv.x : -sv.y) : (pl == 0 ? sv.y : sv.x);
      }
    } else if (MODE == FILL_IN_CPLX) {  // node 8 gm + r, bin R/2, (c Re S, -c Im S)
      int node = 8 * gm + r, q = R >> 1;
      if (node < N && q < H) {
        double c = (q == 0 || q == H - 1) ? 1.0 : 2.0;
        double a = band_val(node, q, R & 1, H, start, len, off, vals);
        v = (R & 1) ? -c * a : c * a;
      }
    } else {                            // node 8 gm + r, degree R
      int node = 8 * gm + r;
      if (node < N && R < t) v = P[(int64_t)R * N + node];
    }
    tiles[tile_at(it.a_off, s, lane, it.mt)] = v;
  }
}

}  // namespace

xc_status fill_tiles(int mode, const FillItem* fi, int n, const int* start, const int* len, const int64_t* off,
                     const double2* vals, const double* P, int t, int N, int H, double* tiles, cudaStream_t st) {
  if (n <= 0) return XC_OK;
  switch (mode) {
    case FILL_OUT_CPLX: fill_k<FILL_OUT_CPLX><<<n, 128, 0, st>>>(fi, start, len, off, vals, P, t, N, H, tiles); break;
    case FILL_OUT_REAL: fill_k<FILL_OUT_REAL><<<n, 128, 0, st>>>(fi, start, len, off, vals, P, t, N, H, tiles); break;
    case FILL_IN_CPLX: fill_k<FILL_IN_CPLX><<<n, 128, 0, st>>>(fi, start, len, off, vals, P, t, N, H, tiles); break;
    case FILL_OUT_CC: fill_k<FILL_OUT_CC><<<n, 128, 0, st>>>(fi, start, len, off, vals, P, t, N, H, tiles); break;
    case FILL_IN_CC: fill_k<FILL_IN_CC><<<n, 128, 0, st>>>(fi, start, len, off, vals, P, t, N, H, tiles); break;
    default: fill_k<FILL_IN_REAL><<<n, 128, 0, st>>>(fi, start, len, off, vals, P, t, N, H, tiles); break;
  }
  XC_CUDA(cudaGetLastError());
  return XC_OK;
}
