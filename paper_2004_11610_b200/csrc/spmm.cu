// spmm.cu -- multiplication by the compressed operator on the FP64 tensor cores.
//
// The hot step of the computation stage (u = Ä_e^T F, Alg. 2 step 2.1, P:218;
// F = Ä_e z, Alg. 1 step 2.2; per block P:281).  "The degree of compression
// ... determines to a great extent the efficiency of the computation step".
//
// The band-sparse operator is pre-tiled (build.cu) into items: an item is an
// 8 x (4*nsteps) dense slice A of the operator (8 output rows = 4 complex bins
// as re/im, or 8 real rows) against 4*nsteps consecutive rows of the operand Bm.
// One warp computes D = A * Bm for 8*NT right-hand sides with DMMA
// (mma.sync.m8n8k4.f64: 37 TF/s measured on B200 vs 34 TF/s for DFMA):
//   A fragment  : lane holds A[lane/4][lane%4]     (one coalesced 256 B load/step)
//   B fragment  : lane holds Bm[lane%4][n], n = lane/4; for DMMA nt the column n is
//                 RHS tile + 16*(nt/2) + 2n + (nt&1): each 16-byte load covers a 128-byte
//                 contiguous run of a row across 8 lanes (coalesced);
//   D fragment  : lane holds D[lane/4][2(lane%4)+i] -> 32 contiguous bytes per nt pair.
// Partial sums of items that split one output group are reduced in fixed order by
// the consumer (FFT prologue / reduce_rows8), so results are deterministic.
#include <algorithm>

#include "xc_internal.cuh"

namespace {

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

constexpr int WPC = 4;  // warps (items) per CTA

template <int NT>
__global__ void __launch_bounds__(WPC * 32) spmm_dmma(const SpmmItem* __restrict__ items, int nitems,
                                                       const double* __restrict__ tiles, SpmmSrcs srcs,
                                                       double* __restrict__ part, int64_t ldp, int ncols) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int it_idx = blockIdx.y * WPC + warp;
  if (it_idx >= nitems) return;
  const SpmmItem it = items[it_idx];
  const int t = lane & 3, g = lane >> 2;
  const int tile0 = blockIdx.x * (8 * NT);

  const double* re = srcs.re[it.src];
  const double* im = srcs.im[it.src];
  const int nrows = srcs.nrows[it.src];
  const int64_t ld = srcs.ld[it.src];
  const bool planes = (im != nullptr);
  const bool full = (tile0 + 8 * NT <= ncols);
  const bool vec_ok = ((ld & 1) == 0) && ((((uintptr_t)re) & 15) == 0) && (!planes || (((uintptr_t)im) & 15) == 0);

  double acc[NT][2];
#pragma unroll
  for (int i = 0; i < NT; ++i) acc[i][0] = acc[i][1] = 0.0;

  // RHS of B-fragment column n for DMMA nt: tile0 + 16*(nt/2) + 2n + (nt&1)  (NT >= 2)
  //                                         tile0 + n                     (NT == 1)
  // so one 16-byte load per lane per nt pair covers 128 contiguous bytes per row.
  const int bcol = (NT == 1) ? tile0 + g : tile0 + 2 * g;
  const double* a_ptr = tiles + it.a_off + lane;
  double a_cur = (it.nsteps > 0) ? __ldg(a_ptr) : 0.0;
  double b_cur[NT];

  auto load_b = [&](int s, double* bv) {
    int r = 4 * s + t;
    int row = planes ? it.k0 + (r >> 1) : it.k0 + r;
    const double* src = (planes && (r & 1)) ? im : re;
    if (row < nrows) {
      const double* p = src + (int64_t)row * ld + bcol;
      if (NT == 1) {
        bv[0] = (bcol < ncols) ? __ldg(p) : 0.0;
      } else if (full && vec_ok) {
#pragma unroll
        for (int m = 0; m < NT / 2; ++m) {
          double2 v = __ldg(reinterpret_cast<const double2*>(p + 16 * m));
          bv[2 * m] = v.x;
          bv[2 * m + 1] = v.y;
        }
      } else {
#pragma unroll
        for (int m = 0; m < NT / 2; ++m) {
          int c = bcol + 16 * m;
          bv[2 * m] = (c < ncols) ? __ldg(p + 16 * m) : 0.0;
          bv[2 * m + 1] = (c + 1 < ncols) ? __ldg(p + 16 * m + 1) : 0.0;
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < NT; ++i) bv[i] = 0.0;
    }
  };

  if (it.nsteps > 0) load_b(0, b_cur);
  for (int s = 0; s < it.nsteps; ++s) {
    double a_nxt = 0.0;
    double b_nxt[NT];
    const bool more = (s + 1 < it.nsteps);
    if (more) {
      a_nxt = __ldg(a_ptr + 32 * (s + 1));
      load_b(s + 1, b_nxt);
    }
#pragma unroll
    for (int i = 0; i < NT; ++i) dmma(acc[i][0], acc[i][1], a_cur, b_cur[i]);
    if (more) {
      a_cur = a_nxt;
#pragma unroll
      for (int i = 0; i < NT; ++i) b_cur[i] = b_nxt[i];
    }
  }

  // D[g][2t+i] of DMMA nt -> RHS tile0 + 16*(nt/2) + 4t + 2i + (nt&1): 32 contiguous bytes per
  // lane per nt pair (NT == 1: RHS tile0 + 2t + i).
  if (it.cplx) {
    // rows g = 2*bin + comp of 4 complex bins: store u_bin interleaved (re, im) per column in
    // the complex row out_row/2 + bin (= double rows out_row + 2 bin, +1).  Lanes g and g^1 (lane ^ 4)
    // trade halves so that each writes whole complex numbers.
    const bool odd = g & 1;
    double2* crow = reinterpret_cast<double2*>(part + (it.out_row + (g & ~1)) * ldp);
    if (NT == 1) {
      int c = tile0 + 2 * t;
      double snd = odd ? acc[0][0] : acc[0][1];
      double rcv = __shfl_xor_sync(0xffffffffu, snd, 4);
      if (!odd) {
        if (c < ldp) crow[c] = make_double2(acc[0][0], rcv);
      } else {
        if (c + 1 < ldp) crow[c + 1] = make_double2(rcv, acc[0][1]);
      }
    } else {
#pragma unroll
      for (int m = 0; m < NT / 2; ++m) {
        int c = tile0 + 16 * m + 4 * t;
        double v0 = acc[2 * m][0], v1 = acc[2 * m + 1][0], v2 = acc[2 * m][1], v3 = acc[2 * m + 1][1];
        double s0 = odd ? v0 : v2, s1 = odd ? v1 : v3;
        double r0 = __shfl_xor_sync(0xffffffffu, s0, 4), r1 = __shfl_xor_sync(0xffffffffu, s1, 4);
        if (!odd) {
          crow[c] = make_double2(v0, r0);
          crow[c + 1] = make_double2(v1, r1);
        } else {
          crow[c + 2] = make_double2(r0, v2);
          crow[c + 3] = make_double2(r1, v3);
        }
      }
    }
    return;
  }
  double* orow = part + (it.out_row + g) * ldp;
  if (NT == 1) {
    int c = tile0 + 2 * t;
    if (c + 1 < ldp) {
      *reinterpret_cast<double2*>(orow + c) = make_double2(acc[0][0], acc[0][1]);
    } else if (c < ldp) {
      orow[c] = acc[0][0];
    }
  } else {
#pragma unroll
    for (int m = 0; m < NT / 2; ++m) {
      int c = tile0 + 16 * m + 4 * t;
      if (c + 3 < ldp) {
        *reinterpret_cast<double2*>(orow + c) = make_double2(acc[2 * m][0], acc[2 * m + 1][0]);
        *reinterpret_cast<double2*>(orow + c + 2) = make_double2(acc[2 * m][1], acc[2 * m + 1][1]);
      }
    }
  }
}

template <int NT>
xc_status launch(const SpmmItem* items, int nitems, const double* tiles, const SpmmSrcs& srcs, double* part,
                 int64_t ldp, int ncols, cudaStream_t st) {
  dim3 grid((ncols + 8 * NT - 1) / (8 * NT), (nitems + WPC - 1) / WPC);
  if (grid.y > 65535) {
    // fold very long item lists into several launches
    int per = 65535 * WPC;
    for (int i0 = 0; i0 < nitems; i0 += per) {
      int n = std::min(per, nitems - i0);
      XC_TRY(launch<NT>(items + i0, n, tiles, srcs, part, ldp, ncols, st));
    }
    return XC_OK;
  }
  spmm_dmma<NT><<<grid, WPC * 32, 0, st>>>(items, nitems, tiles, srcs, part, ldp, ncols);
  XC_CUDA(cudaGetLastError());
  return XC_OK;
}

__global__ void reduce_rows8_kernel(const double* __restrict__ part, int64_t ldp, const int64_t* __restrict__ base,
                                    const int* __restrict__ nch, int nrows, const double* __restrict__ rowscale,
                                    double* __restrict__ Y, int64_t ldy, int ncols) {
  for (int row = blockIdx.y; row < nrows; row += gridDim.y) {
    int g = row >> 3;
    int n = nch[g];
    int64_t r0 = base[g] + (row & 7);
    double sc = rowscale ? rowscale[row] : 1.0;
    for (int col = blockIdx.x * blockDim.x + threadIdx.x; col < ncols; col += gridDim.x * blockDim.x) {
      double s = 0.0;
      for (int c = 0; c < n; ++c) s += part[(r0 + 8 * c) * ldp + col];
      Y[(int64_t)row * ldy + col] = s * sc;
    }
  }
}

}  // namespace

int spmm_nt_for(int64_t B) {
  if (B >= 128) return 16;
  if (B >= 64) return 8;
  if (B >= 32) return 4;
  if (B >= 16) return 2;
  return 1;
}

xc_status spmm_run(const SpmmItem* items, int nitems, const double* tiles, const SpmmSrcs& srcs, double* part,
                   int64_t ldp, int ncols, cudaStream_t st) {
  if (nitems <= 0) return XC_OK;
  switch (spmm_nt_for(ncols)) {
    case 16: return launch<16>(items, nitems, tiles, srcs, part, ldp, ncols, st);
    case 8: return launch<8>(items, nitems, tiles, srcs, part, ldp, ncols, st);
    case 4: return launch<4>(items, nitems, tiles, srcs, part, ldp, ncols, st);
    case 2: return launch<2>(items, nitems, tiles, srcs, part, ldp, ncols, st);
    default: return launch<1>(items, nitems, tiles, srcs, part, ldp, ncols, st);
  }
}

xc_status reduce_rows8(const double* part, int64_t ldp, const int64_t* base, const int* nch, int nrows,
                       const double* rowscale, double* Y, int64_t ldy, int ncols, cudaStream_t st) {
  if (nrows <= 0) return XC_OK;
  int th = ncols >= 256 ? 256 : (ncols >= 64 ? 64 : 32);
  dim3 grid(std::min((ncols + th - 1) / th, 64), std::min(nrows, 65535));
  reduce_rows8_kernel<<<grid, th, 0, st>>>(part, ldp, base, nch, nrows, rowscale, Y, ldy, ncols);
  XC_CUDA(cudaGetLastError());
  return XC_OK;
}
