// spmm.cu -- multiplication by the compressed operator on the FP64 tensor cores.
//
// The hot step of the computation stage (u = Ä_e^T F, Alg. 2 step 2.1, P:218;
// F = Ä_e z, Alg. 1 step 2.2; per block P:281).  "The degree of compression
// ... determines to a great extent the efficiency of the computation step".
//
// The band-sparse operator is pre-tiled (build.cu) into items: an item is a pair of
// 8 x (4*nsteps) dense slices A of the operator (8 output rows = 4 complex bins as re/im,
// or 8 real rows) against 4*nsteps consecutive rows of the operand Bm; items are grouped
// into windows of B rows that one CTA stages in shared memory (the X rows of a node window
// are shared by every block's bins that touch those nodes).
// One warp computes D = A * Bm for 8*NT right-hand sides with DMMA
// (mma.sync.m8n8k4.f64: 37 TF/s measured on B200 vs 34 TF/s for DFMA):
//   A fragment  : lane holds A[lane/4][lane%4]     (one coalesced 256 B load/step)
//   B fragment  : lane holds Bm[lane%4][n], n = lane/4; for DMMA nt the column n is
//                 RHS tile + 16*(nt/2) + 2n + (nt&1): each 16-byte load covers a 128-byte
//                 contiguous run of a row across 8 lanes (coalesced);
//   D fragment  : lane holds D[lane/4][2(lane%4)+i] -> 32 contiguous bytes per nt pair.
// Partial sums of items that split one output group are reduced in fixed order by
// the consumer (FFT prologue / reduce_rows8), so results are deterministic.
#include <stdlib.h>

#include <algorithm>

#include "xc_internal.cuh"

namespace {

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

constexpr int WARPS = XC_WARPS;  // warps per CTA
// zero rows staged after every window: a step past an item's end (the zero A step that pads an odd
// step count, the B-fragment load one step ahead) reads them, so the step loop has no branches
constexpr int kPadRows = 8;

// 32-byte read-only load (LDG.256 on sm_100)
__device__ __forceinline__ double4 ldg4(const double* p) {
  double4 v;
  asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
  return v;
}

// One CTA = one window of B rows [r0, r1) (<= XC_WMAX) x one tile of 8*NT right-hand sides.
// The window's rows are staged once in shared memory; the window's items (all families whose
// B rows lie inside it) are spread over the warps.  Each item holds 2 M-tiles sharing the B
// fragments (2 x NT DMMAs per 4-row step).  B fragments come from shared memory (one step
// ahead), A fragments stream from global memory two steps ahead.
template <int NT, bool PF>
__global__ void __launch_bounds__(WARPS * 32, 2)
    spmm_win(const SpmmWin* __restrict__ wins, const SpmmItem* __restrict__ items,
             const double* __restrict__ tiles, SpmmSrcs srcs, double* __restrict__ part, int64_t ldp, int ncols) {
  constexpr int CW = 8 * NT;   // columns per tile
  constexpr int CWP = CW + 4;  // padded smem row: the 4 rows of a B fragment fall in distinct banks
  extern __shared__ double2 xs2[];
  const double* xs = reinterpret_cast<const double*>(xs2);
  SpmmWin W;  // scalar fields only (the per-warp offsets are read where needed)
  W.r0 = wins[blockIdx.y].r0;
  W.r1 = wins[blockIdx.y].r1;
  W.i0 = wins[blockIdx.y].i0;
  W.i1 = wins[blockIdx.y].i1;
  W.src = wins[blockIdx.y].src;
  // the window's item descriptors, staged next to the X window (8-byte cp.async pieces)
  SpmmItem* its = reinterpret_cast<SpmmItem*>(xs2 + (XC_WMAX + kPadRows) * ((8 * NT + 4) / 2));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int t = lane & 3, g = lane >> 2;
  const int tile0 = blockIdx.x * CW;

  // ---- stage the window: rows [r0, r1) x columns [tile0, tile0 + CW) ----
  {
    const double* re = srcs.re[W.src];
    const double* im = srcs.im[W.src];
    const int nrows = srcs.nrows[W.src];
    const int64_t ld = srcs.ld[W.src];
    const int nr = W.r1 - W.r0;
    const bool vec = (NT >= 2) && ((ld & 1) == 0) && ((((uintptr_t)re) & 15) == 0) &&
                     (!im || (((uintptr_t)im) & 15) == 0) && (tile0 + CW <= ncols);
    if (vec) {
      // cp.async: every 16-byte piece of the window in flight at once (no register round trip;
      // rows past the source are zero-filled)
      for (int idx = tid; idx < (nr + kPadRows) * (CW / 2); idx += WARPS * 32) {
        int rl = idx / (CW / 2), c2 = idx - rl * (CW / 2);
        int R = W.r0 + rl;
        int row = im ? (R >> 1) : R;
        const double* src = (im && (R & 1)) ? im : re;
        const bool ok = row < nrows && rl < nr;
        const double2* g = reinterpret_cast<const double2*>(src + (int64_t)(ok ? row : 0) * ld + tile0) + c2;
        const unsigned sa = (unsigned)__cvta_generic_to_shared(&xs2[rl * (CWP / 2) + c2]);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(g), "r"(ok ? 16 : 0));
      }
    } else {
      double* xw = reinterpret_cast<double*>(xs2);
      for (int idx = tid; idx < (nr + kPadRows) * CW; idx += WARPS * 32) {
        int rl = idx / CW, c = idx - rl * CW;
        int R = W.r0 + rl;
        int row = im ? (R >> 1) : R;
        const double* src = (im && (R & 1)) ? im : re;
        xw[rl * CWP + c] =
            (rl < nr && row < nrows && tile0 + c < ncols) ? __ldg(src + (int64_t)row * ld + tile0 + c) : 0.0;
      }
    }
    constexpr int IW = sizeof(SpmmItem) / 8;
    const int nit = (W.i1 - W.i0) * IW;
    const double* isrc = reinterpret_cast<const double*>(items + W.i0);
    double* idst = reinterpret_cast<double*>(its);
    for (int q = tid; q < nit; q += WARPS * 32) {
      const unsigned sa = (unsigned)__cvta_generic_to_shared(idst + q);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(isrc + q));
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::);
  }
  __syncthreads();

  // B-fragment column n of DMMA nt: 16 (nt/2) + 2n + (nt&1) within the tile (NT >= 2), n (NT == 1)
  const int bcol = (NT == 1) ? g : 2 * g;

  const int iw0 = W.i0 + __ldg(&wins[blockIdx.y].wo[warp]), iw1 = W.i0 + __ldg(&wins[blockIdx.y].wo[warp + 1]);
  for (int ii = iw0; ii < iw1; ++ii) {
    const SpmmItem it = its[ii - W.i0];
    // PF (grids of a few waves, c3): at an item's start its A stream beyond the first 4 steps and
    // the next item's first 4 steps are prefetched into L2 (128-B lines, lane l takes lines l,
    // l + 32, ...): the 4-step register prefetch does not cover a DRAM first touch (c3 SpMM
    // 0.120 -> 0.111 ms; on the long c5 grid it costs more than it gains: 6.65 -> 6.82 ms)
    if constexpr (PF) {
      const char* ab = reinterpret_cast<const char*>(tiles + it.a_off);
      for (int q = 16 + lane; q < 4 * it.nsteps; q += 32) asm volatile("prefetch.global.L2 [%0];" ::"l"(ab + 128 * q));
      if (ii + 1 < iw1 && lane < 16) {
        const SpmmItem& nx = its[ii + 1 - W.i0];
        if (lane < 4 * nx.nsteps)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const char*>(tiles + nx.a_off) + 128 * lane));
      }
    }
    double acc[2][NT][2];
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
      for (int i = 0; i < NT; ++i) acc[m][i][0] = acc[m][i][1] = 0.0;
    const double* xb = xs + (it.k0 - W.r0 + t) * CWP + bcol;
    const int n = it.nsteps;
    double b0[NT], b1[NT];
    auto lds_b = [&](int s, double* bv) {
      const double* p = xb + 4 * s * CWP;
      if (NT == 1) {
        bv[0] = p[0];
      } else {
#pragma unroll
        for (int m = 0; m < NT / 2; ++m) {
          double2 v = *reinterpret_cast<const double2*>(p + 16 * m);
          bv[2 * m] = v.x;
          bv[2 * m + 1] = v.y;
        }
      }
    };
#pragma unroll
    for (int i = 0; i < NT; ++i) b0[i] = b1[i] = 0.0;
    if (n > 0) lds_b(0, b0);
    if (it.out_row[1] >= 0) {
      // two M-tiles sharing the B fragments
      // A fragments streamed four steps ahead, two steps per 32-byte load (the tile stream holds
      // steps 2k, 2k+1 of a lane as (slot 0, slot 1, slot 0, slot 1): build.cu)
      const double* ap = tiles + it.a_off + 4 * lane;
      const double4 z4 = make_double4(0.0, 0.0, 0.0, 0.0);
      double4 a01 = n > 0 ? ldg4(ap) : z4, a23 = n > 2 ? ldg4(ap + 128) : z4;
      int s = 0;
      for (; s + 1 < n; s += 2) {  // step pairs, no bounds branches (the B load one step ahead may read pad rows)
        lds_b(s + 1, b1);
#pragma unroll
        for (int i = 0; i < NT; ++i) {
          dmma(acc[0][i][0], acc[0][i][1], a01.x, b0[i]);
          dmma(acc[1][i][0], acc[1][i][1], a01.y, b0[i]);
        }
        lds_b(s + 2, b0);
#pragma unroll
        for (int i = 0; i < NT; ++i) {
          dmma(acc[0][i][0], acc[0][i][1], a01.z, b1[i]);
          dmma(acc[1][i][0], acc[1][i][1], a01.w, b1[i]);
        }
        a01 = a23;
        a23 = (s + 4 < n) ? ldg4(ap + 64 * (s + 4)) : z4;
      }
      if (s < n) {  // odd n: the last step alone (b0 and a01.xy hold it)
#pragma unroll
        for (int i = 0; i < NT; ++i) {
          dmma(acc[0][i][0], acc[0][i][1], a01.x, b0[i]);
          dmma(acc[1][i][0], acc[1][i][1], a01.y, b0[i]);
        }
      }
    } else {
      // one M-tile (slot 0 of the A stream), A fragments streamed 4 steps ahead, two per load
      const double* ap = tiles + it.a_off + 4 * lane;
      const double4 z4 = make_double4(0.0, 0.0, 0.0, 0.0);
      double4 a01 = n > 0 ? ldg4(ap) : z4, a23 = n > 2 ? ldg4(ap + 128) : z4;
      int s = 0;
      for (; s + 1 < n; s += 2) {
        lds_b(s + 1, b1);
#pragma unroll
        for (int i = 0; i < NT; ++i) dmma(acc[0][i][0], acc[0][i][1], a01.x, b0[i]);
        lds_b(s + 2, b0);
#pragma unroll
        for (int i = 0; i < NT; ++i) dmma(acc[0][i][0], acc[0][i][1], a01.z, b1[i]);
        a01 = a23;
        a23 = (s + 4 < n) ? ldg4(ap + 64 * (s + 4)) : z4;
      }
      if (s < n) {
#pragma unroll
        for (int i = 0; i < NT; ++i) dmma(acc[0][i][0], acc[0][i][1], a01.x, b0[i]);
      }
    }

    // ---- store the two 8 x CW output tiles ----
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      if (it.out_row[mt] < 0) continue;
      if (it.cplx) {
        // rows g = 2 bin + comp of 4 complex bins -> complex row (out_row + 2 bin) / 2, interleaved
        // (re, im) per column; lanes g, g^1 (lane ^ 4) trade halves to write whole numbers.
        const bool odd = g & 1;
        double2* crow = reinterpret_cast<double2*>(part + (it.out_row[mt] + (g & ~1)) * ldp);
        if (NT == 1) {
          int c = tile0 + 2 * t;
          double snd = odd ? acc[mt][0][0] : acc[mt][0][1];
          double rcv = __shfl_xor_sync(0xffffffffu, snd, 4);
          if (!odd) {
            if (c < ldp) __stcs(crow + c, make_double2(acc[mt][0][0], rcv));
          } else {
            if (c + 1 < ldp) __stcs(crow + c + 1, make_double2(rcv, acc[mt][0][1]));
          }
        } else {
#pragma unroll
          for (int m = 0; m < NT / 2; ++m) {
            int c = tile0 + 16 * m + 4 * t;
            double v0 = acc[mt][2 * m][0], v1 = acc[mt][2 * m + 1][0];
            double v2 = acc[mt][2 * m][1], v3 = acc[mt][2 * m + 1][1];
            double s0 = odd ? v0 : v2, s1 = odd ? v1 : v3;
            double r0 = __shfl_xor_sync(0xffffffffu, s0, 4), r1 = __shfl_xor_sync(0xffffffffu, s1, 4);
            // one 32-byte store per lane (two adjacent complex numbers; STG.256 on sm_100)
            double* q = reinterpret_cast<double*>(crow + c + (odd ? 2 : 0));
            const double q0 = odd ? r0 : v0, q1 = odd ? v2 : r0, q2 = odd ? r1 : v1, q3 = odd ? v3 : r1;
            asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(q), "d"(q0), "d"(q1), "d"(q2), "d"(q3)
                         : "memory");
          }
        }
      } else {
        double* orow = part + (it.out_row[mt] + g) * ldp;
        if (NT == 1) {
          int c = tile0 + 2 * t;
          if (c + 1 < ldp) *reinterpret_cast<double2*>(orow + c) = make_double2(acc[mt][0][0], acc[mt][0][1]);
          else if (c < ldp) orow[c] = acc[mt][0][0];
        } else {
#pragma unroll
          for (int m = 0; m < NT / 2; ++m) {
            int c = tile0 + 16 * m + 4 * t;
            asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(orow + c), "d"(acc[mt][2 * m][0]),
                         "d"(acc[mt][2 * m + 1][0]), "d"(acc[mt][2 * m][1]), "d"(acc[mt][2 * m + 1][1])
                         : "memory");
          }
        }
      }
    }
  }
}

template <int NT>
xc_status launch(const SpmmWin* wins, int nwins, const SpmmItem* items, const double* tiles, const SpmmSrcs& srcs,
                 double* part, int64_t ldp, int ncols, cudaStream_t st) {
  const size_t sm =
      (size_t)(XC_WMAX + kPadRows) * (8 * NT + 4) * sizeof(double) + (size_t)XC_WIN_ITEMS * sizeof(SpmmItem);
  static std::atomic<unsigned long long> once{0};
  if (first_on_device(once)) {
    XC_CUDA(cudaFuncSetAttribute(spmm_win<NT, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    XC_CUDA(cudaFuncSetAttribute(spmm_win<NT, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  }
  // the A-stream L2 prefetch instance (XC_SPMM_PF=1; measurement switch).  It paid on grids of 1 to
  // 16 waves with 16-byte A loads (c3 +3 %); with the 32-byte step-pair loads it no longer does
  // (c3 0.1045 vs 0.1049 ms, c4 1.267 vs 1.245 ms without it), so it is off by default
  static const int force = getenv("XC_SPMM_PF") ? atoi(getenv("XC_SPMM_PF")) : -1;
  const bool pf = force > 0;
  for (int w0 = 0; w0 < nwins; w0 += 65535) {
    int nw = std::min(65535, nwins - w0);
    dim3 grid((ncols + 8 * NT - 1) / (8 * NT), nw);
    if (pf) spmm_win<NT, true><<<grid, WARPS * 32, sm, st>>>(wins + w0, items, tiles, srcs, part, ldp, ncols);
    else spmm_win<NT, false><<<grid, WARPS * 32, sm, st>>>(wins + w0, items, tiles, srcs, part, ldp, ncols);
    XC_CUDA(cudaGetLastError());
  }
  return XC_OK;
}

constexpr int kRedBatch = 16;
constexpr int kRedDeepMin = 48;  // chains at least this long take the deep instance

template <bool DEEP>
__global__ void reduce_rows8_kernel(const double* __restrict__ part, int64_t ldp, const int64_t* __restrict__ base,
                                    const int* __restrict__ nch, int nrows, const double* __restrict__ rowscale,
                                    double* __restrict__ Y, int64_t ldy, int ncols) {
  for (int row = blockIdx.y; row < nrows; row += gridDim.y) {
    int g = row >> 3;
    int n = nch[g];
    if (n < 0) continue;  // a group whose SpMM item wrote the rows directly
    int64_t r0 = base[g] + (row & 7);
    double sc = rowscale ? rowscale[row] : 1.0;
    for (int col = blockIdx.x * blockDim.x + threadIdx.x; col < ncols; col += gridDim.x * blockDim.x) {
      // summed in chunk order (the same rounding as the plain loop).  Long chains (the small-L
      // blocks and the tail: up to N / 184 chunks) are latency bound, so the loads run two
      // batches of 16 ahead of the adds (c5 block 8: 356 chunks, 72 us at four in flight)
      const double* p = part + r0 * ldp + col;
      const int64_t st = 8 * ldp;
      double s = 0.0;
      int c = 0;
      if (DEEP && n >= 2 * kRedBatch) {
        double a[kRedBatch];
#pragma unroll
        for (int i = 0; i < kRedBatch; ++i) a[i] = __ldcs(p + (c + i) * st);
        for (c = kRedBatch; c + kRedBatch <= n; c += kRedBatch) {
          double b[kRedBatch];
#pragma unroll
          for (int i = 0; i < kRedBatch; ++i) b[i] = __ldcs(p + (c + i) * st);
#pragma unroll
          for (int i = 0; i < kRedBatch; ++i) s += a[i];
#pragma unroll
          for (int i = 0; i < kRedBatch; ++i) a[i] = b[i];
        }
#pragma unroll
        for (int i = 0; i < kRedBatch; ++i) s += a[i];
      }
      for (; c + 4 <= n; c += 4) {
        const double v0 = __ldcs(p + c * st), v1 = __ldcs(p + (c + 1) * st);
        const double v2 = __ldcs(p + (c + 2) * st), v3 = __ldcs(p + (c + 3) * st);
        s += v0;
        s += v1;
        s += v2;
        s += v3;
      }
      for (; c < n; ++c) s += __ldcs(p + c * st);
      Y[(int64_t)row * ldy + col] = s * sc;
    }
  }
}

}  // namespace

int spmm_nt_for(int64_t B) {
  static const int force = getenv("XC_SPMM_NT") ? atoi(getenv("XC_SPMM_NT")) : 0;  // experiment
  if (force == 1 || force == 2 || force == 4 || force == 8) return (8 * force <= B || force == 1) ? force : 1;
  if (B >= 64) return 8;
  if (B >= 32) return 4;
  if (B >= 16) return 2;
  return 1;
}

xc_status spmm_run(const SpmmWin* wins, int nwins, const SpmmItem* items, const double* tiles,
                   const SpmmSrcs& srcs, double* part, int64_t ldp, int ncols, cudaStream_t st) {
  if (nwins <= 0) return XC_OK;
  // RHS tile: 8 NT columns; a grid smaller than two CTAs per SM takes narrower tiles (more
  // CTAs: c2 0.020 -> 0.013 ms), never below 16 columns
  int nt = spmm_nt_for(ncols);
  static const bool forced = getenv("XC_SPMM_NT") != nullptr;
  while (!forced && nt > 2 && (int64_t)nwins * ((ncols + 8 * nt - 1) / (8 * nt)) < 2 * (int64_t)sm_count()) nt /= 2;
  switch (nt) {
    case 8: return launch<8>(wins, nwins, items, tiles, srcs, part, ldp, ncols, st);
    case 4: return launch<4>(wins, nwins, items, tiles, srcs, part, ldp, ncols, st);
    case 2: return launch<2>(wins, nwins, items, tiles, srcs, part, ldp, ncols, st);
    default: return launch<1>(wins, nwins, items, tiles, srcs, part, ldp, ncols, st);
  }
}

xc_status reduce_rows8(const double* part, int64_t ldp, const int64_t* base, const int* nch, int nrows,
                       const double* rowscale, double* Y, int64_t ldy, int ncols, int maxn, cudaStream_t st) {
  if (nrows <= 0) return XC_OK;
  int th = ncols >= 256 ? 256 : (ncols >= 64 ? 64 : 32);
  dim3 grid(std::min((ncols + th - 1) / th, 64), std::min(nrows, 65535));
  // the deep instance (86 registers) only where chains are long: short chains (c5 block 3, ~2
  // chunks, HBM bound) need the occupancy of the 32-register one
  if (maxn >= kRedDeepMin)
    reduce_rows8_kernel<true><<<grid, th, 0, st>>>(part, ldp, base, nch, nrows, rowscale, Y, ldy, ncols);
  else
    reduce_rows8_kernel<false><<<grid, th, 0, st>>>(part, ldp, base, nch, nrows, rowscale, Y, ldy, ncols);
  XC_CUDA(cudaGetLastError());
  return XC_OK;
}
