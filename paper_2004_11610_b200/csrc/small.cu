// small.cu -- the two-launch apply of small operators (XC_DIR_A, real kinds; c1, c2).
//
// The computation stage of Alg. 2 / its block form for operators whose every
// block fits one CTA's shared memory: there the tiled path (DMMA SpMM over node windows, split-K
// reductions, one or two C2R passes per block, the tail reduction) is launch-bound -- six to ten
// dependent launches for a few microseconds of work.  Here:
//   launch 1 (small_spmm_k): every block's half spectrum u_i[q] = sum_k S_i[k,q] x_k by a
//     bin-major gather (the node bands transposed at build time; nodes ascending, so the sum order
//     is fixed and independent of the batch), and the dense tail rows Y[j] = sum_k phi_j(x_k) x_k
//      straight into Y;
//   launch 2 (small_c2r_k): per (block, column) the real-output inverse DFT of length L = 2M from
//     u in shared memory (the C2R pairing, then Stockham radix stages), times 1/(sqrt(L) w_p) on
//     the kept positions only (W^{-1}, Fe2 discard: P:163-180).
// The choice between this path and the tiled one depends on the operator only (never on B), so a
// column's result does not depend on the batch it is applied in (sharding stays bit-identical).
#include <algorithm>

#include "bfly.cuh"
#include "xc_internal.cuh"

namespace {

using namespace xcb;

// launch 1: rows = every block's bins (complex rows of u) then the tail degrees (real Y rows).
// One launch, two kinds of CTAs (blockIdx.x < nshort: short rows; else long rows):
// * short rows: a CTA of 256 threads takes RB = 256 / (4 CT) rows x CT columns (column tile
//   blockIdx.x % ntile); with STAGE it first copies its CT columns of X to shared memory (N x CT
//   doubles).  Four lanes share a (row, column): each sums a quarter of the row's entries in entry
//   order (nodes ascending) with all its loads issued in one batch, then two shuffles add the
//   quarters as (s0 + s1) + (s2 + s3);
// * long rows (more than kSmallLong entries: the dense tail degrees, the bins of the short blocks
//   that every node touches): one warp per (row, column), lane l sums entries l, l + 32, ... in
//   order, then a fixed shuffle tree.
// Either way the order depends on the row only, never on B: a column's bits do not depend on the
// batch it is applied in.
template <bool STAGE>
__global__ void __launch_bounds__(256, 2) small_spmm_k(const SmallOp op, const double* __restrict__ X, int64_t ldx,
                                                    double2* __restrict__ U, int64_t ldu, double* __restrict__ Y,
                                                    int64_t ldy, int B, int CT, int N, int nshort, int ntile) {
  extern __shared__ double xs[];
  const int tid = threadIdx.x;
  // launch 2 may start now: it only loads its tables before waiting for this grid to complete
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  if ((int)blockIdx.x >= nshort) {  // long rows
    const int64_t pair = (int64_t)(blockIdx.x - nshort) * 8 + (tid >> 5);
    const int lane = tid & 31;
    // a single column (B = 1, c1): X staged in shared memory like the short rows' CTAs
    const bool stx = STAGE && B == 1;
    if (stx) {
      for (int i = tid; i < N; i += 256) xs[i] = __ldg(X + (int64_t)i * ldx);
      __syncthreads();
    }
    if (pair >= (int64_t)op.nlong * B) return;
    const int r = op.longrows[pair / B];
    const int c = (int)(pair % B);
    auto xl = [&](int k) { return stx ? xs[k] : __ldg(X + (int64_t)k * ldx + c); };
    const int64_t e0 = op.ptr[r], e1 = op.ptr[r + 1];
    double re = 0.0, im = 0.0;
    int64_t e = e0 + lane;
    for (; e + 224 < e1; e += 256) {  // eight of this lane's entries in flight, summed in order
      int k[8];
      double2 v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        k[i] = __ldg(op.node + e + 32 * i);
        v[i] = __ldg(op.val + e + 32 * i);
      }
      double x[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = xl(k[i]);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        re = fma(v[i].x, x[i], re);
        im = fma(v[i].y, x[i], im);
      }
    }
    for (; e + 96 < e1; e += 128) {  // four in flight
      const int k0 = __ldg(op.node + e), k1 = __ldg(op.node + e + 32), k2 = __ldg(op.node + e + 64),
                k3 = __ldg(op.node + e + 96);
      const double2 v0 = __ldg(op.val + e), v1 = __ldg(op.val + e + 32), v2 = __ldg(op.val + e + 64),
                    v3 = __ldg(op.val + e + 96);
      const double x0 = xl(k0), x1 = xl(k1), x2 = xl(k2), x3 = xl(k3);
      re = fma(v0.x, x0, re);
      im = fma(v0.y, x0, im);
      re = fma(v1.x, x1, re);
      im = fma(v1.y, x1, im);
      re = fma(v2.x, x2, re);
      im = fma(v2.y, x2, im);
      re = fma(v3.x, x3, re);
      im = fma(v3.y, x3, im);
    }
    for (; e < e1; e += 32) {
      const double x = xl(__ldg(op.node + e));
      const double2 v = __ldg(op.val + e);
      re = fma(v.x, x, re);
      im = fma(v.y, x, im);
    }
    for (int o = 16; o > 0; o >>= 1) {
      re += __shfl_xor_sync(0xffffffffu, re, o);
      im += __shfl_xor_sync(0xffffffffu, im, o);
    }
    if (lane == 0) {
      const int64_t o = op.out[r];
      if (o >= 0) U[o * ldu + c] = make_double2(re, im);
      else Y[(-o - 1) * ldy + c] = re;
    }
    return;
  }
  const int c0 = ((int)blockIdx.x % ntile) * CT;
  if (STAGE) {
    for (int i = tid; i < N * CT; i += 256) {
      const int k = i / CT, lc = i - k * CT;
      xs[i] = (c0 + lc < B) ? __ldg(X + (int64_t)k * ldx + c0 + lc) : 0.0;
    }
    __syncthreads();
  }
  // kSmallSub adjacent lanes per (row, column): sub-lane j sums the j-th quarter of the row's
  // entries in entry order (all of its loads in one batch), then (s0 + s1) + (s2 + s3) by two xor
  // shuffles -- a fixed order per row, independent of B and of the CTA shape
  const int sub = tid % kSmallSub, t = tid / kSmallSub;
  const int r = ((int)blockIdx.x / ntile) * (256 / (CT * kSmallSub)) + t / CT;
  const int lc = t % CT, c = c0 + lc;
  const bool live = r < op.rows && c < B;
  int64_t e0 = 0, e1 = 0;
  if (live) {
    e0 = op.ptr[r];
    e1 = op.ptr[r + 1];
  }
  const bool longrow = e1 - e0 > kSmallLong;  // a long row (the warp CTAs take it)
  auto xv = [&](int k) { return STAGE ? xs[k * CT + lc] : __ldg(X + (int64_t)k * ldx + c); };
  const int q = (int)((e1 - e0 + kSmallSub - 1) / kSmallSub);  // <= kSmallLong / kSmallSub
  const int64_t s0 = e0 + (int64_t)sub * q, s1 = min(e1, s0 + q);
  double re = 0.0, im = 0.0;
  if (live && !longrow) {
    constexpr int Q = kSmallLong / kSmallSub;
    int k[Q];
    double2 v[Q];
#pragma unroll
    for (int i = 0; i < Q; ++i) {
      const bool in = s0 + i < s1;
      k[i] = in ? __ldg(op.node + s0 + i) : 0;
      v[i] = in ? __ldg(op.val + s0 + i) : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int i = 0; i < Q; ++i) {
      if (s0 + i < s1) {
        const double x = xv(k[i]);
        re = fma(v[i].x, x, re);
        im = fma(v[i].y, x, im);
      }
    }
  }
  // lanes of one (row, column) are adjacent and share live / longrow, so whole groups of
  // kSmallSub lanes take part in each shuffle
  re += __shfl_xor_sync(0xffffffffu, re, 1);
  im += __shfl_xor_sync(0xffffffffu, im, 1);
  re += __shfl_xor_sync(0xffffffffu, re, 2);
  im += __shfl_xor_sync(0xffffffffu, im, 2);
  if (!live || longrow || sub != 0) return;
  const int64_t o = op.out[r];
  if (o >= 0) U[o * ldu + c] = make_double2(re, im);   // u row of a block
  else Y[(-o - 1) * ldy + c] = re;                     // tail degree -o-1
}

// One Stockham radix-r stage over M points: in -> out, twiddles w_M^{t k M/(Ns r)} from tw (M entries).
template <int r>
__device__ __forceinline__ void small_stage(const double2* in, double2* out, const double2* tw, int M,
                                            int Ns) {
  const int Mr = M / r, step = M / (Ns * r);
  for (int j = threadIdx.x; j < Mr; j += blockDim.x) {
    const int k = j % Ns;
    double2 v[r];
#pragma unroll
    for (int t = 0; t < r; ++t) v[t] = in[j + t * Mr];
    if (Ns > 1) {
#pragma unroll
      for (int t = 1; t < r; ++t) v[t] = c_mul(v[t], tw[t * k * step]);
    }
    bfly<r>(v);
    const int d = (j / Ns) * Ns * r + k;
#pragma unroll
    for (int t = 0; t < r; ++t) out[d + t * Ns] = v[t];
  }
}

// launch 2: CTA (block i, column c).  Shared: A (H complex; u, then a ping-pong buffer), Bf (M), the
// stage twiddles (M) and, with STG, the pairing twiddles (M) and the kept positions' scales.
// Launched with programmatic dependent launch: everything that does not depend on u (the tables)
// is loaded before griddepcontrol.wait, i.e. while launch 1 still runs.
template <bool STG>
__global__ void __launch_bounds__(1024) small_c2r_k(const SmallBlocks sb, const double2* __restrict__ U, int64_t ldu,
                                                   double* __restrict__ Y, int64_t ldy) {
  extern __shared__ double2 sm[];
  const SmallBlk b = sb.blk[blockIdx.x];
  const int c = blockIdx.y;
  const int M = b.M;
  double2* A = sm;
  double2* Bf = sm + b.M + 1;
  double2* tw = Bf + b.M;  // the stage twiddles e^{2 pi i n / M}, staged once (one coalesced pass)
  double2* th = tw + b.M;  // STG: the pairing twiddles e^{i pi n / M}
  double* ys = reinterpret_cast<double*>(th + b.M);  // STG: yscale[keep_lo + i]
  for (int n = threadIdx.x; n < M; n += blockDim.x) {
    tw[n] = __ldg(b.twM + n);
    if (STG) th[n] = __ldg(b.twh + n);
  }
  if (STG)
    for (int p = b.keep_lo + threadIdx.x; p < b.keep_hi; p += blockDim.x) ys[p - b.keep_lo] = __ldg(b.yscale + p);
  asm volatile("griddepcontrol.wait;\n" ::: "memory");  // launch 1's u (and tail rows) complete
  const double2* u = U + b.urow * ldu + c;
  for (int q = threadIdx.x; q <= M; q += blockDim.x) A[q] = u[(int64_t)q * ldu];
  __syncthreads();
  // pairing: Z[n] = (u_n + conj u_{M-n}) + i e^{i pi n / M} (u_n - conj u_{M-n})
  for (int n = threadIdx.x; n < M; n += blockDim.x) {
    const double2 a = A[n], p = A[M - n], w = STG ? th[n] : __ldg(b.twh + n);
    const double evr = a.x + p.x, evi = a.y - p.y, dr = a.x - p.x, di = a.y + p.y;
    const double odr = dr * w.x - di * w.y, odi = dr * w.y + di * w.x;
    Bf[n] = make_double2(evr - odi, evi + odr);
  }
  __syncthreads();
  double2* in = Bf;
  double2* out = A;
  int Ns = 1;
  for (int s = 0; s < b.nf; ++s) {
    const int r = b.f[s];
    switch (r) {
      case 2: small_stage<2>(in, out, tw, M, Ns); break;
      case 3: small_stage<3>(in, out, tw, M, Ns); break;
      case 4: small_stage<4>(in, out, tw, M, Ns); break;
      case 5: small_stage<5>(in, out, tw, M, Ns); break;
      case 6: small_stage<6>(in, out, tw, M, Ns); break;
      case 9: small_stage<9>(in, out, tw, M, Ns); break;
      default: small_stage<8>(in, out, tw, M, Ns); break;
    }
    Ns *= r;
    __syncthreads();
    double2* t = in;
    in = out;
    out = t;
  }
  // z_k = in[k]: v[2k] = Re z_k, v[2k+1] = Im z_k; Y[p + m_off] = v[p] yscale[p], p in [keep_lo, keep_hi)
  for (int p = b.keep_lo + threadIdx.x; p < b.keep_hi; p += blockDim.x) {
    const double2 z = in[p >> 1];
    Y[(int64_t)(p + b.m_off) * ldy + c] = ((p & 1) ? z.y : z.x) * (STG ? ys[p - b.keep_lo] : __ldg(b.yscale + p));
  }
}

}  // namespace

xc_status small_spmm(const SmallOp& op, const double* X, int64_t ldx, double2* U, int64_t ldu, double* Y, int64_t ldy,
                     int B, int N, cudaStream_t st) {
  int CT = 1;
  while (CT < 32 && CT < B) CT *= 2;
  // stage the CTA's columns of X in shared memory when they fit 48 KB (c1: 4 KB), else L1/L2
  const bool stage = (size_t)N * CT * sizeof(double) <= 48 * 1024;
  for (int c0 = 0; c0 < B; c0 += 65535) {  // keeps the 1D grid small
    const int bc = std::min(B - c0, 65535);
    const int ntile = (bc + CT - 1) / CT;
    const int rb = 256 / (CT * kSmallSub);  // short rows per CTA
    const int64_t nshort = (int64_t)((op.rows + rb - 1) / rb) * ntile;
    const int64_t nlong = ((int64_t)op.nlong * bc + 7) / 8;
    const unsigned grid = (unsigned)(nshort + nlong);
    if (stage)
      small_spmm_k<true><<<grid, 256, (size_t)N * CT * sizeof(double), st>>>(op, X + c0, ldx, U + c0, ldu, Y + c0,
                                                                              ldy, bc, CT, N, (int)nshort, ntile);
    else
      small_spmm_k<false><<<grid, 256, 0, st>>>(op, X + c0, ldx, U + c0, ldu, Y + c0, ldy, bc, CT, N, (int)nshort,
                                                 ntile);
    XC_CUDA(cudaGetLastError());
  }
  return XC_OK;
}

xc_status small_c2r(const SmallBlocks& sb, const double2* U, int64_t ldu, double* Y, int64_t ldy, int B,
                    cudaStream_t st) {
  if (sb.nb == 0) return XC_OK;
  int maxk = 0;  // the longest kept range
  for (int i = 0; i < sb.nb; ++i) maxk = std::max(maxk, sb.blk[i].keep_hi - sb.blk[i].keep_lo);
  const size_t base = (size_t)(3 * sb.maxM + 1) * sizeof(double2);
  const size_t full = base + (size_t)sb.maxM * sizeof(double2) + (size_t)maxk * sizeof(double);
  const bool stg = full <= 200 * 1024;
  const size_t smem = stg ? full : base;
  static std::atomic<unsigned long long> once{0};
  if (first_on_device(once)) {
    XC_CUDA(cudaFuncSetAttribute(small_c2r_k<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (3 * kSmallMaxM + 1) * (int)sizeof(double2)));
    XC_CUDA(cudaFuncSetAttribute(small_c2r_k<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  }
  const int nth = sb.maxM >= 2048 ? 1024 : (sb.maxM >= 512 ? 512 : 256);  // one CTA per column: latency
  for (int c0 = 0; c0 < B; c0 += 65535) {  // grid.y limit
    // programmatic dependent launch on the gather (launch 1) that precedes it on the stream
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(sb.nb, std::min(B - c0, 65535));
    cfg.blockDim = dim3(nth);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (stg) XC_CUDA(cudaLaunchKernelEx(&cfg, small_c2r_k<true>, sb, U + c0, ldu, Y + c0, ldy));
    else XC_CUDA(cudaLaunchKernelEx(&cfg, small_c2r_k<false>, sb, U + c0, ldu, Y + c0, ldy));
  }
  return XC_OK;
}

bool small_radices(int M, int* f, int& nf) {
  nf = 0;
  int x = M;
  for (int r : {8, 9, 6, 4, 2, 5, 3})
    while (x % r == 0 && nf < 16) {
      f[nf++] = r;
      x /= r;
    }
  return x == 1;
}
